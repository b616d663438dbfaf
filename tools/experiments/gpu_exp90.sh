timeout 600 python -m pytest tests -m gpu -q --timeout 300 -p no:cacheprovider -k "misaligned" > gpurun_out/gpu_tests.log 2>&1; echo rc=$? >> gpurun_out/gpu_tests.log
for m in 0 1; do
  IABN_FUSED_MIS=$m timeout 300 python tools/shape_graph.py --layout NCHW --dtype bf16 --shapes 512x196,1024x196,128x196,1024x49,2048x49,128x49 > gpurun_out/sg90_$m.json 2>&1
  IABN_FUSED_MIS=$m timeout 300 python tools/shape_graph.py --layout NCHW --dtype f32 --shapes 1024x49,2048x49,128x49 > gpurun_out/sg90f_$m.json 2>&1
done
echo done
