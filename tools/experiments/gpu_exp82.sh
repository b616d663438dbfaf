timeout 1100 python -m pytest tests -m gpu -q --timeout 600 -p no:cacheprovider > gpurun_out/gpu_tests.log 2>&1; echo rc=$? >> gpurun_out/gpu_tests.log
timeout 600 python tools/shape_graph.py --layout NHWC --dtype bf16 --shapes 64x3136,128x3136,256x784,128x784,128x196,128x49,512x196,1024x196 > gpurun_out/sg82.json 2>&1
timeout 600 python tools/shape_graph.py --layout NCHW --dtype bf16 --shapes 512x196,1024x196,128x49,1024x49 > gpurun_out/sg82n.json 2>&1
for cfg in "densenet264 bf16 NHWC" "rx101 bf16 NCHW" "rx101 f32 NHWC"; do
  set -- $cfg
  timeout 600 python tools/sweep.py --net $1 --dtype $2 --layout $3 > gpurun_out/sw82_$1_$2_$3.json 2> gpurun_out/sw82_$1_$2_$3.err
done
echo done
