for m in 0 1; do
  IABN_FUSED_MIS=$m timeout 600 python tools/shape_graph.py --layout NCHW --dtype bf16 --shapes 512x196,1024x196,128x196,1024x49,2048x49,128x49 > gpurun_out/sg84_$m.json 2>&1
  IABN_FUSED_MIS=$m timeout 600 python tools/shape_graph.py --layout NCHW --dtype f32 --shapes 1024x49,2048x49,128x49 > gpurun_out/sg84f_$m.json 2>&1
done
timeout 600 python tools/shape_graph.py --layout NCHW --dtype f32 --shapes 512x196,1024x196,128x196,256x784 > gpurun_out/sg84a.json 2>&1
echo done
