for g in 0 1; do
  IABN_GRES=$g timeout 600 python tools/shape_graph.py --layout NHWC --dtype bf16 --shapes 64x3136,128x3136,256x784,128x784,128x196,128x49,512x196,1024x196 > gpurun_out/sg81_$g.json 2>&1
  IABN_GRES=$g timeout 600 python tools/shape_graph.py --layout NHWC --dtype f32 --shapes 64x3136,128x3136,256x784,512x196,1024x49 > gpurun_out/sg81f_$g.json 2>&1
done
echo done
