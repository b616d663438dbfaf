IABN_FUSED_MIS=1 IABN_PDL=0 timeout 120 python tools/shape_graph.py --layout NCHW --dtype bf16 --shapes 128x196 > gpurun_out/p87a.log 2>&1; echo rc=$? >> gpurun_out/p87a.log
IABN_FUSED_MIS=1 IABN_PDL=1 timeout 120 python tools/shape_graph.py --layout NCHW --dtype bf16 --shapes 128x196 > gpurun_out/p87b.log 2>&1; echo rc=$? >> gpurun_out/p87b.log
IABN_FUSED_MIS=1 IABN_PDL=1 timeout 120 python tools/shape_graph.py --layout NCHW --dtype bf16 --shapes 128x196 --N 8 > gpurun_out/p87c.log 2>&1; echo rc=$? >> gpurun_out/p87c.log
echo done
