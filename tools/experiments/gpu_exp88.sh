IABN_FUSED_MIS=1 IABN_PDL=0 timeout 120 python tools/shape_graph.py --layout NCHW --dtype bf16 --shapes 512x196 > gpurun_out/p88a.log 2>&1; echo rc=$? >> gpurun_out/p88a.log
IABN_FUSED_MIS=1 IABN_PDL=1 timeout 120 python tools/shape_graph.py --layout NCHW --dtype bf16 --shapes 1024x49 > gpurun_out/p88b.log 2>&1; echo rc=$? >> gpurun_out/p88b.log
IABN_FUSED_MIS=1 IABN_PDL=1 IABN_VERBOSE=1 timeout 120 python tools/shape_graph.py --layout NCHW --dtype bf16 --shapes 512x196 > gpurun_out/p88c.log 2>&1; echo rc=$? >> gpurun_out/p88c.log
echo done
