for sh in 1024x196 2048x49; do
IABN_FUSED_MIS=1 IABN_VERBOSE=1 timeout 90 python tools/shape_graph.py --layout NCHW --dtype bf16 --shapes $sh > gpurun_out/p89_$sh.log 2>&1; echo rc=$? >> gpurun_out/p89_$sh.log
IABN_FUSED_MIS=1 IABN_VERBOSE=1 timeout 60 python tools/layer_probe.py 32 ${sh%x*} ${sh#*x} bf16 NCHW > gpurun_out/p89e_$sh.log 2>&1; echo rc=$? >> gpurun_out/p89e_$sh.log
done
echo done
