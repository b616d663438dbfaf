IABN_FUSED_MIS=1 IABN_VERBOSE=1 timeout 60 python tools/layer_probe.py 32 512 196 bf16 NCHW > gpurun_out/p86a.log 2>&1; echo rc=$? >> gpurun_out/p86a.log
IABN_FUSED_MIS=1 IABN_VERBOSE=1 timeout 60 python tools/layer_probe.py 8 40 196 bf16 NCHW > gpurun_out/p86b.log 2>&1; echo rc=$? >> gpurun_out/p86b.log
IABN_FUSED_MIS=1 IABN_VERBOSE=1 timeout 60 python tools/layer_probe.py 32 128 196 bf16 NCHW > gpurun_out/p86c.log 2>&1; echo rc=$? >> gpurun_out/p86c.log
IABN_FUSED_MIS=1 IABN_VERBOSE=1 timeout 60 python tools/layer_probe.py 32 128 49 f32 NCHW > gpurun_out/p86d.log 2>&1; echo rc=$? >> gpurun_out/p86d.log
nvidia-smi --query-gpu=index,utilization.gpu --format=csv > gpurun_out/p86_smi.txt 2>&1
echo done
