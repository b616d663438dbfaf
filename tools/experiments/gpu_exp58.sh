B="python bench.py --steps 60 --warmup 5 --e2e-steps 0 --no-cpu-baseline"
timeout 300 $B > gpurun_out/e58_base.log 2>&1
IABN_FUSED_CHUNK=784 timeout 300 $B > gpurun_out/e58_c784.log 2>&1
IABN_FUSED_CHUNK=1045 timeout 300 $B > gpurun_out/e58_c1045.log 2>&1
IABN_FUSED_CHUNK=3136 timeout 300 $B > gpurun_out/e58_c3136.log 2>&1
IABN_FUSED_CHUNK=784 IABN_FUSED_DEBUG=4 timeout 300 python tools/trace_fused.py > gpurun_out/t58.log 2>&1
echo done
