B="python bench.py --steps 60 --warmup 5 --e2e-steps 0 --no-cpu-baseline"
timeout 300 $B > gpurun_out/e83_base.log 2>&1
IABN_VERBOSE=1 IABN_FUSED_MINB=4 IABN_FUSED_K=8 IABN_FUSED_NBUF=1 IABN_FUSED_SMALL_KB=50 timeout 300 $B > gpurun_out/e83_m4k8n1.log 2>&1
IABN_VERBOSE=1 IABN_FUSED_MINB=4 IABN_FUSED_K=16 IABN_FUSED_NBUF=2 IABN_FUSED_SMALL_KB=50 timeout 300 $B > gpurun_out/e83_m4k16n2.log 2>&1
IABN_VERBOSE=1 IABN_FUSED_MINB=2 IABN_FUSED_K=8 IABN_FUSED_NBUF=3 IABN_FUSED_SMEM_KB=110 timeout 300 $B > gpurun_out/e83_m2k8n3.log 2>&1
echo done
