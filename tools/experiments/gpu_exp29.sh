# finer phase trace; one 200 KB double-buffered CTA per SM vs two 100 KB single-buffered
B="python bench.py --steps 60 --warmup 5 --e2e-steps 0 --no-cpu-baseline"
IABN_FUSED_DEBUG=4 timeout 300 python tools/trace_fused.py > gpurun_out/t29.log 2>&1
IABN_FUSED_SMEM_KB=210 IABN_FUSED_K=8 IABN_FUSED_NBUF=2 timeout 300 $B > gpurun_out/e29_k8nb2big.log 2>&1
IABN_FUSED_SMEM_KB=210 IABN_FUSED_K=8 IABN_FUSED_NBUF=2 IABN_FUSED_UNIFIED=0 IABN_FUSED_DEBUG=4 timeout 300 python tools/trace_fused.py > gpurun_out/t29big.log 2>&1
IABN_FUSED_K=16 IABN_FUSED_NBUF=2 timeout 300 $B > gpurun_out/e29_k16nb2.log 2>&1
echo done
