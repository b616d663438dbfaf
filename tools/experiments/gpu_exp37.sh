# 4 CTAs/SM (256 threads: 2 reduce + 4 apply warps, <= 64 regs) with clusters of 16 (50 KB slices)
B="python bench.py --steps 60 --warmup 5 --e2e-steps 0 --no-cpu-baseline"
L=paper_1712_02616_b200/libiabn.so
cp $L /tmp/main.so
IABN_VERBOSE=1 IABN_FUSED_K=16 IABN_FUSED_NBUF=1 IABN_FUSED_SMEM_KB=50 timeout 300 $B > gpurun_out/e37_main_k16.log 2>&1
cp tools/libiabn_variant.so $L
IABN_VERBOSE=1 IABN_FUSED_K=16 IABN_FUSED_NBUF=1 IABN_FUSED_SMEM_KB=50 timeout 300 $B > gpurun_out/e37_var_k16.log 2>&1
IABN_VERBOSE=1 timeout 300 $B > gpurun_out/e37_var_default.log 2>&1
IABN_VERBOSE=1 IABN_FUSED_K=16 IABN_FUSED_NBUF=2 IABN_FUSED_SMEM_KB=50 timeout 300 $B > gpurun_out/e37_var_k16nb2.log 2>&1
IABN_VERBOSE=1 IABN_FUSED_K=8 IABN_FUSED_NBUF=1 IABN_FUSED_SMEM_KB=50 IABN_FUSED_CHUNK=784 timeout 300 $B > gpurun_out/e37_var_k8half.log 2>&1
IABN_FUSED_DEBUG=4 IABN_FUSED_K=16 IABN_FUSED_NBUF=1 IABN_FUSED_SMEM_KB=50 timeout 300 python tools/trace_fused.py > gpurun_out/t37.log 2>&1
cp /tmp/main.so $L
echo done
