timeout 600 python -m pytest tests -m "gpu and not slow" -q -x --timeout 300 -p no:cacheprovider > gpurun_out/gpu_tests.log 2>&1; echo rc=$? >> gpurun_out/gpu_tests.log
B="python bench.py --steps 60 --warmup 5 --e2e-steps 0 --no-cpu-baseline"
for dbg in 0 1 3; do for kb in 100 200; do IABN_FUSED_DEBUG=$dbg IABN_FUSED_SMEM_KB=$kb timeout 300 $B > gpurun_out/e6_d${dbg}_kb$kb.log 2>&1; done; done
IABN_FUSED_SMEM_KB=72 timeout 300 $B > gpurun_out/e6_d0_kb72.log 2>&1
echo done
