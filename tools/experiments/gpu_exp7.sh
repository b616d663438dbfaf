timeout 600 python -m pytest tests -m "gpu and not slow" -q -x --timeout 300 -p no:cacheprovider > gpurun_out/gpu_tests.log 2>&1; echo rc=$? >> gpurun_out/gpu_tests.log
B="python bench.py --steps 60 --warmup 5 --e2e-steps 0 --no-cpu-baseline"
for nb in 3 4; do for kb in 100 200; do IABN_FUSED_NBUF=$nb IABN_FUSED_SMEM_KB=$kb timeout 300 $B > gpurun_out/e7_nb${nb}_kb$kb.log 2>&1; done; done
IABN_FUSED_DEBUG=1 IABN_FUSED_NBUF=4 IABN_FUSED_SMEM_KB=100 timeout 300 $B > gpurun_out/e7_d1_nb4_kb100.log 2>&1
IABN_FUSED_DEBUG=3 IABN_FUSED_NBUF=4 IABN_FUSED_SMEM_KB=100 timeout 300 $B > gpurun_out/e7_d3_nb4_kb100.log 2>&1
echo done
