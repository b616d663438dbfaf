timeout 900 python -m pytest tests -m "gpu and not slow" -q --timeout 600 -p no:cacheprovider > gpurun_out/gpu_tests.log 2>&1; echo rc=$? >> gpurun_out/gpu_tests.log
B="python bench.py --steps 60 --warmup 5 --e2e-steps 0 --no-cpu-baseline"
IABN_VERBOSE=1 IABN_FUSED_MINB=4 IABN_FUSED_K=16 IABN_FUSED_NBUF=1 timeout 300 $B > gpurun_out/e68_m4k16.log 2>&1
IABN_VERBOSE=1 IABN_FUSED_MINB=4 IABN_FUSED_K=16 IABN_FUSED_NBUF=1 IABN_FUSED_SMALL_KB=60 timeout 300 $B > gpurun_out/e68_m4k16b.log 2>&1
echo done
