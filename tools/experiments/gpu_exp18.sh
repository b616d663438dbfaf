timeout 600 python -m pytest tests -m "gpu and not slow" -q -x --timeout 300 -p no:cacheprovider > gpurun_out/gpu_tests.log 2>&1; echo rc=$? >> gpurun_out/gpu_tests.log
B="python bench.py --steps 40 --warmup 5 --e2e-steps 0 --no-cpu-baseline"
IABN_VERBOSE=1 timeout 300 $B > gpurun_out/e18_auto.log 2>&1
IABN_VERBOSE=1 IABN_FUSED_K=4 IABN_FUSED_NBUF=1 timeout 300 $B > gpurun_out/e18_k4nb1.log 2>&1
IABN_VERBOSE=1 IABN_FUSED_K=16 IABN_FUSED_NBUF=1 timeout 300 $B > gpurun_out/e18_k16nb1.log 2>&1
IABN_VERBOSE=1 timeout 300 $B --config r50s3 > gpurun_out/e18_r50.log 2>&1
IABN_FUSED_DEBUG=4 timeout 300 python tools/trace_fused.py > gpurun_out/t18.log 2>&1
echo done
