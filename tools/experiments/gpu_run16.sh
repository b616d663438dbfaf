timeout 600 python -m pytest tests -m "gpu and not slow" -q -x --timeout 300 -p no:cacheprovider > gpurun_out/gpu_tests.log 2>&1; echo rc=$? >> gpurun_out/gpu_tests.log
IABN_VERBOSE=1 timeout 600 python bench.py > gpurun_out/bench16.log 2>&1
IABN_FUSED_DEBUG=4 timeout 300 python tools/trace_fused.py > gpurun_out/t16.log 2>&1
B="python bench.py --steps 40 --warmup 5 --e2e-steps 0 --no-cpu-baseline"
IABN_VERBOSE=1 timeout 300 $B --config r50s3 > gpurun_out/b16_r50.log 2>&1
echo done
