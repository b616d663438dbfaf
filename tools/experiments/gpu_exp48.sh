timeout 900 python -m pytest tests -m "gpu and not slow" -q -x --timeout 600 -p no:cacheprovider > gpurun_out/gpu_tests.log 2>&1; echo rc=$? >> gpurun_out/gpu_tests.log
echo done
