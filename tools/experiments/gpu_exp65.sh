timeout 900 python -m pytest tests -m "gpu and not slow" -q --timeout 600 -p no:cacheprovider > gpurun_out/gpu_tests.log 2>&1; echo rc=$? >> gpurun_out/gpu_tests.log
for cfg in "densenet264 bf16 NHWC" "rx101 f32 NHWC"; do
  set -- $cfg
  timeout 600 python tools/sweep.py --net $1 --dtype $2 --layout $3 > gpurun_out/sw65_$1_$2_$3.json 2> gpurun_out/sw65_$1_$2_$3.err
done
echo done
