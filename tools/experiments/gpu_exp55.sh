timeout 900 python -m pytest tests -m "gpu and not slow" -q --timeout 600 -p no:cacheprovider > gpurun_out/gpu_tests.log 2>&1; echo rc=$? >> gpurun_out/gpu_tests.log
for m in 0 1; do
for cfg in "rx101 bf16 NCHW" "densenet264 bf16 NHWC" "rx101 f32 NCHW"; do
  set -- $cfg
  IABN_COOP=$m timeout 600 python tools/sweep.py --net $1 --dtype $2 --layout $3 > gpurun_out/sw55_${m}_$1_$2_$3.json 2> gpurun_out/sw55_${m}_$1_$2_$3.err
done; done
echo done
