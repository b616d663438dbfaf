timeout 900 python -m pytest tests -m gpu -q --timeout 600 -p no:cacheprovider > gpurun_out/gpu_tests.log 2>&1; echo rc=$? >> gpurun_out/gpu_tests.log
B="python bench.py --steps 60 --warmup 5 --e2e-steps 0 --no-cpu-baseline"
IABN_VERBOSE=1 timeout 300 $B > gpurun_out/e61.log 2>&1
IABN_VERBOSE=1 timeout 300 $B --config r50s3 > gpurun_out/e61_r50.log 2>&1
for cfg in "rx101 f32 NCHW" "densenet264 f32 NCHW" "rx101 bf16 NCHW"; do
  set -- $cfg
  timeout 600 python tools/sweep.py --net $1 --dtype $2 --layout $3 > gpurun_out/sw61_$1_$2_$3.json 2> gpurun_out/sw61_$1_$2_$3.err
done
echo done
