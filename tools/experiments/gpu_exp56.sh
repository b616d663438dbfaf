timeout 900 python -m pytest tests -m "gpu and not slow" -q --timeout 600 -p no:cacheprovider > gpurun_out/gpu_tests.log 2>&1; echo rc=$? >> gpurun_out/gpu_tests.log
for cfg in "rx101 bf16 NCHW" "densenet264 bf16 NCHW" "densenet264 f32 NCHW"; do
  set -- $cfg
  timeout 600 python tools/sweep.py --net $1 --dtype $2 --layout $3 > gpurun_out/sw56_$1_$2_$3.json 2> gpurun_out/sw56_$1_$2_$3.err
done
B="python bench.py --steps 60 --warmup 5 --e2e-steps 0 --no-cpu-baseline"
timeout 300 $B > gpurun_out/e56.log 2>&1
timeout 300 $B --schedule streaming > gpurun_out/e56_stream.log 2>&1
echo done
