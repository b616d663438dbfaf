timeout 900 python -m pytest tests -m "gpu and not slow" -q --timeout 600 -p no:cacheprovider > gpurun_out/gpu_tests.log 2>&1; echo rc=$? >> gpurun_out/gpu_tests.log
for lb in 1 0; do
for cfg in "rx101 bf16 NCHW" "densenet264 bf16 NHWC"; do
  set -- $cfg
  IABN_LB=$lb timeout 600 python tools/sweep.py --net $1 --dtype $2 --layout $3 > gpurun_out/sw62_${lb}_$1_$2_$3.json 2> gpurun_out/sw62_${lb}_$1_$2_$3.err
done; done
B="python bench.py --steps 60 --warmup 5 --e2e-steps 0 --no-cpu-baseline --schedule streaming"
for lb in 1 0; do IABN_LB=$lb timeout 300 $B > gpurun_out/e62_$lb.log 2>&1; done
echo done
