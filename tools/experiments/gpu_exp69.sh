# programmatic dependent launch (PDL) on every kernel launch vs plain launches
timeout 1200 python -m pytest tests -m gpu -q --timeout 600 -p no:cacheprovider > gpurun_out/gpu_tests.log 2>&1; echo rc=$? >> gpurun_out/gpu_tests.log
B="python bench.py --steps 60 --warmup 5 --e2e-steps 0 --no-cpu-baseline"
for p in 1 0; do
IABN_PDL=$p timeout 300 $B > gpurun_out/e69_$p.log 2>&1
IABN_PDL=$p timeout 300 $B --config r50s3 > gpurun_out/e69_r50_$p.log 2>&1
for cfg in "rx101 f32 NCHW" "rx101 bf16 NCHW" "densenet264 bf16 NHWC"; do
  set -- $cfg
  IABN_PDL=$p timeout 600 python tools/sweep.py --net $1 --dtype $2 --layout $3 > gpurun_out/sw69_${p}_$1_$2_$3.json 2> gpurun_out/sw69_${p}_$1_$2_$3.err
done; done
echo done
