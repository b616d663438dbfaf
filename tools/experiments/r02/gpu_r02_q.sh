timeout 1500 python -m pytest -q tests -m gpu -p no:cacheprovider > gpurun_out/q_all.log 2>&1; echo rc=$? >> gpurun_out/q_all.log
timeout 600 python bench.py --e2e-steps 0 --no-cpu-baseline --sync-emulated 0 > gpurun_out/q_bench.log 2>&1
for cfg in "densenet264 bf16 NHWC" "rx101 bf16 NHWC"; do
  set -- $cfg
  timeout 600 python tools/sweep.py --net $1 --dtype $2 --layout $3 > gpurun_out/q_sweep_$1_$2_$3.json 2>/dev/null
done
