timeout 600 python -m pytest -x -q tests/test_small_layers_gpu.py tests/test_parity_networks_gpu.py tests/test_guard_gpu.py tests/test_fault_injection_gpu.py -p no:cacheprovider > gpurun_out/t_t.log 2>&1; echo rc=$? >> gpurun_out/t_t.log
timeout 600 python tools/small_tune.py --dtype bf16 > gpurun_out/t_tune_bf16.log 2>&1
timeout 600 python tools/small_tune.py --dtype f32 > gpurun_out/t_tune_f32.log 2>&1
for cfg in "rx101 bf16 NCHW" "rx101 f32 NCHW" "densenet264 bf16 NCHW" "densenet264 f32 NCHW"; do
  set -- $cfg
  timeout 600 python tools/sweep.py --net $1 --dtype $2 --layout $3 > gpurun_out/t_sweep_$1_$2_$3.json 2>/dev/null
done
