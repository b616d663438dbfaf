timeout 600 python -m pytest -x -q tests/test_small_layers_gpu.py -p no:cacheprovider > gpurun_out/p_t.log 2>&1; echo rc=$? >> gpurun_out/p_t.log
timeout 1500 python -m pytest -q tests -m gpu -p no:cacheprovider > gpurun_out/p_all.log 2>&1; echo rc=$? >> gpurun_out/p_all.log
for cfg in "rx101 bf16 NCHW" "rx101 f32 NCHW" "densenet264 bf16 NCHW" "densenet264 f32 NCHW"; do
  set -- $cfg
  timeout 600 python tools/sweep.py --net $1 --dtype $2 --layout $3 > gpurun_out/p_sweep_$1_$2_$3.json 2>/dev/null
done
