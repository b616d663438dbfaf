timeout 600 python -m pytest -x -q tests/test_small_layers_gpu.py -p no:cacheprovider > gpurun_out/s_t.log 2>&1; echo rc=$? >> gpurun_out/s_t.log
timeout 600 python tools/small_tune.py --dtype bf16 --shapes 512x196,1024x196,1024x49,2048x49,2688x49,128x196,128x49 > gpurun_out/s_tune_bf16.log 2>&1
timeout 600 python tools/small_tune.py --dtype f32 --shapes 1024x49,2048x49,128x49 > gpurun_out/s_tune_f32.log 2>&1
for cfg in "rx101 bf16 NCHW" "densenet264 bf16 NCHW" "densenet264 f32 NCHW"; do
  set -- $cfg
  timeout 600 python tools/sweep.py --net $1 --dtype $2 --layout $3 > gpurun_out/s_sweep_$1_$2_$3.json 2>/dev/null
done
