timeout 600 python -m pytest -x -q tests/test_small_layers_gpu.py -p no:cacheprovider > gpurun_out/o_t.log 2>&1; echo rc=$? >> gpurun_out/o_t.log
timeout 600 python tools/small_tune.py --dtype bf16 > gpurun_out/o_tune_bf16.log 2>&1
timeout 600 python tools/small_tune.py --dtype f32 > gpurun_out/o_tune_f32.log 2>&1
