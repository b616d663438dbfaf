timeout 600 python -m pytest -x -q tests/test_nhwc_reg_gpu.py -p no:cacheprovider > gpurun_out/x_t.log 2>&1; echo rc=$? >> gpurun_out/x_t.log
timeout 900 python tools/nhwc_tune.py --dtype bf16 --shapes 128x49,128x196,512x196,1024x49,2688x49,1024x196,256x196 --gs 16,32 --ks 2,4,8 > gpurun_out/x_tune_bf16.log 2>&1
timeout 600 python tools/nhwc_tune.py --dtype f32 --shapes 128x49,128x196,512x196,1024x49 --gs 8,16 --ks 2,4,8 > gpurun_out/x_tune_f32.log 2>&1
