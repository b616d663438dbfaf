timeout 600 python -m pytest -x -q tests/test_nhwc_fused_gpu.py -p no:cacheprovider > gpurun_out/e_nhwc.log 2>&1; echo rc=$? >> gpurun_out/e_nhwc.log
timeout 600 python tools/nhwc_tune.py --dtype bf16 --shapes 128x49,128x196,512x196,1024x49 --ks 1,2,4,6,8 --gs 8,16,32 > gpurun_out/e_tune.log 2>&1
for s in "128 196 bf16 0" "128 196 bf16 1" "128 49 bf16 0" "512 196 bf16 0"; do
  set -- $s
  IABN_NHWC_TRACE=1 timeout 120 python tools/nhwc_trace.py $1 $2 $3 $4 > gpurun_out/e_trace_$1_$2_$3_$4.log 2>&1
done
