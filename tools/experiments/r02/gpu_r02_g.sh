timeout 600 python -m pytest -x -q tests/test_nhwc_fused_gpu.py tests/test_parity_networks_gpu.py -p no:cacheprovider > gpurun_out/g_t.log 2>&1; echo rc=$? >> gpurun_out/g_t.log
timeout 600 python tools/sweep.py --net densenet264 --dtype bf16 --layout NHWC > gpurun_out/g_sweep_dn_bf16_nhwc.json 2> /dev/null
for s in "128 196 bf16 0" "128 196 bf16 1"; do
  set -- $s
  IABN_NHWC_TRACE=1 timeout 120 python tools/nhwc_trace.py $1 $2 $3 $4 > gpurun_out/g_trace_$1_$2_$3_$4.log 2>&1
done
