timeout 600 python -m pytest -x -q tests/test_nhwc_fused_gpu.py tests/test_parity_gpu.py -p no:cacheprovider > gpurun_out/f_t.log 2>&1; echo rc=$? >> gpurun_out/f_t.log
timeout 600 python -m pytest -x -q tests/test_parity_networks_gpu.py -k NHWC -p no:cacheprovider > gpurun_out/f_net.log 2>&1; echo rc=$? >> gpurun_out/f_net.log
IABN_VERBOSE=1 timeout 600 python tools/sweep.py --net densenet264 --dtype bf16 --layout NHWC > gpurun_out/f_sweep_dn_bf16_nhwc.json 2> gpurun_out/f_sweep_dn.err
timeout 600 python tools/sweep.py --net densenet264 --dtype f32 --layout NHWC > gpurun_out/f_sweep_dn_f32_nhwc.json 2> /dev/null
timeout 600 python tools/sweep.py --net rx101 --dtype bf16 --layout NHWC > gpurun_out/f_sweep_rx_bf16_nhwc.json 2> /dev/null
for s in "128 196 bf16 0" "128 196 bf16 1"; do
  set -- $s
  IABN_NHWC_TRACE=1 timeout 120 python tools/nhwc_trace.py $1 $2 $3 $4 > gpurun_out/f_trace_$1_$2_$3_$4.log 2>&1
done
