# NHWC channel-group schedule: parity first, then sweeps
timeout 600 python -m pytest -x -q tests/test_nhwc_fused_gpu.py -p no:cacheprovider > gpurun_out/c_nhwc.log 2>&1; echo rc=$? >> gpurun_out/c_nhwc.log
timeout 900 python -m pytest -x -q tests/test_parity_gpu.py tests/test_parity_networks_gpu.py tests/test_guard_gpu.py -p no:cacheprovider > gpurun_out/c_par.log 2>&1; echo rc=$? >> gpurun_out/c_par.log
IABN_VERBOSE=1 timeout 600 python tools/sweep.py --net densenet264 --dtype bf16 --layout NHWC > gpurun_out/c_sweep_dn_bf16_nhwc.json 2> gpurun_out/c_sweep_dn.err
timeout 600 python tools/sweep.py --net densenet264 --dtype f32 --layout NHWC > gpurun_out/c_sweep_dn_f32_nhwc.json 2> gpurun_out/c_sweep_dn32.err
timeout 600 python tools/sweep.py --net rx101 --dtype bf16 --layout NHWC > gpurun_out/c_sweep_rx_bf16_nhwc.json 2> gpurun_out/c_sweep_rx.err
