# round 2: changed tests + full suite after the one-launch removal / coherent loads; streaming bench
timeout 900 python -m pytest -x -q tests/test_parity_gpu.py tests/test_sync_fused_gpu.py tests/test_fault_injection_gpu.py -p no:cacheprovider > gpurun_out/b_t.log 2>&1; echo rc=$? >> gpurun_out/b_t.log
timeout 300 python bench.py --schedule streaming --steps 100 --e2e-steps 0 --no-cpu-baseline --sync-emulated 0 > gpurun_out/b_stream.log 2>&1; echo rc=$? >> gpurun_out/b_stream.log
timeout 600 python tools/sweep.py --net densenet264 --dtype bf16 --layout NHWC > gpurun_out/b_sweep_dn_bf16_nhwc.json 2> gpurun_out/b_sweep_dn.err
timeout 600 python tools/sweep.py --net rx101 --dtype bf16 --layout NCHW > gpurun_out/b_sweep_rx_bf16_nchw.json 2> gpurun_out/b_sweep_rx.err
