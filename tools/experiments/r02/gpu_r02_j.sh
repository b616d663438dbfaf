timeout 900 python -m pytest -x -q tests/test_parity_gpu.py tests/test_parity_full_gpu.py tests/test_sync_fused_gpu.py tests/test_guard_gpu.py tests/test_parity_networks_gpu.py -p no:cacheprovider > gpurun_out/j_t.log 2>&1; echo rc=$? >> gpurun_out/j_t.log
timeout 600 python bench.py --e2e-steps 0 --no-cpu-baseline --sync-emulated 0 > gpurun_out/j_bench_dyn.log 2>&1
IABN_FUSED_DYN=0 timeout 600 python bench.py --e2e-steps 0 --no-cpu-baseline --sync-emulated 0 > gpurun_out/j_bench_static.log 2>&1
timeout 600 python bench.py --config r50s3 --e2e-steps 0 --no-cpu-baseline --sync-emulated 0 > gpurun_out/j_bench_r50_dyn.log 2>&1
IABN_FUSED_DYN=0 timeout 600 python bench.py --config r50s3 --e2e-steps 0 --no-cpu-baseline --sync-emulated 0 > gpurun_out/j_bench_r50_static.log 2>&1
timeout 600 python tools/sweep.py --net rx101 --dtype bf16 --layout NCHW > gpurun_out/j_sweep_rx_bf16.json 2>/dev/null
IABN_FUSED_DYN=0 timeout 600 python tools/sweep.py --net rx101 --dtype bf16 --layout NCHW > gpurun_out/j_sweep_rx_bf16_static.json 2>/dev/null
