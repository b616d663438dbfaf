timeout 900 python -m pytest -x -q tests/test_dynamic_sched_gpu.py tests/test_parity_gpu.py tests/test_parity_full_gpu.py tests/test_sync_fused_gpu.py -p no:cacheprovider > gpurun_out/k_t.log 2>&1; echo rc=$? >> gpurun_out/k_t.log
timeout 600 python bench.py > gpurun_out/k_bench.log 2>&1
timeout 600 python bench.py --config r50s3 --e2e-steps 0 --no-cpu-baseline --sync-emulated 0 > gpurun_out/k_bench_r50.log 2>&1
