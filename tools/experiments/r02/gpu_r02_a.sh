# round 2: new sync/guard/fault tests, whole GPU suite, bench (1 GPU) and the N=2 dry run
timeout 900 python -m pytest -x -q tests/test_sync_shim_gpu.py tests/test_guard_gpu.py tests/test_fault_injection_gpu.py > gpurun_out/a_new.log 2>&1; echo rc=$? >> gpurun_out/a_new.log
timeout 1500 python -m pytest -q tests -m gpu -p no:cacheprovider > gpurun_out/a_all.log 2>&1; echo rc=$? >> gpurun_out/a_all.log
timeout 600 python bench.py > gpurun_out/a_bench.log 2>&1; echo rc=$? >> gpurun_out/a_bench.log
timeout 600 python bench.py --emulate-ranks 2 --steps 20 --e2e-steps 2 > gpurun_out/a_dry2.log 2>&1; echo rc=$? >> gpurun_out/a_dry2.log
timeout 600 python bench.py --emulate-ranks 4 --config r50s3 --steps 20 --e2e-steps 2 > gpurun_out/a_dry4.log 2>&1; echo rc=$? >> gpurun_out/a_dry4.log
