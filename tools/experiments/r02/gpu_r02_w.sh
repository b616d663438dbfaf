timeout 1200 python -m pytest -x -q tests/test_sync_fused_gpu.py tests/test_dynamic_sched_gpu.py -p no:cacheprovider > gpurun_out/w_t.log 2>&1; echo rc=$? >> gpurun_out/w_t.log
for c in wrn38 r50s3 rx101_14; do
  timeout 300 python tools/sync_emulated.py --cfg $c > gpurun_out/w_sync_emu_$c.json 2>&1
done
timeout 600 python bench.py --e2e-steps 0 --no-cpu-baseline > gpurun_out/w_bench.log 2>&1
