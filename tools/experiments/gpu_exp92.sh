# fused-collective sync: tests + emulated scaling; regression check of the plain schedules
timeout 300 python -m pytest tests/test_sync_fused_gpu.py -x -q 2>&1 | tail -3
for c in wrn38 r50s3 rx101_14; do timeout 300 python tools/sync_emulated.py --cfg $c > gpurun_out/sync_emu_$c.json 2>&1; grep variant gpurun_out/sync_emu_$c.json | grep -v rows; done
timeout 300 python bench.py --steps 20 --e2e-steps 0 --no-cpu-baseline 2>&1 | tail -1 | cut -c1-300
timeout 300 python bench.py --config r50s3 --e2e-steps 0 --no-cpu-baseline 2>&1 | tail -1 | cut -c1-300
timeout 600 python tools/sweep.py --net rx101 --dtype bf16 --layout NCHW 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print({k:v for k,v in d.items() if not isinstance(v,(list,dict))})"
