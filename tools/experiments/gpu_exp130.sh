# warp-wide producer (chunks of >= 4 planes), serial loop kept for narrow chunks: parity, A/B vs _prev
timeout 900 python -m pytest tests/test_parity_gpu.py tests/test_sync_fused_gpu.py tests/test_parity_full_gpu.py -x -q 2>&1 | tail -2
R="python bench.py --config r50s3 --e2e-steps 0 --no-cpu-baseline --sync-emulated 0"
W="python bench.py --steps 100 --e2e-steps 0 --no-cpu-baseline --sync-emulated 0"
p() { python -c 'import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(d["fwd_ms"], d["bwd_ms"])'; }
for i in 1 2 3; do for d in _prev .; do
  echo "wrn38 $d $(cd $d && $W 2>/dev/null | p)"
  echo "r50s3 $d $(cd $d && $R 2>/dev/null | p)"
done; done
