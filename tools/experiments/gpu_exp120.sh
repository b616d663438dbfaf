# L2 hints compiled out of the 4-CTA/SM variant: r50s3 / wrn38 vs ec9efaf (_old); GPU tests
R="python bench.py --config r50s3 --e2e-steps 0 --no-cpu-baseline --sync-emulated 0"
W="python bench.py --steps 100 --e2e-steps 0 --no-cpu-baseline --sync-emulated 0"
p() { python -c 'import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(d["fwd_ms"], d["bwd_ms"], d["pct_of_peak"])'; }
for i in 1 2; do for d in _old .; do
  echo "r50s3 $d $(cd $d && timeout 120 $R 2>/dev/null | p)"
  echo "wrn38 $d $(cd $d && timeout 120 $W 2>/dev/null | p)"
done; done
timeout 600 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
