# wrn38 / r50s3: HEAD (lane-0 producer, _prev) vs warp-wide producer, alternating on one box
R="python bench.py --config r50s3 --e2e-steps 0 --no-cpu-baseline --sync-emulated 0"
W="python bench.py --steps 100 --e2e-steps 0 --no-cpu-baseline --sync-emulated 0"
p() { python -c 'import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(d["fwd_ms"], d["bwd_ms"], d["pct_of_peak"])'; }
for i in 1 2 3; do for d in _prev .; do
  echo "wrn38 $d $(cd $d && $W 2>/dev/null | p)"
  echo "r50s3 $d $(cd $d && $R 2>/dev/null | p)"
done; done
