# r50s3: ec9efaf (_old) vs HEAD on the same box
R="python bench.py --config r50s3 --e2e-steps 0 --no-cpu-baseline --sync-emulated 0"
for i in 1 2 3; do for d in _old .; do
  echo "$d $(cd $d && timeout 120 $R 2>&1 | tail -1 | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["fwd_ms"], d["bwd_ms"], d["pct_of_peak"])')"
done; done
