# r50s3 regression bisect: _old (ec9efaf), _ka (old kernels_fused.cuh), _kb (old iabn.cu), HEAD
R="python bench.py --config r50s3 --e2e-steps 0 --no-cpu-baseline --sync-emulated 0"
p() { python -c 'import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(d["fwd_ms"], d["bwd_ms"], d["pct_of_peak"])'; }
for i in 1 2; do for d in _old _ka _kb .; do
  echo "r50s3 $d $(cd $d && timeout 120 $R 2>/dev/null | p)"
done; done
(cd _old && IABN_VERBOSE=1 timeout 120 $R 2>&1 | grep iabn | sort -u | head -4)
IABN_VERBOSE=1 timeout 120 $R 2>&1 | grep iabn | sort -u | head -4
