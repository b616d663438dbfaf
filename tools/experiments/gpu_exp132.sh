# default bench (12 e2e steps) + smoke
s=$(date +%s); timeout 600 python bench.py > gpurun_out/e132_bench.log 2>&1; echo "bench wall $(( $(date +%s) - s )) s"
grep '^{' gpurun_out/e132_bench.log | tail -1 | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["pct_of_peak"], d["fwd_ms"], d["bwd_ms"], d["e2e"])'
