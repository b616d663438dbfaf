# small-slab variant only with whole planes per CTA
timeout 600 python -m pytest tests -m gpu -x -q -p no:cacheprovider 2>&1 | tail -1
for c in wrn38 r50s3; do timeout 300 python tools/sync_emulated.py --cfg $c 2>&1 | grep '^{"variant"' | python -c "
import sys, json
for l in sys.stdin:
    d = json.loads(l); print('  $c', d['variant'][:32], d.get('fwd_us'), d.get('bwd_us'), d.get('pct_of_peak'))"; done
timeout 200 python bench.py --steps 50 --e2e-steps 0 --no-cpu-baseline 2>&1 | tail -1 | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["fwd_ms"], d["bwd_ms"], d["pct_of_peak"], d["sync_emulated"]["pct_of_peak"])'
for cfg in "rx101 bf16" "densenet264 bf16"; do set -- $cfg; echo "$cfg $(timeout 600 python tools/sweep.py --net $1 --dtype $2 2>/dev/null | tail -1 | grep -o '"graph_pct_of_peak": [0-9.]*')"; done
