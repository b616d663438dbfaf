# every slice bulk copy with L2 evict_first (IABN_FUSED_LOAD_EVICT_FIRST)
B="python bench.py --steps 50 --e2e-steps 0 --no-cpu-baseline --sync-emulated 0"
R="python bench.py --config r50s3 --e2e-steps 0 --no-cpu-baseline --sync-emulated 0"
for e in 0 1 0 1; do
  echo "EF=$e wrn38 $(IABN_FUSED_LOAD_EVICT_FIRST=$e timeout 120 $B 2>&1 | tail -1 | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["fwd_ms"], d["bwd_ms"], d["pct_of_peak"])') r50s3 $(IABN_FUSED_LOAD_EVICT_FIRST=$e timeout 120 $R 2>&1 | tail -1 | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["fwd_ms"], d["bwd_ms"], d["pct_of_peak"])')"
done
for e in 0 1; do
  echo "EF=$e rx101 bf16 $(IABN_FUSED_LOAD_EVICT_FIRST=$e timeout 600 python tools/sweep.py --net rx101 --dtype bf16 2>/dev/null | tail -1 | grep -o '"graph_pct_of_peak": [0-9.]*')"
done
