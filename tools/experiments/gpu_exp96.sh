# cluster shape experiments for cfg4 (fwd/bwd split)
B="python bench.py --steps 30 --e2e-steps 0 --no-cpu-baseline --sync-emulated 0"
run() { echo "$1 :: $(env $2 timeout 300 $B 2>&1 | tail -1 | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["fwd_ms"], d["bwd_ms"], d["pct_of_peak"], d["config"]["schedule"])')"; }
run default "X=1"
run "K16 nb1 minb4" "IABN_FUSED_K=16 IABN_FUSED_NBUF=1 IABN_FUSED_MINB=4"
run "K16 nb2 minb4" "IABN_FUSED_K=16 IABN_FUSED_NBUF=2 IABN_FUSED_MINB=4"
run "K16 nb2 minb2" "IABN_FUSED_K=16 IABN_FUSED_NBUF=2 IABN_FUSED_MINB=2"
run "K8 nb1 minb2" "IABN_FUSED_K=8 IABN_FUSED_NBUF=1 IABN_FUSED_MINB=2"
IABN_VERBOSE=1 IABN_FUSED_K=16 IABN_FUSED_NBUF=1 IABN_FUSED_MINB=4 timeout 300 $B 2>&1 | grep "\[iabn\]" | head -4
