# cfg4 backward plans with the L2 prefetch + cache hints
B="python bench.py --steps 50 --e2e-steps 0 --no-cpu-baseline --sync-emulated 0"
run() { echo "$1 :: $(env $2 timeout 120 $B 2>&1 | tail -1 | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["fwd_ms"], d["bwd_ms"], d["pct_of_peak"])')"; }
run default "X=1"
run "K16 nb2 pf" "IABN_FUSED_K=16 IABN_FUSED_NBUF=2 IABN_FUSED_MINB=2 IABN_FUSED_PREFETCH=1"
run "K16 nb2" "IABN_FUSED_K=16 IABN_FUSED_NBUF=2 IABN_FUSED_MINB=2"
run "K8 nb1 pf hint1" "IABN_FUSED_PF_HINT=1"
run "K8 nb1 pf hint2" "IABN_FUSED_PF_HINT=2"
run default "X=1"
