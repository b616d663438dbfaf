# with L2 prefetch: cluster shapes for cfg4 backward; prefetch policy for r50s3 / sweeps
B="python bench.py --steps 30 --e2e-steps 0 --no-cpu-baseline --sync-emulated 0"
R="python bench.py --config r50s3 --e2e-steps 0 --no-cpu-baseline --sync-emulated 0"
run() { echo "$1 :: $(env $2 timeout 120 $3 2>&1 | tail -1 | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["fwd_ms"], d["bwd_ms"], d["pct_of_peak"])')"; }
run "wrn38 default" "X=1" "$B"
run "wrn38 K16 nb2 minb2" "IABN_FUSED_K=16 IABN_FUSED_NBUF=2 IABN_FUSED_MINB=2 IABN_FUSED_PREFETCH=1" "$B"
run "wrn38 K16 nb1 minb4" "IABN_FUSED_K=16 IABN_FUSED_NBUF=1 IABN_FUSED_MINB=4 IABN_FUSED_PREFETCH=1" "$B"
run "wrn38 K8 nb1 minb2 pf2" "IABN_FUSED_PREFETCH=2" "$B"
run "r50s3 default" "X=1" "$R"
run "r50s3 pf2" "IABN_FUSED_PREFETCH=2" "$R"
run "r50s3 K8 nb1 pf" "IABN_FUSED_K=8 IABN_FUSED_NBUF=1 IABN_FUSED_MINB=4 IABN_FUSED_PREFETCH=1" "$R"
run "r50s3 K4 nb1 pf" "IABN_FUSED_K=4 IABN_FUSED_NBUF=1 IABN_FUSED_MINB=4 IABN_FUSED_PREFETCH=1" "$R"
for pf in -1 2; do
  echo "PF=$pf rx101 f32 $(IABN_FUSED_PREFETCH=$pf timeout 600 python tools/sweep.py --net rx101 --dtype f32 2>/dev/null | tail -1 | grep -o '"graph_pct_of_peak": [0-9.]*')"
done
