# fused-collective sync over virtual ranks (wrn38): slab plans per G
S="python tools/sync_emulated.py --cfg wrn38 --iters 10"
run() { echo "== $1"; env $2 timeout 200 $S --G $3 2>&1 | grep '"fused-collective' | python -c '
import sys,json
for l in sys.stdin:
    d=json.loads(l); print(d["G"], d["fwd_us"], d["bwd_us"], d["pct_of_peak"])'; }
run default "X=1" 2,4,8
run "K4 nb1" "IABN_FUSED_K=4 IABN_FUSED_NBUF=1" 2
run "K8 nb1" "IABN_FUSED_K=8 IABN_FUSED_NBUF=1" 2,4
run "K2 nb1" "IABN_FUSED_K=2 IABN_FUSED_NBUF=1" 4,8
run "K1 nb1" "IABN_FUSED_K=1 IABN_FUSED_NBUF=1" 8
run "pf on" "IABN_FUSED_PREFETCH=1" 2,4,8
run "K4 nb2 minb4?" "IABN_FUSED_K=4 IABN_FUSED_NBUF=2 IABN_FUSED_MINB=4" 4
