# fused-collective sync over virtual ranks (wrn38): L2 prefetch of double-buffered slices
S="python tools/sync_emulated.py --cfg wrn38 --iters 10"
run() { echo "== $1"; env $2 timeout 200 $S --G $3 2>&1 | grep '"fused-collective' | python -c '
import sys,json
for l in sys.stdin:
    d=json.loads(l)
    if "G" in d and "fwd_us" in d: print(d["G"], d["fwd_us"], d["bwd_us"], d["pct_of_peak"])'; }
run default "X=1" 2,8
run "pf on" "IABN_FUSED_PREFETCH=1" 2,4,8
run "pf bwd" "IABN_FUSED_PREFETCH=2" 2,8
run "pf on hint0" "IABN_FUSED_PREFETCH=1 IABN_FUSED_PF_HINT=0" 2,8
run "pf on hint1" "IABN_FUSED_PREFETCH=1 IABN_FUSED_PF_HINT=1" 2,8
run "K8 nb1" "IABN_FUSED_K=8 IABN_FUSED_NBUF=1" 2
run "K4 nb1" "IABN_FUSED_K=4 IABN_FUSED_NBUF=1" 2
S="python tools/sync_emulated.py --cfg r50s3 --iters 10"
run "r50s3 default" "X=1" 2,8
run "r50s3 pf on" "IABN_FUSED_PREFETCH=1" 2,8
S="python tools/sync_emulated.py --cfg rx101_14 --iters 10"
run "rx101_14 default" "X=1" 2,8
run "rx101_14 pf on" "IABN_FUSED_PREFETCH=1" 2,8
B="python bench.py --steps 50 --e2e-steps 0 --no-cpu-baseline --sync-emulated 0"
p() { python -c 'import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(d["fwd_ms"], d["bwd_ms"], d["pct_of_peak"])'; }
echo "plain wrn38 default $($B 2>/dev/null | p)"
echo "plain wrn38 pf on $(IABN_FUSED_PREFETCH=1 $B 2>/dev/null | p)"
B="python bench.py --config r50s3 --e2e-steps 0 --no-cpu-baseline --sync-emulated 0"
echo "plain r50s3 default $($B 2>/dev/null | p)"
echo "plain r50s3 pf on $(IABN_FUSED_PREFETCH=1 $B 2>/dev/null | p)"
