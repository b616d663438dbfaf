# r50s3: cluster size vs channel balance (1024 channels over the co-resident clusters)
R="python bench.py --config r50s3 --e2e-steps 0 --no-cpu-baseline --sync-emulated 0"
run() { echo "$1 :: $(env $2 timeout 120 $R 2>&1 | tail -1 | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["fwd_ms"], d["bwd_ms"], d["pct_of_peak"], d["config"]["schedule"])')"; }
run default "X=1"
run "K4 minb4" "IABN_FUSED_K=4 IABN_FUSED_MINB=4 IABN_FUSED_NBUF=2"
run "K8 minb4" "IABN_FUSED_K=8 IABN_FUSED_MINB=4 IABN_FUSED_NBUF=2"
run "K4 minb4 nb3" "IABN_FUSED_K=4 IABN_FUSED_MINB=4 IABN_FUSED_NBUF=3"
run "K2 minb2 nb2" "IABN_FUSED_K=2 IABN_FUSED_MINB=2 IABN_FUSED_NBUF=2"
run "K4 minb2 nb2" "IABN_FUSED_K=4 IABN_FUSED_MINB=2 IABN_FUSED_NBUF=2"
IABN_VERBOSE=1 timeout 120 $R 2>&1 | grep "\[iabn\]" | sort | uniq
