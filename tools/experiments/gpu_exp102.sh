# TMEM kernels: does the hardware co-schedule 2 CTAs per SM (occupancy API says 1)?
B="python bench.py --steps 30 --e2e-steps 0 --no-cpu-baseline --sync-emulated 0"
run() { echo "$1 :: $(env $2 timeout 120 $B 2>&1 | tail -1 | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["fwd_ms"], d["bwd_ms"], d["pct_of_peak"])')"; }
run default "X=1"
run "tmem occ2" "IABN_FUSED_TMEM=1 IABN_FUSED_TM_OCC=2"
run "tmem occ2 kb100" "IABN_FUSED_TMEM=1 IABN_FUSED_TM_OCC=2 IABN_FUSED_TMEM_KB=100"
IABN_FUSED_TMEM=1 IABN_FUSED_TM_OCC=2 IABN_VERBOSE=1 timeout 120 $B 2>&1 | grep "\[iabn\]" | sort | uniq | head
IABN_FUSED_TMEM=1 IABN_FUSED_TM_OCC=2 timeout 300 python -m pytest tests/test_parity_gpu.py -x -q -p no:cacheprovider -k "cfg1 or fused_and_streaming or deterministic or large_planes or backward_variants or cfg2" 2>&1 | tail -2
