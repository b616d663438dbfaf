# plain wrn38 with the prefetch policy: repeat, and bwd-only prefetch
B="python bench.py --steps 100 --e2e-steps 0 --no-cpu-baseline --sync-emulated 0"
p() { python -c 'import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(d["fwd_ms"], d["bwd_ms"], d["pct_of_peak"], d["clocks"])'; }
for i in 1 2 3; do
echo "auto  $($B 2>/dev/null | p)"
echo "pf=2  $(IABN_FUSED_PREFETCH=2 $B 2>/dev/null | p)"
echo "_old  $(cd _old && $B 2>/dev/null | p)"
done
