# plain wrn38: chunk size (16-byte vectors per chunk; a plane is 1568) with the L2 prefetch on
B="python bench.py --steps 100 --e2e-steps 0 --no-cpu-baseline --sync-emulated 0"
p() { python -c 'import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(d["fwd_ms"], d["bwd_ms"], d["pct_of_peak"])'; }
for i in 1 2; do
for c in 0 392 784 3136; do
echo "chunk=$c  $(IABN_FUSED_CHUNK=$c $B 2>/dev/null | p)"
done; done
S="python tools/sync_emulated.py --cfg wrn38 --iters 10"
for c in 0 392 784; do
  IABN_FUSED_CHUNK=$c timeout 200 $S --G 2,8 2>&1 | grep '"fused-collective' | python -c '
import sys,json
for l in sys.stdin:
    d=json.loads(l)
    if "G" in d and "fwd_us" in d: print("sync chunk='$c'", d["G"], d["fwd_us"], d["bwd_us"], d["pct_of_peak"])'
done
