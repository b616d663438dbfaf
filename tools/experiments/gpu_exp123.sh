# prefetch auto-on for double-buffered slices of >= 16 KB planes: sync emulation, plain, sweeps
for c in wrn38 r50s3 rx101_14; do
  timeout 300 python tools/sync_emulated.py --cfg $c --iters 10 2>&1 | grep '"fused' | python -c '
import sys,json
for l in sys.stdin:
    d=json.loads(l)
    if "G" in d and "fwd_us" in d: print("'$c'", d["G"], d["fwd_us"], d["bwd_us"], d["pct_of_peak"])'
done
B="python bench.py --steps 50 --e2e-steps 0 --no-cpu-baseline --sync-emulated 0"
p() { python -c 'import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(d["fwd_ms"], d["bwd_ms"], d["pct_of_peak"])'; }
echo "plain wrn38 $($B 2>/dev/null | p)"
echo "plain r50s3 $($B --config r50s3 2>/dev/null | p)"
for cfg in "rx101 f32 NCHW" "rx101 bf16 NCHW" "densenet264 f32 NCHW"; do
  set -- $cfg
  timeout 600 python tools/sweep.py --net $1 --dtype $2 --layout $3 > gpurun_out/e123_sweep_$1_$2_$3.json 2>/dev/null
done
