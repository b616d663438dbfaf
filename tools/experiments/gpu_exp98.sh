# covering-range kernels: partial slots out of the main loops
timeout 600 python -m pytest tests -m gpu -x -q -p no:cacheprovider -k "misaligned or sync or any_alignment or cfg1 or edge" 2>&1 | tail -2
IABN_FUSED_DEBUG=4 timeout 120 python tools/trace_fused.py --shape 32,1024,196,bf16 2>&1 | grep -E "==|last chunk|apply \(|residence|CTA first"
for cfg in "rx101 bf16 NCHW" "densenet264 bf16 NCHW" "rx101 f32 NCHW"; do
  set -- $cfg
  timeout 600 python tools/sweep.py --net $1 --dtype $2 --layout $3 > gpurun_out/sw_$1_$2_$3.json 2> gpurun_out/sw_$1_$2_$3.err
  python - gpurun_out/sw_$1_$2_$3.json <<'PY'
import json, sys
d = json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
print(d["net"], d["dtype"], d["layout"], "graph", d["graph_ms"], "ms", d["graph_pct_of_peak"], "%")
for r in sorted(d["per_shape"], key=lambda r: -r["share_pct"])[:4]:
    print("   ", r)
PY
done
