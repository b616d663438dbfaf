# DenseNet-264 NHWC per-shape device times (streaming vs grid-resident)
for g in 0 1; do
  IABN_GRES=$g timeout 600 python tools/sweep.py --net densenet264 --dtype bf16 --layout NHWC > gpurun_out/sw_dn_nhwc_gres$g.json 2>/dev/null
  python - gpurun_out/sw_dn_nhwc_gres$g.json <<'PY'
import json, sys
d = json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
print(sys.argv[1], "graph", d["graph_ms"], "ms", d["graph_pct_of_peak"], "%")
for r in sorted(d["per_shape"], key=lambda r: -r["share_pct"])[:8]:
    print("   ", r)
PY
done
