# NHWC: channel-group schedule off (streaming everywhere) -- per-shape comparison
for net in densenet264 rx101; do for dt in bf16 f32; do
  IABN_NHWC_FUSED=0 python tools/sweep.py --net $net --dtype $dt --layout NHWC > gpurun_out/nb_sweep_${net}_${dt}_stream.json 2>&1
  python -c "import json; d=json.loads(open('gpurun_out/nb_sweep_${net}_${dt}_stream.json').read().strip().splitlines()[-1]); print('$net $dt', d['graph_ms'], d['graph_pct_of_peak'])"
done; done
