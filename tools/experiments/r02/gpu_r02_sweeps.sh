# all eight whole-network sweeps + the full GPU suite
python -m pytest tests -m gpu -x -q 2>&1 | tail -1
for net in rx101 densenet264; do for dt in f32 bf16; do for ly in NCHW NHWC; do
  python tools/sweep.py --net $net --dtype $dt --layout $ly > gpurun_out/sw_${net}_${dt}_${ly}.json 2>&1
  python -c "import json; d=json.loads(open('gpurun_out/sw_${net}_${dt}_${ly}.json').read().strip().splitlines()[-1]); print('$net $dt $ly', d['graph_ms'], d['graph_pct_of_peak'])"
done; done; done
