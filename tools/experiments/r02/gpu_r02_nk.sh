# NHWC channel-group K target ~96 CTAs for <= 16 groups: tune auto column + NHWC sweeps + NHWC tests
python -m pytest tests -m gpu -x -q -k "nhwc or NHWC" 2>&1 | tail -1
python tools/nhwc_tune.py --dtype bf16 --shapes 256x196,128x784,160x784,192x196 --gs 16 --ks 6,8 2>&1 | grep -v '^{"dtype' | cut -c1-200
python tools/nhwc_tune.py --dtype f32 --shapes 128x196,128x784,64x784 --gs 8 --ks 6,8 2>&1 | grep -v '^{"dtype' | cut -c1-200
for net in densenet264 rx101; do for dt in bf16 f32; do
  python tools/sweep.py --net $net --dtype $dt --layout NHWC > gpurun_out/nk_sweep_${net}_${dt}.json 2>&1
  python -c "import json; d=json.loads(open('gpurun_out/nk_sweep_${net}_${dt}.json').read().strip().splitlines()[-1]); print('$net $dt', d['graph_ms'], d['graph_pct_of_peak'])"
done; done
