# NHWC bulk-ring reductions (cluster-summed records): GPU tests, phase times, NHWC sweeps
python -m pytest tests -m gpu -x -q > gpurun_out/nb_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/nb_tests.log
tail -3 gpurun_out/nb_tests.log
for sh in 32x128x3136 32x1216x196 32x64x12544 32x256x784; do python tools/phase_time.py --shape $sh; done
for net in densenet264 rx101; do for dt in bf16 f32; do
  python tools/sweep.py --net $net --dtype $dt --layout NHWC > gpurun_out/nb_sweep_${net}_${dt}_on.json 2>&1
  python -c "import json; d=json.loads(open('gpurun_out/nb_sweep_${net}_${dt}_on.json').read().strip().splitlines()[-1]); print('$net $dt', d['graph_ms'], d['graph_pct_of_peak'])"
done; done
