# NHWC bulk-ring reductions: GPU tests, then whole-network NHWC sweeps with and without
python -m pytest tests -m gpu -x -q > gpurun_out/nb_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/nb_tests.log
for net in densenet264 rx101; do for dt in bf16 f32; do
  IABN_NHWC_BULK=0 python tools/sweep.py --net $net --dtype $dt --layout NHWC > gpurun_out/nb_sweep_${net}_${dt}_off.json 2>&1
  python tools/sweep.py --net $net --dtype $dt --layout NHWC > gpurun_out/nb_sweep_${net}_${dt}_on.json 2>&1
done; done
tail -3 gpurun_out/nb_tests.log
for f in gpurun_out/nb_sweep_*; do echo $f; python -c "import json,sys; d=json.loads(open('$f').read().strip().splitlines()[-1]); print(d['graph_ms'], d['graph_pct_of_peak'])"; done
