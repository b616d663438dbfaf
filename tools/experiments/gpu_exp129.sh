# warp-wide producer issue only for chunks of >= 4 planes: parity, A/B vs HEAD (_prev), sweeps
timeout 900 python -m pytest tests/test_parity_gpu.py tests/test_sync_fused_gpu.py tests/test_parity_full_gpu.py -x -q 2>&1 | tail -2
R="python bench.py --config r50s3 --e2e-steps 0 --no-cpu-baseline --sync-emulated 0"
W="python bench.py --steps 100 --e2e-steps 0 --no-cpu-baseline --sync-emulated 0"
p() { python -c 'import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(d["fwd_ms"], d["bwd_ms"], d["pct_of_peak"])'; }
for i in 1 2 3; do for d in _prev .; do
  echo "wrn38 $d $(cd $d && $W 2>/dev/null | p)"
  echo "r50s3 $d $(cd $d && $R 2>/dev/null | p)"
done; done
for cfg in "rx101 bf16 NCHW" "rx101 f32 NCHW" "densenet264 bf16 NCHW" "densenet264 f32 NCHW"; do
  set -- $cfg
  timeout 600 python tools/sweep.py --net $1 --dtype $2 --layout $3 > gpurun_out/e129_$1_$2_$3.json 2>/dev/null
  python -c "import json; d=json.load(open('gpurun_out/e129_$1_$2_$3.json')); print('$1 $2', d['graph_ms'], d['graph_pct_of_peak'])"
done
for c in r50s3 rx101_14 wrn38; do
  timeout 300 python tools/sync_emulated.py --cfg $c --iters 10 2>&1 | grep '^{' | tail -1 > gpurun_out/e129_sync_$c.json
  python -c "import json; d=json.load(open('gpurun_out/e129_sync_$c.json')); print('$c', [(r['G'], r['pct_of_peak']) for r in d['rows']])"
done
