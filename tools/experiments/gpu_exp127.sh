# producer bulk copies spread over the warp (default) vs lane 0 only (IABN_FUSED_DEBUG=8)
timeout 900 python -m pytest tests/test_parity_gpu.py tests/test_sync_fused_gpu.py tests/test_parity_full_gpu.py -x -q 2>&1 | tail -2
R="python bench.py --config r50s3 --e2e-steps 0 --no-cpu-baseline --sync-emulated 0"
W="python bench.py --steps 100 --e2e-steps 0 --no-cpu-baseline --sync-emulated 0"
p() { python -c 'import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(d["fwd_ms"], d["bwd_ms"], d["pct_of_peak"])'; }
for i in 1 2; do
  echo "r50s3 warp   $($R 2>/dev/null | p)"
  echo "r50s3 lane0  $(IABN_FUSED_DEBUG=8 $R 2>/dev/null | p)"
  echo "wrn38 warp   $($W 2>/dev/null | p)"
  echo "wrn38 lane0  $(IABN_FUSED_DEBUG=8 $W 2>/dev/null | p)"
done
for cfg in "rx101 bf16 NCHW" "rx101 f32 NCHW" "densenet264 bf16 NCHW"; do
  set -- $cfg
  for m in 0 8; do
    IABN_FUSED_DEBUG=$m timeout 600 python tools/sweep.py --net $1 --dtype $2 --layout $3 > gpurun_out/e127_$1_$2_$m.json 2>/dev/null
    python -c "import json; d=json.load(open('gpurun_out/e127_$1_$2_$m.json')); print('$1 $2 dbg=$m', d['graph_ms'], d['graph_pct_of_peak'])"
  done
done
