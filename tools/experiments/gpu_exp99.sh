# joint reduce/apply warps for few channels per CTA
timeout 600 python -m pytest tests -m gpu -x -q -p no:cacheprovider 2>&1 | tail -1
R="python bench.py --config r50s3 --e2e-steps 0 --no-cpu-baseline --sync-emulated 0"
for j in 0 2 4 16; do
  echo "JOINT=$j r50s3 $(IABN_FUSED_JOINT=$j timeout 300 $R 2>&1 | tail -1 | grep -o '"ms_per_step": [0-9.]*')"
  for cfg in "rx101 bf16" "rx101 f32" "densenet264 bf16"; do
    set -- $cfg
    echo "JOINT=$j $cfg $(IABN_FUSED_JOINT=$j timeout 600 python tools/sweep.py --net $1 --dtype $2 2>/dev/null | tail -1 | grep -o '"graph_pct_of_peak": [0-9.]*')"
  done
done
