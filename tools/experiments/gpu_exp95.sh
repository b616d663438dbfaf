# deeper slab rings for small slabs (IABN_FUSED_DEEP=1 default) vs nbuf 2
R="python bench.py --config r50s3 --e2e-steps 0 --no-cpu-baseline"
for d in 0 1; do
  echo "DEEP=$d r50s3 $(IABN_FUSED_DEEP=$d timeout 300 $R 2>&1 | tail -1 | grep -o '"ms_per_step": [0-9.]*')"
  for cfg in "rx101 bf16" "rx101 f32" "densenet264 bf16"; do
    set -- $cfg
    echo "DEEP=$d $cfg $(IABN_FUSED_DEEP=$d timeout 600 python tools/sweep.py --net $1 --dtype $2 2>/dev/null | tail -1 | grep -o '"graph_pct_of_peak": [0-9.]*')"
  done
  IABN_FUSED_DEEP=$d timeout 300 python tools/sync_emulated.py --cfg r50s3 --G 8 2>&1 | grep '"G": 8'
  IABN_FUSED_DEEP=$d timeout 300 python tools/sync_emulated.py --cfg wrn38 --G 8 2>&1 | grep '"G": 8'
done
IABN_VERBOSE=1 timeout 300 python tools/sync_emulated.py --cfg r50s3 --G 8 2>&1 | grep "\[iabn\]" | head
