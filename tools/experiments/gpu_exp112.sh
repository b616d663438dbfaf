# L2 cache hints on the prefetch / refill copies (IABN_FUSED_PF_HINT bits)
B="python bench.py --steps 50 --e2e-steps 0 --no-cpu-baseline --sync-emulated 0"
C="python bench.py --steps 2 --warmup 3 --e2e-steps 0 --no-cpu-baseline --sync-emulated 0"
for h in 0 1 2 3 0; do
  echo "HINT=$h $(IABN_FUSED_PF_HINT=$h timeout 120 $B 2>&1 | tail -1 | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["fwd_ms"], d["bwd_ms"], d["pct_of_peak"])')"
done
for h in 0 3; do
  IABN_FUSED_PF_HINT=$h timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:fused_kernel --csv $C 2>/dev/null | grep "fused_kernel<__nv_bfloat16, 1" | awk -F'","' '{print $(NF-3), $NF}' | tail -3 | sed "s/^/HINT=$h /"
done
