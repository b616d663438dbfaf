B="python bench.py --config r50s3 --steps 100 --warmup 5 --e2e-steps 0 --no-cpu-baseline"
for cfgv in "0 0 0" "1 1 4" "4 2 4" "2 1 4" "2 2 4" "1 2 2" "2 3 4" "4 1 4"; do
  set -- $cfgv
  if [ $1 = 0 ]; then timeout 300 $B > gpurun_out/e75_default.log 2>&1; continue; fi
  IABN_VERBOSE=1 IABN_FUSED_K=$1 IABN_FUSED_NBUF=$2 IABN_FUSED_MINB=$3 IABN_FUSED_SMALL_KB=100 timeout 300 $B > gpurun_out/e75_k$1_n$2_m$3.log 2>&1
done
echo done
