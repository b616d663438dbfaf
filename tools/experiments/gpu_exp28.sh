# unified reduce+apply group for single-buffered slices vs specialised warps
timeout 600 python -m pytest tests -m "gpu and not slow" -q -x --timeout 300 -p no:cacheprovider > gpurun_out/gpu_tests.log 2>&1; echo rc=$? >> gpurun_out/gpu_tests.log
B="python bench.py --steps 60 --warmup 5 --e2e-steps 0 --no-cpu-baseline"
for u in 1 0; do
  IABN_FUSED_UNIFIED=$u timeout 300 $B > gpurun_out/e28_u$u.log 2>&1
  IABN_FUSED_UNIFIED=$u timeout 300 $B --config r50s3 > gpurun_out/e28_r50_u$u.log 2>&1
done
# forward forced single-buffered too
IABN_FUSED_NBUF=1 IABN_FUSED_UNIFIED=1 timeout 300 $B > gpurun_out/e28_nb1_u1.log 2>&1
IABN_FUSED_NBUF=1 IABN_FUSED_UNIFIED=0 timeout 300 $B > gpurun_out/e28_nb1_u0.log 2>&1
IABN_FUSED_DEBUG=4 timeout 300 python tools/trace_fused.py > gpurun_out/t28.log 2>&1
echo done
