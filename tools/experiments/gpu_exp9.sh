timeout 600 python -m pytest tests -m "gpu and not slow" -q -x --timeout 300 -p no:cacheprovider > gpurun_out/gpu_tests.log 2>&1; echo rc=$? >> gpurun_out/gpu_tests.log
B="python bench.py --steps 60 --warmup 5 --e2e-steps 0 --no-cpu-baseline"
IABN_VERBOSE=1 timeout 300 $B > gpurun_out/e9_auto.log 2>&1
for k in 2 4 8; do for nb in 2 3; do IABN_VERBOSE=1 IABN_FUSED_K=$k IABN_FUSED_NBUF=$nb timeout 300 $B > gpurun_out/e9_k${k}_nb$nb.log 2>&1; done; done
IABN_VERBOSE=1 IABN_FUSED_K=16 IABN_FUSED_NBUF=2 timeout 300 $B > gpurun_out/e9_k16_nb2.log 2>&1
IABN_VERBOSE=1 timeout 300 $B --config r50s3 > gpurun_out/e9_r50.log 2>&1
echo done
