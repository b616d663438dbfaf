timeout 600 python -m pytest tests -m "gpu and not slow" -q -x --timeout 300 -p no:cacheprovider > gpurun_out/gpu_tests.log 2>&1; echo rc=$? >> gpurun_out/gpu_tests.log
B="python bench.py --steps 40 --warmup 5 --e2e-steps 0 --no-cpu-baseline"
IABN_VERBOSE=1 timeout 300 $B > gpurun_out/e11_auto.log 2>&1
for cfg in "2 1" "4 1" "4 2" "6 2" "8 1" "8 2" "8 3" "12 2" "16 2" "16 1"; do set -- $cfg; IABN_VERBOSE=1 IABN_FUSED_K=$1 IABN_FUSED_NBUF=$2 timeout 300 $B > gpurun_out/e11_k$1_nb$2.log 2>&1; done
IABN_VERBOSE=1 timeout 300 $B --config r50s3 > gpurun_out/e11_r50.log 2>&1
echo done
