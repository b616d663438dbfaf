timeout 600 python -m pytest tests -m "gpu and not slow" -q -x --timeout 300 -p no:cacheprovider > gpurun_out/gpu_tests.log 2>&1; echo rc=$? >> gpurun_out/gpu_tests.log
B="python bench.py --steps 40 --warmup 5 --e2e-steps 0 --no-cpu-baseline"
IABN_VERBOSE=1 timeout 300 $B > gpurun_out/e13_auto.log 2>&1
for cfg in "4 1" "4 2" "8 1" "8 2" "6 2" "9 2"; do set -- $cfg; IABN_VERBOSE=1 IABN_FUSED_K=$1 IABN_FUSED_NBUF=$2 timeout 300 $B > gpurun_out/e13_k$1_nb$2.log 2>&1; done
C="python bench.py --steps 1 --warmup 3 --e2e-steps 0 --no-cpu-baseline"
export IABN_FUSED_K=8
IABN_FUSED_NBUF=1 timeout 900 ncu --set full --clock-control none --import-source on -k regex:fused_kernel -s 3 -c 1 -o gpurun_out/prof13_bwd $C > gpurun_out/ncu13.log 2>&1
echo done
