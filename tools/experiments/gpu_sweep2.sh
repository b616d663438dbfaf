# parity first, then schedule sweeps of the persistent fused kernels
timeout 600 python -m pytest tests -m "gpu and not slow" -q -x --timeout 300 -p no:cacheprovider > gpurun_out/gpu_tests.log 2>&1; echo rc=$? >> gpurun_out/gpu_tests.log
B="python bench.py --steps 60 --warmup 5 --e2e-steps 0 --no-cpu-baseline"
for kb in 100 200; do for nb in 2 3; do IABN_FUSED_SMEM_KB=$kb IABN_FUSED_NBUF=$nb timeout 300 $B > gpurun_out/sweep_kb${kb}_nb${nb}.log 2>&1; done; done
IABN_FUSED_SMEM_KB=64 IABN_FUSED_NBUF=2 timeout 300 $B > gpurun_out/sweep_kb64_nb2.log 2>&1
IABN_FUSED_SMEM_KB=150 IABN_FUSED_NBUF=3 timeout 300 $B > gpurun_out/sweep_kb150_nb3.log 2>&1
timeout 300 $B --config r50s3 > gpurun_out/sweep_r50.log 2>&1
echo done
