timeout 600 python -m pytest tests -m "gpu and not slow" -q -x --timeout 300 -p no:cacheprovider > gpurun_out/gpu_tests.log 2>&1; echo rc=$? >> gpurun_out/gpu_tests.log
B="python bench.py --steps 60 --warmup 5 --e2e-steps 0 --no-cpu-baseline"
for kb in 64 100 200; do IABN_FUSED_SMEM_KB=$kb timeout 300 $B > gpurun_out/s4_kb$kb.log 2>&1; done
timeout 300 $B --config r50s3 > gpurun_out/s4_r50.log 2>&1
echo done
