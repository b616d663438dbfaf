timeout 900 python -m pytest tests -m "gpu and not slow" -q --timeout 600 -p no:cacheprovider -k "fused or cfg2 or wrn or edge or tiny or variant or beta" > gpurun_out/gpu_tests.log 2>&1; echo rc=$? >> gpurun_out/gpu_tests.log
B="python bench.py --steps 60 --warmup 5 --e2e-steps 0 --no-cpu-baseline"
for j in 1 0; do
IABN_FUSED_JOINT=$j timeout 300 $B > gpurun_out/e59_j$j.log 2>&1
IABN_FUSED_JOINT=$j timeout 300 $B --config r50s3 > gpurun_out/e59_r50_j$j.log 2>&1
done
IABN_FUSED_DEBUG=4 timeout 300 python tools/trace_fused.py > gpurun_out/t59.log 2>&1
echo done
