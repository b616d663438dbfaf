timeout 600 python -m pytest tests -m "gpu and not slow" -q -x --timeout 300 -p no:cacheprovider > gpurun_out/gpu_tests.log 2>&1; echo rc=$? >> gpurun_out/gpu_tests.log
B="python bench.py --steps 60 --warmup 5 --e2e-steps 0 --no-cpu-baseline"
L=paper_1712_02616_b200/libiabn.so
for i in 1 2; do
timeout 300 $B > gpurun_out/e34_o1_$i.log 2>&1
timeout 300 $B --config r50s3 > gpurun_out/e34_r50_o1_$i.log 2>&1
done
IABN_FUSED_DEBUG=4 timeout 300 python tools/trace_fused.py > gpurun_out/t34.log 2>&1
echo done
