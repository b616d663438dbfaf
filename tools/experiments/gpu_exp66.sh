# backward with dz from L2 (z-only slabs, double-buffered) vs default
IABN_FUSED_DZG=1 timeout 900 python -m pytest tests -m gpu -q --timeout 600 -p no:cacheprovider -k "fused or cfg2 or wrn or variant or beta or large or graph or edge" > gpurun_out/gpu_tests.log 2>&1; echo rc=$? >> gpurun_out/gpu_tests.log
B="python bench.py --steps 60 --warmup 5 --e2e-steps 0 --no-cpu-baseline"
IABN_VERBOSE=1 IABN_FUSED_DZG=1 timeout 300 $B > gpurun_out/e66_dzg.log 2>&1
timeout 300 $B > gpurun_out/e66_base.log 2>&1
IABN_FUSED_DZG=1 IABN_FUSED_DEBUG=4 timeout 300 python tools/trace_fused.py > gpurun_out/t66.log 2>&1
echo done
