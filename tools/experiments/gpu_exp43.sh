B="python bench.py --steps 60 --warmup 5 --e2e-steps 0 --no-cpu-baseline --config r50s3"
for k in 1 2 4 8; do IABN_VERBOSE=1 IABN_FUSED_K=$k timeout 300 $B > gpurun_out/e43_k$k.log 2>&1; done
IABN_VERBOSE=1 timeout 300 $B > gpurun_out/e43_auto.log 2>&1
echo done
