B="python bench.py --steps 40 --warmup 5 --e2e-steps 0 --no-cpu-baseline"
for ch in 512 1024 2048 3072; do IABN_FUSED_CHUNK=$ch IABN_VERBOSE=1 timeout 300 $B > gpurun_out/e17_ch$ch.log 2>&1; done
for ch in 1024 2048; do IABN_FUSED_CHUNK=$ch IABN_FUSED_K=4 IABN_FUSED_NBUF=1 IABN_VERBOSE=1 timeout 300 $B > gpurun_out/e17_k4_ch$ch.log 2>&1; done
echo done
