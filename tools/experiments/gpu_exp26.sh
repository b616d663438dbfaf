B="python bench.py --steps 60 --warmup 5 --e2e-steps 0 --no-cpu-baseline"
for ch in 784 1568; do IABN_FUSED_CHUNK=$ch timeout 300 $B > gpurun_out/e26_ch$ch.log 2>&1; done
for rw in "6 8" "3 9" "5 9"; do set -- $rw
IABN_NVCC_EXTRA="-DIABN_REDUCE_WARPS=$1 -DIABN_APPLY_WARPS=$2" python paper_1712_02616_b200/build.py --force > gpurun_out/b26.log 2>&1
timeout 300 $B > gpurun_out/e26_r$1a$2.log 2>&1
done
echo done
