# ResNet-50 stage 3 (64x1024x14^2 fp32): fused-plan knobs
run() { echo "$*"; env "$@" timeout 120 python bench.py --config r50s3 --steps 50 --warmup 5 --e2e-steps 0 --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.readline()); print('  ms', d['ms_per_step'], 'pct', round(100*d['value']/6449.4,1), 'fwd', d['roofline']['forward']['frac'], 'bwd', d['roofline']['frac'])"; }
run IABN_X=0
for k in 1 2 4 8; do for mb in 2 4; do run IABN_FUSED_K=$k IABN_FUSED_MINB=$mb; done; done
run IABN_FUSED_DYN=2
run IABN_FUSED_DEEP=0
run IABN_FUSED_SMALL_KB=70
run IABN_FUSED_SMALL_KB=35
run IABN_SMALL_MAX_KB=64
