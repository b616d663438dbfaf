# NHWC bulk-ring statistics: L2 evict_last policy on x (the apply re-reads it) vs default, A/B
for v in base el base el; do cp ab/lib_$v.so paper_1712_02616_b200/libiabn.so; echo $v
  for sh in 32x128x3136 32x64x12544 32x256x784; do python tools/phase_time.py --shape $sh | python -c "import json,sys; d=json.loads(sys.stdin.readline()); print(' ', d['shape'], d['fwd_reduce'], d['fwd_apply'], d['fwd_whole'], d['bwd_whole'])"; done
done
cp ab/lib_base.so paper_1712_02616_b200/libiabn.so
