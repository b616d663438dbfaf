# NHWC bulk-ring reductions: cluster size 1 / 4 / 8 (records summed over DSMEM), A/B on one box
for v in k8 k4 k1 k8 k4 k1; do cp ab/lib_$v.so paper_1712_02616_b200/libiabn.so; echo $v
  for sh in 32x128x3136 32x64x12544 32x256x784; do python tools/phase_time.py --shape $sh | python -c "import json,sys; d=json.loads(sys.stdin.readline()); print(' ', d['shape'], d['fwd_reduce'], d['fwd_whole'], d['bwd_reduce'], d['bwd_whole'])"; done
done
cp ab/lib_k8.so paper_1712_02616_b200/libiabn.so
