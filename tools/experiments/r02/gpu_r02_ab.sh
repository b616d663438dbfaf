# A/B of the headline bench between two builds of libiabn.so on one box (ab/ is scratch)
B="python bench.py --steps 150 --warmup 5 --e2e-steps 0 --no-cpu-baseline"
for i in 1 2; do for v in head d515e36; do
  cp ab/libiabn_$v.so paper_1712_02616_b200/libiabn.so
  $B 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.readline()); print('$v', d['ms_per_step'], d['pct_of_peak'], d['roofline']['frac'], d['roofline']['forward']['frac'], d['clocks']['sm_mhz'])"
done; done
cp ab/libiabn_head.so paper_1712_02616_b200/libiabn.so
