# small-layer kernels: explicit early PDL trigger vs none, A/B on one box (small_tune + NCHW bf16 sweeps)
for v in base et base et; do cp ab/lib_$v.so paper_1712_02616_b200/libiabn.so
  echo $v; python tools/small_tune.py --dtype bf16 --shapes 512x196,1024x196,2048x49,128x196 2>&1 | grep -v '^{' | python -c "
import sys, json
for l in sys.stdin:
    sh, r = l.split(' ', 1); print(' ', sh, json.loads(r)['auto'])"
  for net in rx101 densenet264; do python tools/sweep.py --net $net --dtype bf16 --layout NCHW 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.readline()); print('  $net', d['graph_ms'], d['graph_pct_of_peak'])"; done
done
cp ab/lib_base.so paper_1712_02616_b200/libiabn.so
