# small-layer backward: CTAs-per-SM register cap 4 (spills) vs 3 (no spills), A/B on one box
for v in b4 b3 b4 b3; do cp ab/lib_$v.so paper_1712_02616_b200/libiabn.so
  echo $v; python tools/small_tune.py --dtype bf16 --shapes 512x196,1024x196,2048x49,128x196 2>&1 | grep -v '^{' | python -c "
import sys, json
for l in sys.stdin:
    sh, r = l.split(' ', 1); print(' ', sh, json.loads(r)['auto'])"
done
cp ab/lib_b4.so paper_1712_02616_b200/libiabn.so
