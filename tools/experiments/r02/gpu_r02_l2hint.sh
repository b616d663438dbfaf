# small-layer loads: L2 prefetch-size hint none / 128B / 256B, A/B on one box
for v in h0 h128 h256 h0 h128 h256; do cp ab/lib_$v.so paper_1712_02616_b200/libiabn.so
  echo $v; python tools/small_tune.py --dtype bf16 --shapes 512x196,1024x196,2048x49,128x196 2>&1 | grep -v '^{' | python -c "
import sys, json
for l in sys.stdin:
    sh, r = l.split(' ', 1); print(' ', sh, json.loads(r)['auto'])"
done
cp ab/lib_h0.so paper_1712_02616_b200/libiabn.so
