# host cost per call: before this session's changes (_old = 576d211) vs now
for d in _old .; do
  echo "$d $(cd $d && timeout 120 python tools/call_overhead.py 2>&1 | tail -1)"
done
for d in _old .; do
  echo "$d $(cd $d && timeout 300 python tools/fig4_blocks.py --dtype f32 --iters 100 2>/dev/null | python -c "
import json,sys; d=json.load(sys.stdin); print([(b['block'], b['standard']['ms'], b['inplace_abn']['ms']) for b in d['blocks']])")"
done
