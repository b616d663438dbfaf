# fused-collective sync (emulated): plans with more slices in flight per CTA
for e in "X=1" "IABN_FUSED_K=2 IABN_FUSED_NBUF=2" "IABN_FUSED_K=2 IABN_FUSED_NBUF=2 IABN_FUSED_MINB=4"; do
  echo "== $e"
  env $e timeout 300 python tools/sync_emulated.py --cfg wrn38 --G 2,8 2>&1 | grep '^{"variant"' | python -c "
import sys, json
for l in sys.stdin:
    d = json.loads(l); print('  ', d['variant'][:32], d.get('fwd_us'), d.get('bwd_us'), d.get('pct_of_peak'), d.get('error', ''))"
done
