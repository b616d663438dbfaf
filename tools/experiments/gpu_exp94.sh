# regression hunt 2: base vs default (late release) vs _v2 (early relaxed release)
B="python bench.py --steps 20 --e2e-steps 0 --no-cpu-baseline"
R="python bench.py --config r50s3 --e2e-steps 0 --no-cpu-baseline"
for i in 1 2; do
for d in _base . _v2; do
  echo "$d wrn38 $(cd $d && timeout 300 $B 2>&1 | tail -1 | grep -o '"ms_per_step": [0-9.]*')  r50s3 $(cd $d && timeout 300 $R 2>&1 | tail -1 | grep -o '"ms_per_step": [0-9.]*')"
done
done
(cd _v2 && timeout 300 python -m pytest tests/test_sync_fused_gpu.py -x -q 2>&1 | tail -1)
for c in wrn38 r50s3; do (cd _v2 && timeout 300 python tools/sync_emulated.py --cfg $c --G 2,8 2>&1 | grep '"G": [28]'); done
