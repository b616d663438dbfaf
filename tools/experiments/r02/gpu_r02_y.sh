# lockstep dynamic order of the fused-collective sync (IABN_SYNC_DYN=3): parity, then timing
IABN_SYNC_DYN=3 IABN_FUSED_DYN=1 timeout 900 python -m pytest -x -q tests/test_sync_fused_gpu.py -p no:cacheprovider > gpurun_out/y_t3.log 2>&1; echo rc=$? >> gpurun_out/y_t3.log
for d in 0 3; do
  for c in wrn38 r50s3; do
    IABN_SYNC_DYN=$d timeout 300 python tools/sync_emulated.py --cfg $c > gpurun_out/y_sync_emu_${c}_dyn$d.json 2>&1
  done
done
