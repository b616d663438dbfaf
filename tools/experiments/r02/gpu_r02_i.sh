# ncu: the fused-collective sync kernel (one-GPU emulation, plain launch) and the plain fused kernels
export IABN_EMU_NONCOOP=1
timeout 300 python tools/emu_probe.py 16 4096 12544 8 > gpurun_out/i_emu_plain.log 2>&1 && timeout 1200 ncu --set full --clock-control none --import-source on -k regex:fused_kernel -s 2 -c 2 -o gpurun_out/i_sync_emu python tools/emu_probe.py 16 4096 12544 8 > gpurun_out/i_ncu_sync.log 2>&1; echo rc=$? >> gpurun_out/i_ncu_sync.log
unset IABN_EMU_NONCOOP
C="python bench.py --steps 2 --warmup 3 --e2e-steps 0 --no-cpu-baseline --sync-emulated 0"
timeout 300 $C > gpurun_out/i_plain.log 2>&1 && timeout 900 ncu --set full --clock-control none --import-source on -k regex:fused_kernel -s 2 -c 2 -o gpurun_out/i_fused $C > gpurun_out/i_ncu_fused.log 2>&1; echo rc=$? >> gpurun_out/i_ncu_fused.log
