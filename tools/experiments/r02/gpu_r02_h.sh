./tools/membench quick > gpurun_out/h_membench.txt 2>&1
timeout 120 python tools/emu_probe.py 4 24 196 2 > gpurun_out/h_emu_plain.log 2>&1 && timeout 180 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/h_emu_launches.csv python tools/emu_probe.py 4 24 196 2 > gpurun_out/h_emu_ncu.log 2>&1; echo ncu_rc=$? >> gpurun_out/h_emu_ncu.log
