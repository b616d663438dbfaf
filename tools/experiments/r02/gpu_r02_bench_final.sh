# final bench line (default arguments) + its ncu launch list, after the last code changes
IABN_VERBOSE=0 timeout 600 python bench.py > gpurun_out/fb_bench.log 2>&1; echo rc=$? >> gpurun_out/fb_bench.log
timeout 600 python bench.py --impl reference --steps 5 --warmup 1 > gpurun_out/fb_ref.log 2>&1
C="python bench.py --steps 2 --warmup 3 --e2e-steps 0 --no-cpu-baseline --sync-emulated 0"
timeout 300 $C > gpurun_out/fb_plain.log 2>&1 && timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/fb_launches.csv $C > gpurun_out/fb_ncu.log 2>&1
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/fb_smoke.log 2>&1; echo rc=$? >> gpurun_out/fb_smoke.log
tail -2 gpurun_out/fb_bench.log | cut -c1-300; tail -2 gpurun_out/fb_smoke.log
