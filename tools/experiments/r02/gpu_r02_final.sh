# round-2 measurement set: tests, bench (default + reference arm + r50s3 + streaming + N>1 dry
# runs), sweeps, sync emulation, Fig. 4 blocks, phase trace, then ncu (launch list of the bench,
# full captures of the fused kernels, two small-layer shapes, the NHWC streaming kernels;
# act launch list)
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/fin_tests.log 2>&1; echo rc=$? >> gpurun_out/fin_tests.log
IABN_VERBOSE=1 timeout 600 python bench.py > gpurun_out/fin_bench.log 2>&1; echo rc=$? >> gpurun_out/fin_bench.log
timeout 600 python bench.py --impl reference --steps 5 --warmup 1 > gpurun_out/fin_ref.log 2>&1
timeout 300 python bench.py --config r50s3 --e2e-steps 1 > gpurun_out/fin_r50.log 2>&1
timeout 300 python bench.py --schedule streaming --steps 100 --e2e-steps 0 --no-cpu-baseline > gpurun_out/fin_stream.log 2>&1
timeout 600 python bench.py --emulate-ranks 2 --steps 50 --e2e-steps 2 > gpurun_out/fin_dry2.log 2>&1
timeout 600 python bench.py --emulate-ranks 4 --steps 50 --e2e-steps 2 > gpurun_out/fin_dry4.log 2>&1
for cfg in "rx101 f32 NCHW" "rx101 bf16 NCHW" "rx101 f32 NHWC" "rx101 bf16 NHWC" "densenet264 f32 NCHW" "densenet264 bf16 NCHW" "densenet264 f32 NHWC" "densenet264 bf16 NHWC"; do
  set -- $cfg
  timeout 600 python tools/sweep.py --net $1 --dtype $2 --layout $3 > gpurun_out/fin_sweep_$1_$2_$3.json 2> gpurun_out/fin_sweep_$1_$2_$3.err
done
for c in wrn38 r50s3 rx101_14; do
  timeout 300 python tools/sync_emulated.py --cfg $c > gpurun_out/fin_sync_emu_$c.json 2>&1
done
timeout 900 python tools/fig4_blocks.py --dtype f32 > gpurun_out/fin_fig4_f32.json 2> gpurun_out/fin_fig4_f32.err
timeout 900 python tools/fig4_blocks.py --dtype bf16 > gpurun_out/fin_fig4_bf16.json 2> gpurun_out/fin_fig4_bf16.err
IABN_FUSED_DEBUG=4 timeout 300 python tools/trace_fused.py > gpurun_out/fin_trace.log 2>&1
IABN_NHWC_TRACE=1 timeout 120 python tools/nhwc_trace.py 128 196 bf16 0 > gpurun_out/fin_nhwc_trace_fwd.log 2>&1
IABN_NHWC_TRACE=1 timeout 120 python tools/nhwc_trace.py 128 196 bf16 1 > gpurun_out/fin_nhwc_trace_bwd.log 2>&1
timeout 300 python tools/act_bench.py > gpurun_out/fin_act_nchw.log 2>&1
timeout 300 python tools/act_bench.py --layout NHWC --shapes 32x256x3136,32x512x784,32x1024x196,32x2048x49 > gpurun_out/fin_act_nhwc.log 2>&1
for sh in 32x128x3136 32x64x12544 32x256x784 32x1216x196; do timeout 120 python tools/phase_time.py --shape $sh; done > gpurun_out/fin_phase_nhwc.jsonl 2>&1
timeout 120 python tools/latency_floor.py > gpurun_out/fin_latency_floor.json 2>&1
IABN_NB_TRACE=1 timeout 120 python tools/nb_trace.py 128 3136 bf16 0 > gpurun_out/fin_nb_trace_fwd.log 2>&1
IABN_NB_TRACE=1 timeout 120 python tools/nb_trace.py 128 3136 bf16 1 > gpurun_out/fin_nb_trace_bwd.log 2>&1
echo measurements-done
C="python bench.py --steps 2 --warmup 3 --e2e-steps 0 --no-cpu-baseline --sync-emulated 0"
timeout 300 $C > gpurun_out/fin_plain.log 2>&1 && timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/fin_launches.csv $C > gpurun_out/fin_ncu_launch.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:fused_kernel -s 2 -c 2 -o gpurun_out/fin_fused $C > gpurun_out/fin_ncu_full.log 2>&1
# gpurun_out must stay under 64 MiB: keep the fused report, summarise the others here
summ() { [ -f gpurun_out/$1.ncu-rep ] && python tools/ncu_summary.py gpurun_out/$1.ncu-rep > gpurun_out/$1_summary.txt 2>&1 && rm -f gpurun_out/$1.ncu-rep; }
P1="python tools/layer_probe.py 32 128 196 bf16 NHWC"
timeout 120 $P1 > gpurun_out/fin_probe1.log 2>&1 && timeout 600 ncu --set full --clock-control none --import-source on -k regex:nhwc_fused -s 2 -c 2 -o gpurun_out/fin_nhwc_128x196 $P1 > gpurun_out/fin_ncu_nhwc.log 2>&1; summ fin_nhwc_128x196
P2="python tools/layer_probe.py 32 512 196 bf16 NCHW"
timeout 120 $P2 > gpurun_out/fin_probe2.log 2>&1 && timeout 600 ncu --set full --clock-control none --import-source on -k regex:small_kernel -s 2 -c 2 -o gpurun_out/fin_small_512x196 $P2 > gpurun_out/fin_ncu_small.log 2>&1; summ fin_small_512x196
P3="python tools/act_once.py leaky_relu NHWC 32x128x3136 bf16"
timeout 120 $P3 > gpurun_out/fin_probe3.log 2>&1 && timeout 600 ncu --set full --clock-control none --import-source on -k regex:"nhwc_bulk_reduce|apply_nhwc" -c 4 -o gpurun_out/fin_nhwc_stream_128x3136 $P3 > gpurun_out/fin_ncu_nhwc_stream.log 2>&1; summ fin_nhwc_stream_128x3136
P4="python tools/act_once.py sigmoid NCHW 32x256x3136"
timeout 120 $P4 > gpurun_out/fin_probe4.log 2>&1 && timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/fin_act_launches.csv $P4 > gpurun_out/fin_ncu_act.log 2>&1
python tools/ncu_summary.py gpurun_out/fin_fused.ncu-rep > gpurun_out/fin_fused_summary.txt 2>&1
du -sh gpurun_out
echo ncu-done
