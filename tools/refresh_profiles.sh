# copy the outputs of tools/experiments/gpu_final.sh (gpurun_out/fin_*) into profiles/ (round $1, default r01)
set -e
R=${1:-r01}; G=gpurun_out; P=profiles
grep '^{' $G/fin_bench.log | tail -1 > $P/${R}_bench.jsonl
grep '^{' $G/fin_r50.log | tail -1 > $P/${R}_bench_r50s3.jsonl
grep '^{' $G/fin_ref.log | tail -1 > $P/${R}_bench_reference_arm.jsonl
grep '^{' $G/fin_stream.log | tail -1 > $P/${R}_bench_streaming_schedule.jsonl
cp $G/fin_fused.ncu-rep $P/${R}_fused_kernels.ncu-rep
cp $G/fin_fused_summary.txt $P/${R}_ncu_full_fused_summary.txt
python tools/launch_csv.py $G/fin_launches.csv > $P/${R}_launches.csv
cp $G/fin_trace.log $P/${R}_trace_phases_k8.txt
for f in $G/fin_sweep_*.json; do b=$(basename $f .json); cp $f $P/${R}_sweep_${b#fin_sweep_}.json; done
for c in wrn38 r50s3 rx101_14; do grep '^{' $G/fin_sync_emu_$c.json | tail -1 > $P/${R}_sync_emulated_$c.json; done
cp $G/fin_fig4_f32.json $P/${R}_fig4_blocks_f32.json; cp $G/fin_fig4_bf16.json $P/${R}_fig4_blocks_bf16.json
for f in fin_act_nchw fin_act_nhwc; do [ -f $G/$f.log ] && grep '^{' $G/$f.log | tail -1 > $P/${R}_${f#fin_}_bench.json; done
[ -f $G/fin_phase_nhwc.jsonl ] && grep '^{' $G/fin_phase_nhwc.jsonl > $P/${R}_phase_times_nhwc.jsonl
[ -f $G/fin_latency_floor.json ] && cp $G/fin_latency_floor.json $P/${R}_latency_floor.json
[ -f $G/fin_nb_trace_fwd.log ] && cat $G/fin_nb_trace_fwd.log $G/fin_nb_trace_bwd.log > $P/${R}_nb_trace_128x3136_bf16.txt
for f in fin_nhwc_trace_fwd fin_nhwc_trace_bwd; do [ -f $G/$f.log ] && cp $G/$f.log $P/${R}_${f#fin_}.txt; done
[ -f $G/fin_nhwc_stream_128x3136_summary.txt ] && cp $G/fin_nhwc_stream_128x3136_summary.txt $P/${R}_ncu_full_nhwc_streaming_128x3136_bf16_summary.txt
[ -f $G/fin_nhwc_128x196_summary.txt ] && cp $G/fin_nhwc_128x196_summary.txt $P/${R}_ncu_full_nhwc_128x196_bf16_summary.txt
[ -f $G/fin_small_512x196_summary.txt ] && cp $G/fin_small_512x196_summary.txt $P/${R}_ncu_full_small_512x196_bf16_summary.txt
[ -f $G/fin_act_launches.csv ] && python tools/launch_csv.py $G/fin_act_launches.csv > $P/${R}_act_launches.csv
for n in 2 4; do [ -f $G/fin_dry$n.log ] && grep '^{' $G/fin_dry$n.log | tail -1 > $P/${R}_bench_dryrun_${n}ranks_shim.jsonl; done
tail -2 $G/fin_tests.log
