# copy the outputs of tools/experiments/gpu_final.sh (gpurun_out/fin_*) into profiles/ (round $1, default r01)
set -e
R=${1:-r01}; G=gpurun_out; P=profiles
grep '^{' $G/fin_bench.log | tail -1 > $P/${R}_bench.jsonl
grep '^{' $G/fin_r50.log | tail -1 > $P/${R}_bench_r50s3.jsonl
grep '^{' $G/fin_ref.log | tail -1 > $P/${R}_bench_reference_arm.jsonl
grep '^{' $G/fin_stream.log | tail -1 > $P/${R}_bench_streaming_schedule.jsonl
cp $G/fin_fused.ncu-rep $P/${R}_fused_kernels.ncu-rep
python tools/ncu_summary.py $G/fin_fused.ncu-rep > $P/${R}_ncu_full_fused_summary.txt
python tools/launch_csv.py $G/fin_launches.csv > $P/${R}_launches.csv
cp $G/fin_trace.log $P/${R}_trace_phases_k8.txt
for f in $G/fin_sweep_*.json; do b=$(basename $f .json); cp $f $P/${R}_sweep_${b#fin_sweep_}.json; done
for c in wrn38 r50s3 rx101_14; do grep '^{' $G/fin_sync_emu_$c.json | tail -1 > $P/${R}_sync_emulated_$c.json; done
cp $G/fin_fig4_f32.json $P/${R}_fig4_blocks_f32.json; cp $G/fin_fig4_bf16.json $P/${R}_fig4_blocks_bf16.json
tail -2 $G/fin_tests.log
