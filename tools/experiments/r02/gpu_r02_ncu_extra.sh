# ncu --set full summaries (on the box, keeps gpurun_out small): BN + sigmoid channel-resident
# kernels (fp32 32x256x56^2) and the small-layer kernels after the division-free coefficients
P1="python tools/act_once.py sigmoid NCHW 32x256x3136"
timeout 120 $P1 > gpurun_out/x_probe1.log 2>&1 && timeout 600 ncu --set full --clock-control none --import-source on -k regex:fused_kernel -s 2 -c 2 -o gpurun_out/x_act_fused $P1 > gpurun_out/x_ncu1.log 2>&1
python tools/ncu_summary.py gpurun_out/x_act_fused.ncu-rep > gpurun_out/x_act_fused_summary.txt 2>&1; rm -f gpurun_out/x_act_fused.ncu-rep
P2="python tools/layer_probe.py 32 512 196 bf16 NCHW"
timeout 120 $P2 > gpurun_out/x_probe2.log 2>&1 && timeout 600 ncu --set full --clock-control none --import-source on -k regex:small_kernel -s 2 -c 2 -o gpurun_out/x_small $P2 > gpurun_out/x_ncu2.log 2>&1
python tools/ncu_summary.py gpurun_out/x_small.ncu-rep > gpurun_out/x_small_summary.txt 2>&1; rm -f gpurun_out/x_small.ncu-rep
head -40 gpurun_out/x_act_fused_summary.txt | grep -v "^ *[0-9.]*%"
