timeout 600 python tools/fig4_blocks.py --dtype f32 > gpurun_out/fig4_f32.json 2> gpurun_out/fig4_f32.err
timeout 600 python tools/fig4_blocks.py --dtype bf16 > gpurun_out/fig4_bf16.json 2> gpurun_out/fig4_bf16.err
echo done
