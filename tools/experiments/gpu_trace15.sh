for cfg in "8 2" "8 1" "4 1"; do set -- $cfg; IABN_FUSED_DEBUG=4 IABN_FUSED_K=$1 IABN_FUSED_NBUF=$2 timeout 300 python tools/trace_fused.py > gpurun_out/t15_k$1_nb$2.log 2>&1; done
echo done
