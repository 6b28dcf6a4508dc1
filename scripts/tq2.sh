#!/bin/bash
# tq.sh + ncu --set full of one kernel (KRX) of the bench step
OUT=${1:-gpurun_out/tq}
bash scripts/tq.sh $OUT
timeout 300 bash scripts/ncu_kernel.sh $OUT/k "${KRX:-k_counters_seg}" 4 ${KSKIP:-3} 1
