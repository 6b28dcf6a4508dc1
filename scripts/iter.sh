#!/bin/bash
# one GPU iteration: parity subset, a bench line, ncu of one kernel.  scripts/iter.sh OUT [KREGEX] [PYTEST_K]
OUT=${1:-gpurun_out/it}; RX=${2:-k_events_l}; TK=${3:-"config1 or small_counters or config2 or random_traces or multi_stream or tables_only or zero_events or dense_spans"}
mkdir -p $OUT
timeout 900 python -m pytest tests -m gpu -q -x -k "$TK" > $OUT/tests.log 2>&1; echo rc=$? >> $OUT/tests.log
timeout 600 python bench.py --no-cpu-baseline --no-e2e --no-full > $OUT/bench.log 2>&1
bash scripts/ncu_kernel.sh $OUT/prof "$RX"
ncu -i $OUT/prof.ncu-rep --page details --csv > $OUT/prof_details.csv 2>/dev/null
ncu -i $OUT/prof.ncu-rep --page source --csv > $OUT/prof_source.csv 2>/dev/null
