#!/bin/bash
# Profiling pass for one bench configuration (run under gpurun, 1 GPU).
#   launches.csv : every kernel launch of warm-up + 1 timed step, device time (cold, serialized)
#   prof_events  : ncu --set full of the fused event pass (k_events), one launch
set -x
OUT=${1:-gpurun_out}
mkdir -p $OUT
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches.csv \
    python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > $OUT/launches_bench.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_events -s 3 -c 1 -f -o $OUT/prof_events \
    python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > $OUT/prof_events.log 2>&1
ls -la $OUT
