#!/bin/bash
# Profiling pass for one bench configuration (run under gpurun, 1 GPU):
#   bench.log       : the bench JSON line (default flags, CPU baseline included)
#   launches.csv    : every kernel launch of 3 warm-up + 1 timed step, device time (cold, serialised)
#   prof_events     : ncu --set full of the event pass (k_events_w), one launch of the timed step
#   prof_tables     : ncu --set full of the counter pass and the sub-run -> instance sum, timed step
OUT=${1:-gpurun_out}
mkdir -p $OUT
timeout 600 python bench.py > $OUT/bench.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches.csv \
    python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > $OUT/launches_bench.log 2>&1
python scripts/launches.py $OUT/launches.csv 4 40 > $OUT/launches.txt 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_events -s 3 -c 1 -f -o $OUT/prof_events \
    python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > $OUT/prof_events.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:"k_counters_tiled|k_sum_rows_chunked|k_sum_rows_cols" \
    -s 9 -c 3 -f -o $OUT/prof_tables \
    python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > $OUT/prof_tables.log 2>&1
ls -la $OUT
