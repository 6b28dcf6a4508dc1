#!/bin/bash
# every kernel launch of 3 warm-up + 1 timed bench step (device time, cold, serialised) + per-kernel share table
OUT=${1:-gpurun_out}
mkdir -p $OUT
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches.csv \
    python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e --no-full > $OUT/launches_bench.log 2>&1
python scripts/launches.py $OUT/launches.csv 4 > $OUT/launches.txt 2>&1
