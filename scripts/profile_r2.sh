#!/bin/bash
# Round-2 measurement pass (one GPU, under gpurun):
#   bench4.log / bench5.log : bench JSON lines, config 4 (default) and config 5 (1B events)
#   launches4.csv/.txt      : every kernel launch of 3 warm-up + 1 timed config-4 step (cold, serialised)
#   prof_events4 / 5        : ncu --set full of the event pass k_events_w (config 4 / config 5)
#   prof_tables4            : ncu --set full of the counter pass and the sub-run -> instance sums (config 4)
OUT=${1:-gpurun_out}
mkdir -p $OUT
nvidia-smi --query-gpu=name,memory.total,clocks.max.sm --format=csv > $OUT/gpu.txt
timeout 900 python bench.py > $OUT/bench4.log 2>&1
timeout 1200 python bench.py --config 5 --steps 5 > $OUT/bench5.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches4.csv \
    python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e --no-full > $OUT/launches_bench.log 2>&1
python scripts/launches.py $OUT/launches4.csv 4 45 > $OUT/launches4.txt 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_events_w -s 3 -c 1 -f -o $OUT/prof_events4 \
    python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e --no-full > $OUT/prof_events4.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:"k_counters_tiled|k_sum_rows_chunked|k_sum_rows_cols|k_validate_events|k_lean_chain" \
    -s 15 -c 5 -f -o $OUT/prof_tables4 \
    python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e --no-full > $OUT/prof_tables4.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_events_w -s 3 -c 1 -f -o $OUT/prof_events5 \
    python bench.py --config 5 --steps 1 --warmup 3 --no-cpu-baseline --no-e2e --no-full > $OUT/prof_events5.log 2>&1
ls -la $OUT
