#!/bin/bash
# ncu --set full with source of the event pass and the counter pass (config 4), plus per-line source pages
OUT=${1:-gpurun_out/src}
mkdir -p $OUT
bash scripts/ncu_kernel.sh $OUT/ev k_events_l 4
bash scripts/ncu_kernel.sh $OUT/ct k_counters_tiled 4
for f in ev ct; do
  ncu -i $OUT/$f.ncu-rep --page source --csv --print-source sass > $OUT/$f.sass.csv 2>/dev/null
  ncu -i $OUT/$f.ncu-rep --page source --csv --print-source cuda > $OUT/$f.cuda.csv 2>/dev/null
  ncu -i $OUT/$f.ncu-rep --page raw --csv > $OUT/$f.raw.csv 2>/dev/null
done
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches_shard.csv \
    python bench.py --traced 0 --steps 1 --warmup 3 --no-cpu-baseline --no-e2e --no-full > $OUT/launches_shard.log 2>&1
python scripts/launches.py $OUT/launches_shard.csv 4 > $OUT/launches_shard.txt 2>&1
ls -la $OUT
