#!/bin/bash
# Round-2 measurement pass (one GPU, under gpurun): tests, bench lines, launch list, ncu captures
OUT=${1:-gpurun_out/r2m}
mkdir -p $OUT
nvidia-smi --query-gpu=name,memory.total,clocks.max.sm,driver_version --format=csv > $OUT/gpu.txt
timeout 1500 python -m pytest tests -m gpu -q > $OUT/gpu_tests.log 2>&1; echo rc=$? >> $OUT/gpu_tests.log
timeout 900 python bench.py > $OUT/bench4.log 2>&1
timeout 1200 python bench.py --config 5 --steps 5 > $OUT/bench5.log 2>&1
timeout 600 python bench.py --impl reference --steps 3 > $OUT/bench4_ref.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches4.csv \
    python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e --no-full > $OUT/launches_bench.log 2>&1
python scripts/launches.py $OUT/launches4.csv 4 60 > $OUT/launches4.txt 2>&1
bash scripts/ncu_kernel.sh $OUT/prof_events4 k_events_l 4
bash scripts/ncu_kernel.sh $OUT/prof_counters4 k_counters_tiled 4
bash scripts/ncu_kernel.sh $OUT/prof_tables4 "k_sum_rows_chunked|k_sum_rows_cols|k_points_iter|k_rx_onesweep|k_lean_chain|k_validate_events|k_meta_apply|k_keytab_blk" 4 24 8
bash scripts/ncu_kernel.sh $OUT/prof_events5 k_events_l 5
for f in prof_events4 prof_counters4 prof_tables4 prof_events5; do
  ncu -i $OUT/$f.ncu-rep --page details --csv > $OUT/$f.details.csv 2>/dev/null
  ncu -i $OUT/$f.ncu-rep --page raw --csv > $OUT/$f.raw.csv 2>/dev/null
done
ls -la $OUT
