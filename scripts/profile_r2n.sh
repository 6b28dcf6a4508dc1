#!/bin/bash
# Round-2 measurement pass (one GPU, under gpurun): every GPU test, bench lines (config 4, shard, config 5,
# reference arm), launch lists, ncu --set full captures of the top kernels
OUT=${1:-gpurun_out/r2n}
mkdir -p $OUT
nvidia-smi --query-gpu=name,memory.total,clocks.max.sm,driver_version --format=csv > $OUT/gpu.txt
timeout 1800 python -m pytest tests -m gpu -q > $OUT/gpu_tests.log 2>&1; echo rc=$? >> $OUT/gpu_tests.log
timeout 900 python bench.py > $OUT/bench4.log 2>&1
timeout 600 python bench.py --traced 0 --no-cpu-baseline --no-e2e --no-full > $OUT/bench4_shard.log 2>&1
timeout 1200 python bench.py --config 5 --steps 5 > $OUT/bench5.log 2>&1
timeout 600 python bench.py --impl reference --steps 3 > $OUT/bench4_ref.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches4.csv \
    python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e --no-full > $OUT/launches_bench.log 2>&1
python scripts/launches.py $OUT/launches4.csv 4 60 > $OUT/launches4.txt 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches_shard.csv \
    python bench.py --traced 0 --steps 1 --warmup 3 --no-cpu-baseline --no-e2e --no-full > $OUT/launches_shard.log 2>&1
python scripts/launches.py $OUT/launches_shard.csv 4 60 > $OUT/launches_shard.txt 2>&1
timeout 600 bash scripts/ncu_kernel.sh $OUT/prof_events4 k_events_l 4
timeout 600 bash scripts/ncu_kernel.sh $OUT/prof_counters4 k_counters_tiled 4
timeout 900 bash scripts/ncu_kernel.sh $OUT/prof_tables4 "k_sum_rows_chunked|k_sum_rows_cols|k_points_iter|k_rx_onesweep|k_lean_chain|k_validate_events|k_meta_apply|k_keytab_blk|k_tile_heads" 4 27 9
timeout 900 bash scripts/ncu_kernel.sh $OUT/prof_events5 k_events_l 5
for f in prof_events4 prof_counters4 prof_tables4 prof_events5; do
  python scripts/ncu_summary.py $OUT/$f.ncu-rep > $OUT/$f.summary.txt 2>&1
  python scripts/src_lines.py $OUT/$f.ncu-rep 30 > $OUT/$f.lines.txt 2>&1
done
ls -la $OUT
