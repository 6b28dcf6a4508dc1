#!/bin/bash
# quick iteration: parity (non-slow gpu tests), bench line (config 4), shard bench, tables stage ticks
OUT=${1:-gpurun_out/tq}
mkdir -p $OUT
timeout 300 python -m pytest tests -m "gpu and not slow" -q -x -k "not sanitizer" > $OUT/tests.log 2>&1; echo rc=$? >> $OUT/tests.log
timeout 300 python bench.py --no-cpu-baseline --no-e2e --no-full > $OUT/bench.log 2>&1
timeout 300 python bench.py --traced 0 --no-cpu-baseline --no-e2e --no-full > $OUT/bench_shard.log 2>&1
CHOPPER_DBG_TICKS=1 timeout 300 python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e --no-full > $OUT/b_ticks.log 2> $OUT/ticks.txt
CHOPPER_DBG_TICKS=1 timeout 300 python bench.py --traced 0 --steps 2 --warmup 3 --no-cpu-baseline --no-e2e --no-full > $OUT/b_ticks_shard.log 2> $OUT/ticks_shard.txt
timeout 300 python scripts/step_gaps.py 4 shard > $OUT/gaps_shard.txt 2>&1
