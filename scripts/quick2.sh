#!/bin/bash
# parity (all non-slow gpu tests) + bench line + launch list: scripts/quick2.sh OUT
OUT=${1:-gpurun_out/q}
mkdir -p $OUT
timeout 1200 python -m pytest tests -m "gpu and not slow" -q -x -k "not sanitizer" > $OUT/tests.log 2>&1; echo rc=$? >> $OUT/tests.log
timeout 600 python bench.py --no-cpu-baseline --no-e2e --no-full > $OUT/bench.log 2>&1
bash scripts/launches_only.sh $OUT
timeout 300 python bench.py --traced 0 --no-cpu-baseline --no-e2e --no-full > $OUT/bench_shard.log 2>&1
CHOPPER_DBG_TICKS=1 timeout 300 python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e --no-full > $OUT/b_ticks.log 2> $OUT/ticks.txt
