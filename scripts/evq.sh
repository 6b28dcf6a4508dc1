#!/bin/bash
# event-pass iteration: parity (non-slow gpu tests), bench line, ncu --set full of the lean pass
OUT=${1:-gpurun_out/evq}
mkdir -p $OUT
timeout 300 python -m pytest tests -m "gpu and not slow" -q -x -k "not sanitizer" > $OUT/tests.log 2>&1; echo rc=$? >> $OUT/tests.log
timeout 300 python bench.py --no-cpu-baseline --no-e2e --no-full > $OUT/bench.log 2>&1
timeout 300 bash scripts/ncu_kernel.sh $OUT/ev "${EVK:-k_events_c}" 4
ncu -i $OUT/ev.ncu-rep --page raw --csv > $OUT/ev.raw.csv 2>/dev/null
