#!/bin/bash
# quick GPU iteration: parity tests, one bench line, one ncu --set full capture of the event pass
OUT=${1:-gpurun_out}
mkdir -p $OUT
timeout 600 python -m pytest tests -m gpu -x -q > $OUT/gpu_tests.log 2>&1; echo "tests rc=$?" >> $OUT/gpu_tests.log
timeout 300 python bench.py --no-cpu-baseline > $OUT/bench.log 2>&1; echo "bench rc=$?" >> $OUT/bench.log
ncu --set full --clock-control none --import-source on -k regex:${KREGEX:-k_events} -s ${KSKIP:-3} -c ${KCOUNT:-1} -f -o $OUT/prof_events \
    python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > $OUT/prof_events.log 2>&1
