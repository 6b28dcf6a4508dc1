#!/bin/bash
# A/B of an environment switch on the config-4 bench: scripts/ab.sh OUT VAR "v1 v2 ..." [extra bench args]
OUT=$1; VAR=$2; VALS=$3; shift 3
mkdir -p $OUT
for v in $VALS; do
  env $VAR=$v timeout 600 python bench.py --no-cpu-baseline --no-e2e --no-full "$@" > $OUT/bench_$v.log 2>&1
  python -c "
import json,sys; d=json.loads(open('$OUT/bench_$v.log').read().strip().splitlines()[-1]); r=d['roofline']
print('$VAR=$v', 'ms/step', round(d['ms_per_step'],3), 'ev', round(r['avg_launch_ms'],4), 'frac', round(r['frac'],3), 'evpass', round(r['event_pass_phase_ms'],3))" >> $OUT/ab.txt 2>&1
done
