#!/bin/bash
# A/B of the counter-pass slot grouping and the sub-run -> instance fold (config 4 and the traced-GPU-0 shard)
OUT=${1:-gpurun_out/ab2}
mkdir -p $OUT
timeout 300 python -m pytest tests -m "gpu and not slow" -q -x -k "not sanitizer" > $OUT/tests.log 2>&1; echo rc=$? >> $OUT/tests.log
for v in default sg2 staged; do
  case $v in default) E="";; sg2) E="CHOPPER_COUNTER_SG=2";; staged) E="CHOPPER_SUBRUN_SUM=staged";; esac
  env $E timeout 300 python bench.py --no-cpu-baseline --no-e2e --no-full > $OUT/bench_$v.log 2>&1
  env $E CHOPPER_DBG_TICKS=1 timeout 300 python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e --no-full > /dev/null 2> $OUT/ticks_$v.txt
done
timeout 300 python bench.py --traced 0 --no-cpu-baseline --no-e2e --no-full > $OUT/bench_shard.log 2>&1
