#!/bin/bash
# ncu --set full of one kernel of the timed bench step: scripts/ncu_kernel.sh OUT REGEX [CONFIG] [SKIP] [COUNT]
OUT=$1; RX=$2; CFG=${3:-4}; SKIP=${4:-3}; CNT=${5:-1}
mkdir -p $(dirname $OUT)
ncu --set full --clock-control none --import-source on -k regex:"$RX" -s $SKIP -c $CNT -f -o $OUT \
    python bench.py --config $CFG --steps 1 --warmup 3 --no-cpu-baseline --no-e2e --no-full > $OUT.log 2>&1
