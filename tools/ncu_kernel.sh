#!/bin/bash
# ncu --set full of one kernel (regex) inside a short bench run.  Usage: tools/ncu_kernel.sh <tag> <kernel-regex> [env...]
TAG=$1; K=$2; shift 2
OUT=gpurun_out/$TAG
mkdir -p $OUT
env "$@" timeout 900 ncu --set full --clock-control none --import-source on -k regex:$K -s 2 -c 1 -f -o $OUT/prof_$K \
    python bench.py --steps 1 --warmup 3 --no-cpu-baseline > $OUT/ncu_$K.log 2>&1
ls -la $OUT
