#!/bin/bash
# ncu --set full of several kernels, one short bench run each: tools/ncu_many.sh <tag> <workload> k1 k2 ...
TAG=$1; WL=$2; shift 2
OUT=gpurun_out/$TAG
mkdir -p $OUT
for K in "$@"; do
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:$K -s 2 -c 1 -f -o $OUT/prof_${WL}_$K \
      python bench.py --steps 1 --warmup 3 --no-cpu-baseline --workload $WL > $OUT/ncu_${WL}_$K.log 2>&1
done
ls -la $OUT
