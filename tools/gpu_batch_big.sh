#!/bin/bash
# cfg5env lines at large batch sizes: tools/gpu_batch_big.sh <tag> "<envs list>" "<lanes list>" [steps]
TAG=$1; OUT=gpurun_out/$TAG; mkdir -p $OUT
for l in $3; do for n in $2; do
  t0=$(date +%s)
  timeout 1200 python bench.py --workload cfg5env --envs-per-gpu $n --lanes $l --steps ${4:-10} --warmup 3 --no-cpu-baseline 2>$OUT/err_${n}_$l.txt > $OUT/bench_${n}_$l.json
  t1=$(date +%s)
  python -c "
import json
d=json.loads(open('$OUT/bench_${n}_$l.json').read()); print('envs $n lanes $l', 'ms/step', round(d['ms_per_step'],4), 'per env', round(d['ms_per_step']/$n,4), 'e2e', round(d['e2e']['ms_per_step'],4), 'Gcells/s', round(d['value']/1e9,2), d['graph'], 'wall s', $t1-$t0)"
  tail -3 $OUT/err_${n}_$l.txt
done; done
