#!/bin/bash
# Environment-batch checks on the GPU box: the batch tests, the two-rank bench test, cfg5env lines at several batch sizes / lane counts.
# Usage: tools/gpu_batch.sh [tag] ["envs list"] ["lanes list"]
TAG=${1:-batch}
OUT=gpurun_out/$TAG
mkdir -p $OUT
timeout 900 python -m pytest tests/test_gpu_env_batch.py tests/test_bench_multirank.py -m gpu -x -q 2>&1 | tail -15 | tee $OUT/pytest.txt
for n in ${2:-4 16}; do
  for l in ${3:-1 2 4}; do
    timeout 900 python bench.py --workload cfg5env --envs-per-gpu $n --lanes $l --steps 20 --warmup 3 --no-cpu-baseline 2>$OUT/err_${n}_$l.txt | tee $OUT/bench_${n}_$l.json | python -c "
import json,sys
d=json.loads(sys.stdin.read()); print('envs $n lanes $l', 'ms/step', round(d['ms_per_step'],4), 'per env', round(d['ms_per_step']/$n,4), 'e2e', round(d['e2e']['ms_per_step'],4), 'Gcells/s', round(d['value']/1e9,2), d['graph'])"
    tail -3 $OUT/err_${n}_$l.txt
  done
done
