#!/bin/bash
# Quick loop on the GPU box: the parity tests that cover the ESDF kernels + a short bench (no CPU baseline).
# Usage: tools/gpu_quick.sh [tag] [extra pytest args]
TAG=${1:-q}
mkdir -p gpurun_out/$TAG
timeout 300 python -m pytest tests/test_gpu_parity.py -m gpu -x -q --timeout 120 2>&1 | tail -4 | tee gpurun_out/$TAG/pytest.txt
for wl in ${WORKLOADS:-cfg2}; do
  timeout 600 python bench.py --steps 100 --warmup 5 --no-cpu-baseline --workload $wl 2>gpurun_out/$TAG/err_$wl.txt | tee gpurun_out/$TAG/bench_$wl.json | python -c "
import json,sys
d=json.loads(sys.stdin.read()); print('$wl', 'ms/step', round(d['ms_per_step'],4), 'e2e', round(d['e2e']['ms_per_step'],4), d['stage_ms'])"
done
