#!/bin/bash
# like gpu_env_sweep.sh with several workloads: WLS="cfg2 cfg5env" tools/gpu_env_sweep2.sh VAR v1 v2 ...
VAR=$1; shift
for wl in ${WLS:-cfg2}; do for v in "$@"; do
  env $VAR=$v timeout 300 python bench.py --steps 60 --warmup 5 --no-cpu-baseline --workload $wl 2>/dev/null | python -c "
import json,sys
d=json.loads(sys.stdin.read()); print('$wl $VAR=$v', 'ms/step', round(d['ms_per_step'],4), 'y', d['stage_ms']['sweep_y'], 'x', d['stage_ms']['sweep_x'])"
done; done
