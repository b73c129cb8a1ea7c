#!/bin/bash
# bench cfg2 stage times under several settings of one environment variable: tools/gpu_env_sweep.sh VAR v1 v2 ...
VAR=$1; shift
for v in "$@"; do
  env $VAR=$v timeout 300 python bench.py --steps 100 --warmup 5 --no-cpu-baseline --workload ${WL:-cfg2} 2>/dev/null | python -c "
import json,sys
d=json.loads(sys.stdin.read()); print('$VAR=$v', 'ms/step', round(d['ms_per_step'],4), 'y', d['stage_ms']['sweep_y'], 'x', d['stage_ms']['sweep_x'])"
done
