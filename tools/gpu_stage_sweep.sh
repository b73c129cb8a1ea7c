#!/bin/bash
# all stage times under settings of one environment variable: WLS="cfg2" tools/gpu_stage_sweep.sh VAR v1 v2 ...
VAR=$1; shift
for wl in ${WLS:-cfg2}; do for v in "$@"; do
  env $VAR=$v timeout 300 python bench.py --steps 60 --warmup 5 --no-cpu-baseline --workload $wl 2>/dev/null | python -c "
import json,sys
d=json.loads(sys.stdin.read()); print('$wl $VAR=$v', 'ms/step', round(d['ms_per_step'],4), 'e2e', round(d['e2e']['ms_per_step'],4), {k: round(1e3*v,1) for k,v in d['stage_ms'].items()})"
done; done
