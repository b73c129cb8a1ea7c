#!/bin/bash
for v in 0 1; do
  if [ $v = 1 ]; then export KS_EXPERIMENT_NO_SIGNS=1; fi
  python bench.py --steps 30 --warmup 3 --no-cpu-baseline 2>/dev/null | python -c "
import json,sys
d=json.loads(sys.stdin.read())
print('no_signs=$v ms %.4f' % d['ms_per_step'], {k: round(v,4) for k,v in d['stage_ms'].items() if k.startswith('sweep')})"
done
