#!/bin/bash
# sweep the band-size knobs of the EDT sweeps (tuning aid; results land in gpurun_out/tune_bands.txt)
mkdir -p gpurun_out
for cfg in "24 16" "16 16" "13 32" "17 24" "32 12" "50 8" "100 4"; do
  set -- $cfg
  echo "== target=$1 max_warps=$2"
  KS_BAND_TARGET=$1 KS_MAX_WARPS=$2 python bench.py --steps 30 --warmup 3 --no-cpu-baseline 2>/dev/null | python -c "
import json,sys
d=json.loads(sys.stdin.read())
print('ms %.4f' % d['ms_per_step'], {k: round(v,4) for k,v in d['stage_ms'].items() if k.startswith('sweep')})"
done | tee gpurun_out/tune_bands.txt
