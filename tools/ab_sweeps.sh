#!/bin/bash
# A/B on the GPU box: sweep variants and knobs.  Usage: tools/ab_sweeps.sh <tag> "ENV1=a ENV2=b" "ENV1=c" ...
OUT=gpurun_out/${1:-ab}; shift
mkdir -p $OUT
echo "== pytest -m gpu (default sweeps)"; timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -5 | tee $OUT/pytest_gpu.txt
run() { echo "== $*"; env $* timeout 600 python bench.py --steps 100 --warmup 5 --no-cpu-baseline 2>/dev/null | python -c "
import json,sys
d=json.loads(sys.stdin.read()); print(round(d['ms_per_step'],4), {k:round(v,4) for k,v in d['stage_ms'].items()})"; }
run X=1
for cfg in "$@"; do run $cfg; done
