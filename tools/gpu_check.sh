#!/bin/bash
# Run on the GPU box via gpurun: GPU tests, bench (both arms), ncu launch list and one full capture.
# Usage: tools/gpu_check.sh [tag] [kernel-regex-for-full-capture]
TAG=${1:-r1}
KREGEX=${2:-k_sweep_x_dc}
OUT=gpurun_out/$TAG
mkdir -p $OUT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > $OUT/gpu.txt 2>&1
echo "== pytest -m gpu"; timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -15 | tee $OUT/pytest_gpu.txt
echo "== bench ours"; timeout 900 python bench.py --steps 200 --warmup 5 2> $OUT/bench_err.txt | tee $OUT/bench.json
tail -5 $OUT/bench_err.txt
if [ "$SKIP_REF" != "1" ]; then
  echo "== bench reference"; timeout 900 python bench.py --impl reference --steps 3 --warmup 1 2>&1 | tee $OUT/bench_reference.json
fi
if [ "$SKIP_NCU" != "1" ]; then
  echo "== ncu launch list"
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $OUT/launches.csv \
      python bench.py --steps 2 --warmup 3 --no-cpu-baseline > $OUT/ncu_bench.log 2>&1
  python tools/summarize_launches.py $OUT/launches.csv | tee $OUT/launches_summary.txt
  echo "== ncu full: $KREGEX"
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:$KREGEX -s 2 -c 2 -f -o $OUT/prof_$KREGEX \
      python bench.py --steps 1 --warmup 3 --no-cpu-baseline > $OUT/ncu_full.log 2>&1
  ls -la $OUT
fi
