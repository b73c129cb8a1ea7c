#!/bin/bash
# End-of-round evidence in one call: full GPU test suite, both bench arms at the default workload, every other workload,
# the 128-environment batch, launch list, and dominant-kernel DRAM traffic per workload.   tools/gpu_final.sh <tag>
TAG=${1:-z}; OUT=gpurun_out/$TAG; mkdir -p $OUT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > $OUT/gpu.txt 2>&1
echo "== pytest -m gpu"; timeout 1500 python -m pytest tests -m gpu -x -q 2>&1 | tail -6 | tee $OUT/pytest_gpu.txt
echo "== bench ours (default)"; timeout 900 python bench.py 2> $OUT/bench_err.txt | tee $OUT/bench.json | cut -c1-300
echo "== bench reference"; timeout 900 python bench.py --impl reference --steps 3 --warmup 1 2>&1 | tee $OUT/bench_reference.json | cut -c1-200
: > $OUT/workloads.jsonl
for wl in cfg1 cfg2 cfg3 cfg4 cfg5env; do
  timeout 900 python bench.py --workload $wl --steps 100 --warmup 5 --no-cpu-baseline 2>/dev/null >> $OUT/workloads.jsonl
done
timeout 1200 python bench.py --workload cfg5env --envs-per-gpu 128 --lanes 4 --steps 10 --warmup 3 --no-cpu-baseline 2>/dev/null >> $OUT/workloads.jsonl
python - <<PY
import json
for line in open("$OUT/workloads.jsonl"):
    d = json.loads(line)
    print(d["config"]["workload"][:11], "envs", d["config"]["environments"], "ms", round(d["ms_per_step"], 4), "e2e", round(d["e2e"]["ms_per_step"], 4),
          "Gcells/s", round(d["value"] / 1e9, 2), "cold", round(d["cold_frame_ms"]["value"], 3), "frac", round(d["roofline"]["frac"], 3), d["roofline"]["kernel"])
PY
echo "== ncu launch list"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $OUT/launches.csv \
    python bench.py --steps 2 --warmup 3 --no-cpu-baseline > $OUT/ncu_bench.log 2>&1
python tools/summarize_launches.py $OUT/launches.csv | tee $OUT/launches_summary.txt
echo "== dram traffic of the sweeps per workload"
for wl in cfg1 cfg2 cfg3 cfg4 cfg5env; do
  timeout 600 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none -k regex:k_sweep -s 4 -c 2 --csv \
      --log-file $OUT/traffic_$wl.csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline --workload $wl > /dev/null 2>&1
done
ls $OUT
