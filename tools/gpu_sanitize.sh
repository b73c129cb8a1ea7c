#!/bin/bash
# compute-sanitizer memcheck + racecheck over the small GPU parity tests that reach the round-2 kernels
# (x sweep with the table bit in the candidate + bulk-copy tile fill, sorted-tile allocation ranks, batched stamps, environment batch).
OUT=gpurun_out/${1:-san}; mkdir -p $OUT
SEL='scene_pipeline_against_oracle or propagate_matches_reference_vectors or graph_replay_equals_eager or dynamic_scene_lifecycle'
{
  echo "== memcheck: tests/test_gpu_parity.py -k '$SEL'"
  timeout 1500 compute-sanitizer --tool memcheck --error-exitcode 9 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "$SEL" 2>&1 | tail -6; echo "memcheck rc=$?"
  echo "== memcheck: sorted-tile ranks forced (KS_RANK_DIRECT=64), tests/test_gpu_large_alloc.py -k '0.05 or 0.118 or recycling'"
  KS_RANK_DIRECT=64 timeout 1500 compute-sanitizer --tool memcheck --error-exitcode 9 python -m pytest tests/test_gpu_large_alloc.py -m gpu -q -x -k "0.05 or 0.118 or recycling" 2>&1 | tail -6
  echo "== memcheck: environment batch, small worlds"
  timeout 1500 compute-sanitizer --tool memcheck --error-exitcode 9 python -m pytest tests/test_gpu_env_batch.py -m gpu -q -x -k "small_environments or failing_environment" 2>&1 | tail -6
  echo "== racecheck: tests/test_gpu_parity.py -k 'scene_pipeline_against_oracle'"
  timeout 1500 compute-sanitizer --tool racecheck --error-exitcode 9 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "scene_pipeline_against_oracle" 2>&1 | tail -6
  echo "== racecheck: sorted-tile ranks forced, one sphere"
  KS_RANK_DIRECT=64 timeout 1500 compute-sanitizer --tool racecheck --error-exitcode 9 python -m pytest tests/test_gpu_large_alloc.py -m gpu -q -x -k "0.118" 2>&1 | tail -6
  echo "== synccheck: tests/test_gpu_parity.py -k 'scene_pipeline_against_oracle'"
  timeout 1500 compute-sanitizer --tool synccheck --error-exitcode 9 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "scene_pipeline_against_oracle" 2>&1 | tail -6
} > $OUT/sanitizer.txt 2>&1
cat $OUT/sanitizer.txt
