"""bench.py's N > 1 control flow (rank-local environments, summary all-gather, max-over-ranks timing, rank-0
JSON line) on a one-GPU box: two ranks share device 0 and the collective runs on gloo."""
import json
import os
import subprocess
import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parent.parent


@pytest.mark.gpu
def test_two_ranks_share_one_gpu(tmp_path):
    env = dict(os.environ, KS_BENCH_SHARE_GPU="1")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2", "--master-addr", "127.0.0.1",
           "--master-port", "29731", str(ROOT / "bench.py"), "--gpus", "2", "--steps", "5", "--warmup", "3", "--workload", "cfg1",
           "--no-cpu-baseline"]
    out = subprocess.run(cmd, env=env, capture_output=True, text=True, timeout=600, cwd=str(ROOT))
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [ln for ln in out.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, out.stdout
    rec = json.loads(lines[0])
    assert rec["n_gpus"] == 2 and rec["scaling"] == "weak" and rec["config"]["environments"] == 2
    assert rec["value"] > 0 and rec["e2e"]["value"] > 0 and rec["gpu_launches"] > 0
    assert "ncclAllGather" in rec["run"]["collective"]


def test_reference_arm_only_rank0_prints(tmp_path):
    env = dict(os.environ, RANK="1", WORLD_SIZE="2")
    out = subprocess.run([sys.executable, str(ROOT / "bench.py"), "--impl", "reference", "--gpus", "2", "--steps", "1", "--warmup", "0",
                          "--workload", "cfg1"], env=env, capture_output=True, text=True, timeout=300, cwd=str(ROOT))
    assert out.returncode == 0 and out.stdout.strip() == ""
    env["RANK"] = "0"
    out = subprocess.run([sys.executable, str(ROOT / "bench.py"), "--impl", "reference", "--gpus", "2", "--steps", "1", "--warmup", "0",
                          "--workload", "cfg1"], env=env, capture_output=True, text=True, timeout=300, cwd=str(ROOT))
    rec = json.loads(out.stdout.strip().splitlines()[-1])
    assert rec["impl"] == "reference" and rec["cpu_baseline"]["cores"] == 1 and rec["e2e"]["h2d_bytes_per_step"] == 0
