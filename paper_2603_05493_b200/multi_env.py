"""Independent environments across GPUs.

A single scene does not shard (each EDT pass is global along its axis), so the multi-GPU axis is the
environment: every rank owns a contiguous range of environments with their own TSDF/ESDF handles and
runs them through the same kernels with no data-path collective.  The only exchange is one all-gather
of a fixed-size per-environment collision summary per update (NCCL over NVLink/NVSwitch on the GPU box;
the same code runs on gloo in the CPU tests).
"""
from __future__ import annotations

from typing import List, Tuple

import torch
import torch.distributed as dist

SUMMARY_FIELDS = ("env", "min_distance", "colliding", "seeds")  # 4 x float64 = 32 bytes per environment


def partition_envs(n_envs: int, world: int, rank: int) -> Tuple[int, int]:
    """Contiguous range [lo, hi) of environments owned by `rank`; earlier ranks take the remainder."""
    from . import api
    return api.partition_envs(n_envs, world, rank)  # ks_partition_envs: the C ABI owns the rule (host code, no device needed)


def owner_of(env: int, n_envs: int, world: int) -> int:
    for rank in range(world):
        lo, hi = partition_envs(n_envs, world, rank)
        if lo <= env < hi:
            return rank
    raise ValueError("environment out of range")


def summary_buffers(n_envs: int, world: int, rank: int, device) -> Tuple[torch.Tensor, torch.Tensor, List[int]]:
    """(local [max_local, 4], gathered [world * max_local, 4], rows of `gathered` that are real environments)."""
    per_rank = [partition_envs(n_envs, world, r) for r in range(world)]
    max_local = max(hi - lo for lo, hi in per_rank)
    local = torch.full((max_local, len(SUMMARY_FIELDS)), float("nan"), dtype=torch.float64, device=device)
    gathered = torch.empty((world * max_local, len(SUMMARY_FIELDS)), dtype=torch.float64, device=device)
    valid = [r * max_local + i for r, (lo, hi) in enumerate(per_rank) for i in range(hi - lo)]
    return local, gathered, valid


def gather_summaries(local: torch.Tensor, gathered: torch.Tensor, world: int) -> torch.Tensor:
    """All-gather the per-environment summaries; a no-op copy on one rank."""
    if world == 1:
        gathered.copy_(local)
    else:
        dist.all_gather_into_tensor(gathered, local)
    return gathered
