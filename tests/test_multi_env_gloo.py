"""The N > 1 host logic (environment partitioning + summary all-gather) on CPU with gloo, world_size 2."""
import os

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2603_05493_b200 import multi_env


def test_partition_is_contiguous_and_complete():
    for n_envs in (0, 1, 7, 128, 129):
        for world in (1, 2, 3, 8):
            ranges = [multi_env.partition_envs(n_envs, world, r) for r in range(world)]
            assert ranges[0][0] == 0 and ranges[-1][1] == n_envs
            assert all(a[1] == b[0] for a, b in zip(ranges, ranges[1:]))
            sizes = [hi - lo for lo, hi in ranges]
            assert max(sizes) - min(sizes) <= 1
            for env in range(n_envs):
                lo, hi = ranges[multi_env.owner_of(env, n_envs, world)]
                assert lo <= env < hi
    with pytest.raises(ValueError):
        multi_env.partition_envs(4, 2, 2)


def _worker(rank, world, port, n_envs, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    lo, hi = multi_env.partition_envs(n_envs, world, rank)
    local, gathered, valid = multi_env.summary_buffers(n_envs, world, rank, "cpu")
    for i, env in enumerate(range(lo, hi)):
        local[i] = torch.tensor([env, 0.01 * env - 0.02, env % 3, 1000 + env], dtype=torch.float64)
    multi_env.gather_summaries(local, gathered, world)
    rows = gathered[valid]
    ok = rows.shape[0] == n_envs and torch.equal(rows[:, 0], torch.arange(n_envs, dtype=torch.float64)) and \
        torch.equal(rows[:, 3], 1000 + torch.arange(n_envs, dtype=torch.float64))
    out[rank] = bool(ok)
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("n_envs", [5, 8])
def test_summary_all_gather_world2(n_envs):
    ctx = mp.get_context("spawn")
    with ctx.Manager() as mgr:
        out = mgr.dict()
        port = 29500 + (os.getpid() + n_envs) % 2000
        procs = [ctx.Process(target=_worker, args=(r, 2, port, n_envs, out)) for r in range(2)]
        for p in procs:
            p.start()
        for p in procs:
            p.join(120)
            assert p.exitcode == 0
        assert dict(out) == {0: True, 1: True}
