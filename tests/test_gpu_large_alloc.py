"""Allocation of many new blocks in ONE call (a cold start): above 512 new keys the allocation kernel ranks them through
sorted tiles of 1024 instead of direct counting (csrc/tsdf.cu "ranks of the new keys").  The world must still be the
reference's: key -> pool assignment, hash slot order and free list identical to allocate_keys' sorted sequential
insertion (sdf_world.hpp:307-323), for single stamps, batches (rank = first primitive, then key) and depth frames,
with tombstones and a free list left behind by recycle_blocks."""
import numpy as np
import pytest

from paper_2603_05493_b200 import api
from parity_util import assert_world_parity

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _built():
    from paper_2603_05493_b200 import build
    build.build()
    assert api.load_library().ks_device_count() > 0, "GPU tests need a CUDA device"


@pytest.fixture(params=["default", "sorted tiles from 64 new keys"])
def rank_mode(request, monkeypatch):
    """KS_RANK_DIRECT is read when a world is created: 64 forces the sorted-tile ranks for everything these tests allocate."""
    if request.param != "default":
        monkeypatch.setenv("KS_RANK_DIRECT", "64")
    return request.param


def _worlds(oracle_lib, voxel, capacity, **kw):
    cfg = api.make_tsdf_config(voxel)
    cfg.capacity = capacity
    for k, v in kw.items():
        setattr(cfg, k, v)
    return api.make_tsdf(cfg), oracle_lib.make_tsdf(voxel, capacity=capacity, **kw)


@pytest.mark.parametrize("radius", [0.05, 0.118, 0.12, 0.2, 0.33, 0.5])
def test_one_sphere_many_new_blocks(oracle_lib, radius, rank_mode):
    """A sphere shell at 5 mm voxels: from ~200 to ~20 000 new blocks in one stamp (tile counts 0, 1, 2, ... 20)."""
    gpu, cpu = _worlds(oracle_lib, 0.005, 32768)
    api.stamp_primitive(gpu, api.SphereShape((0.013, -0.021, 0.4), radius))
    cpu.stamp_sphere((0.013, -0.021, 0.4), radius)
    n = cpu.allocated_block_count()
    assert api.allocated_block_count(gpu) == n and n > 50
    assert assert_world_parity(gpu, cpu)


def test_batch_of_large_primitives_after_recycling(oracle_lib, rank_mode):
    """Frame -> decay -> recycle (free list + tombstones), then a batch of four overlapping primitives that allocates
    several thousand blocks at once: pool indices come from the free list (LIFO) first, then fresh ones; ranks are
    (first primitive, key)."""
    from paper_2603_05493_b200 import scenes
    sc = scenes.config2()
    gpu, cpu = _worlds(oracle_lib, sc.tsdf_voxel, 16384, weight_threshold=1.2, alpha_time=0.5)
    f = sc.frames[0]
    from parity_util import frame_of
    assert api.integrate_depth(gpu, frame_of(f)) == cpu.integrate_depth(f.depth, f.width, f.height, f.intr, f.R, f.t)
    moved = np.array(f.t) + np.array([0.4, 0.0, 0.0])  # a second view: blocks only the first one saw decay below the threshold
    view = api.DepthFrame(f.width, f.height, f.intr[0], f.intr[1], f.intr[2], f.intr[3], f.R, moved, f.depth)
    for _ in range(2):
        api.decay_weights(gpu, view)
        cpu.decay_weights(f.width, f.height, f.intr, f.R, moved)
    r0 = cpu.recycle_blocks()
    assert api.recycle_blocks(gpu) == r0 and r0 > 50
    assert np.array_equal(gpu.free_list(), cpu.free_list())
    prims = [api.Cuboid(np.eye(3), (0.9, 0.5, 0.5), (0.3, 0.25, 0.2)), api.SphereShape((0.6, 0.4, 0.45), 0.27),
             api.Cuboid(np.eye(3), (1.3, 0.6, 0.3), (0.2, 0.2, 0.25)), api.SphereShape((1.5, 0.3, 0.6), 0.15)]
    api.stamp_primitives(gpu, prims)
    for p in prims:
        if isinstance(p, api.Cuboid):
            cpu.stamp_cuboid(p.pose_R, p.pose_t, p.half_extents)
        else:
            cpu.stamp_sphere(p.center, p.radius)
    assert cpu.allocated_block_count() > 4000
    assert assert_world_parity(gpu, cpu)
    assert np.array_equal(gpu.free_list(), cpu.free_list())
