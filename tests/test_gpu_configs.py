"""Full-size parity for the BASELINE.json configurations the round-1 suite did not reach, and the two
randomised parity runs as collected tests.

  configs[2]  500^3 cells @ 2 mm, four cameras (four staging slots) + two cuboids: the only configuration
              that runs the 32-warp x-sweep tiles, four y rows per lane and ~2.8 M seeds on a real TSDF.
  configs[4]  independent 300 x 200 x 200 environments: two of them alone, and several enqueued into ONE
              captured graph, each compared with its own oracle world.
  fuzz        tests/fuzz_parity.py and tests/fuzz_lifecycle.py, a bounded seeded run of each.

Reference: integrate_depth sdf_world.hpp:340-389, stamp_primitive :394-444, build_esdf esdf.hpp:323-327.
"""
import ctypes as C
import time

import numpy as np
import pytest

from paper_2603_05493_b200 import api, scenes
from parity_util import assert_world_parity, cpu_world, esdf_config, frame_of, gpu_world, same_bits

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _built():
    from paper_2603_05493_b200 import build
    build.build()
    assert api.load_library().ks_device_count() > 0, "GPU tests need a CUDA device"


def _d2_matches_sites(d2, site, dims, slab=16):
    """d2 == |cell - site|^2 for every cell, checked z-slab by z-slab (a 500^3 grid must not need 12 GB of int64)."""
    nx, ny, nz = dims
    d2 = d2.reshape(nz, ny, nx)
    site = site.reshape(nz, ny, nx, 3)
    xs = np.arange(nx, dtype=np.int32)[None, None, :]
    ys = np.arange(ny, dtype=np.int32)[None, :, None]
    for z0 in range(0, nz, slab):
        s = site[z0:z0 + slab]
        zs = np.arange(z0, min(nz, z0 + slab), dtype=np.int32)[:, None, None]
        want = (xs - s[..., 0]) ** 2 + (ys - s[..., 1]) ** 2 + (zs - s[..., 2]) ** 2
        if not np.array_equal(d2[z0:z0 + slab], want):
            return False
    return True


def _compare_esdf(oracle_lib, scene, e, cpu, n_queries=200_000, seed=7):
    site, dist, d2 = e.download()
    mask0, has0, site0, dist0 = cpu.build_esdf(scene.esdf_origin, scene.esdf_dims, scene.esdf_voxel)
    assert e.has_sites == has0
    assert int(e.report().seed_count) == int(mask0.sum())
    assert np.array_equal(site, site0), "nearest sites differ"
    assert _d2_matches_sites(d2, site0, scene.esdf_dims), "squared distances differ"
    assert np.array_equal(dist, dist0) and np.array_equal(np.signbit(dist), np.signbit(dist0)), "signed distances differ"
    del site, d2, site0, mask0
    rng = np.random.RandomState(seed)
    pts = scene.esdf_origin + (rng.random_sample((n_queries, 3)) * 1.1 - 0.05) * np.array(scene.esdf_dims) * scene.esdf_voxel
    s = api.query(e, pts)
    d0, g0, i0 = oracle_lib.query_esdf(scene.esdf_origin, scene.esdf_dims, scene.esdf_voxel, has0, dist0, pts)
    assert same_bits(s.distance, d0) and same_bits(s.gradient, g0) and np.array_equal(s.inside, i0)


def test_config3_full_size_against_oracle(oracle_lib):
    """BASELINE configs[2] at full size: 4 cameras fused + 2 cuboids into 500^3 cells at 2 mm (oracle ~45 s)."""
    scene = scenes.config3()
    tsdf, touched = gpu_world(scene)
    cpu, touched0 = cpu_world(oracle_lib, scene)
    assert touched == touched0 and len(touched) == 4
    assert api.allocated_block_count(tsdf) == cpu.allocated_block_count()
    assert assert_world_parity(tsdf, cpu), "TSDF channels within 1e-5 but not bit-identical"
    e = api.build_esdf(tsdf, esdf_config(scene))
    _compare_esdf(oracle_lib, scene, e, cpu)
    # the same update as the bench runs it: four staging slots in one captured graph, replayed
    lib = api.load_library()
    stream = C.c_void_p()
    assert lib.ks_stream_create(C.byref(stream)) == 0
    cfg = api.make_tsdf_config(scene.tsdf_voxel)
    cfg.capacity = scene.capacity
    t2 = api.make_tsdf(cfg, stream.value)
    e2 = api.DenseEsdf(esdf_config(scene), stream.value)
    prims = [api.Cuboid(c.R, c.t, c.half_extents) for c in scene.cuboids]

    def enqueue():
        for slot in range(4):
            t2.upload_frame_async(slot)
            t2.integrate_async(slot)
        for p in prims:
            t2.stamp_async(p)
        e2.build_async(t2)

    for slot, f in enumerate(scene.frames):
        t2.stage_frame(frame_of(f), slot)
    enqueue()
    t2.sync()
    g = api.Graph(stream.value)
    with g:
        enqueue()
    g.launch()
    t2.sync()
    for f in scene.frames:  # the oracle world after the second pass over the four cameras
        cpu.integrate_depth(f.depth, f.width, f.height, f.intr, f.R, f.t)
    assert_world_parity(t2, cpu)
    site, dist, _ = e2.download(d2=False)
    _, _, site0, dist0 = cpu.build_esdf(scene.esdf_origin, scene.esdf_dims, scene.esdf_voxel)
    assert np.array_equal(site, site0) and np.array_equal(dist, dist0)
    g.close()


@pytest.mark.parametrize("env", [0, 77])
def test_config5_environment_against_oracle(oracle_lib, env):
    """One environment of BASELINE configs[4] (300 x 200 x 200 @ 5 mm, jittered cuboids) at full size."""
    scene = scenes.config5_env(env)
    tsdf, touched = gpu_world(scene)
    cpu, touched0 = cpu_world(oracle_lib, scene)
    assert touched == touched0
    assert assert_world_parity(tsdf, cpu)
    e = api.build_esdf(tsdf, esdf_config(scene))
    _compare_esdf(oracle_lib, scene, e, cpu, n_queries=50_000, seed=env)


def test_config5_three_environments_in_one_graph(oracle_lib):
    """Three configs[4] environments on one stream, their updates captured into ONE graph and replayed twice;
    every environment must equal its own oracle world (no cross-talk through shared scratch or the directory)."""
    lib = api.load_library()
    stream = C.c_void_p()
    assert lib.ks_stream_create(C.byref(stream)) == 0
    ids = [3, 64, 127]
    worlds = []
    for env in ids:
        sc = scenes.config5_env(env)
        cfg = api.make_tsdf_config(sc.tsdf_voxel)
        cfg.capacity = sc.capacity
        t = api.make_tsdf(cfg, stream.value)
        e = api.DenseEsdf(esdf_config(sc), stream.value)
        t.stage_frame(frame_of(sc.frames[0]))
        worlds.append((sc, t, e, [api.Cuboid(c.R, c.t, c.half_extents) for c in sc.cuboids]))

    def enqueue():
        for _, t, e, prims in worlds:
            t.upload_frame_async()
            t.integrate_async()
            for p in prims:
                t.stamp_async(p)
            e.build_async(t)

    enqueue()
    for _, t, _, _ in worlds:
        t.sync()
    g = api.Graph(stream.value)
    with g:
        enqueue()
    for _ in range(2):
        g.launch()
    for sc, t, e, _ in worlds:
        t.sync()
        cpu = oracle_lib.make_tsdf(sc.tsdf_voxel, capacity=sc.capacity)
        f = sc.frames[0]
        for _ in range(3):  # eager warm-up + two replays
            cpu.integrate_depth(f.depth, f.width, f.height, f.intr, f.R, f.t)
        for c in sc.cuboids:
            cpu.stamp_cuboid(c.R, c.t, c.half_extents)
        assert_world_parity(t, cpu)
        _compare_esdf(oracle_lib, sc, e, cpu, n_queries=20_000)
    g.close()


def _run_for(seconds, one, *args):
    t0, n = time.time(), 0
    while time.time() - t0 < seconds or n < 3:
        one(*args)
        n += 1
    return n


def test_fuzz_parity_bounded(oracle_lib):
    """tests/fuzz_parity.py for ~40 s: random grid shapes, voxel ratios, origins, primitives and meshes."""
    import fuzz_parity
    rng = np.random.RandomState(20261017)
    counter = iter(range(10**9))
    n = _run_for(40.0, lambda: fuzz_parity.one_case(oracle_lib, rng, next(counter), meshes=True))
    assert n >= 3


def test_fuzz_lifecycle_bounded(oracle_lib):
    """tests/fuzz_lifecycle.py for ~30 s: integrate / stamp / decay / recycle with small pools, exhaustion included."""
    import fuzz_lifecycle
    rng = np.random.RandomState(20261018)
    n = _run_for(30.0, fuzz_lifecycle.one_world, oracle_lib, rng)
    assert n >= 3
