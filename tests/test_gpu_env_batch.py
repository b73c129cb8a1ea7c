"""The C-ABI environment batch (ks_batch_*, include/ks_b200.h) against the oracle, one environment at a time.

BASELINE.json configs[4] = independent environments; the reference has no batch API, so the contract is:
every world of a batch equals what the per-handle calls -- i.e. the reference's integrate_depth (sdf_world.hpp:340-389),
stamp_primitive (:394-444) and build_esdf (esdf.hpp:323-327) -- produce for that environment alone.
"""
import numpy as np
import pytest

from paper_2603_05493_b200 import api, scenes
from parity_util import assert_world_parity, esdf_config, frame_of, same_bits

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _built():
    from paper_2603_05493_b200 import build
    build.build()
    assert api.load_library().ks_device_count() > 0, "GPU tests need a CUDA device"


def _make_batch(ids, lanes, scene_of=scenes.config5_env):
    scs = [scene_of(e) for e in ids]
    cfg = api.make_tsdf_config(scs[0].tsdf_voxel)
    cfg.capacity = scs[0].capacity
    batch = api.EnvBatch(len(ids), cfg, esdf_config(scs[0]), lanes=lanes, first_env=ids[0])
    for i, sc in enumerate(scs):
        for slot, f in enumerate(sc.frames):
            batch.tsdf[i].stage_frame(frame_of(f), slot)
        prims = [api.Cuboid(c.R, c.t, c.half_extents) for c in sc.cuboids] + [api.SphereShape(s.center, s.radius) for s in sc.spheres]
        batch.set_inputs(i, len(sc.frames), prims)
        rng = np.random.RandomState(100 + ids[i])
        probes = sc.esdf_origin + rng.random_sample((512, 3)) * np.array(sc.esdf_dims) * sc.esdf_voxel
        batch.set_probes(i, probes, 0.02)
        sc.probes = probes
    return batch, scs


def _oracle_world(oracle_lib, sc, updates):
    cpu = oracle_lib.make_tsdf(sc.tsdf_voxel, capacity=sc.capacity)
    for _ in range(updates):
        for f in sc.frames:
            cpu.integrate_depth(f.depth, f.width, f.height, f.intr, f.R, f.t)
        for c in sc.cuboids:
            cpu.stamp_cuboid(c.R, c.t, c.half_extents)
        for s in sc.spheres:
            cpu.stamp_sphere(s.center, s.radius)
    return cpu


def _check_env(oracle_lib, sc, tsdf, esdf, summary, env_id, updates):
    cpu = _oracle_world(oracle_lib, sc, updates)
    assert assert_world_parity(tsdf, cpu)
    site, dist, _ = esdf.download(d2=False)
    mask0, has0, site0, dist0 = cpu.build_esdf(sc.esdf_origin, sc.esdf_dims, sc.esdf_voxel)
    assert np.array_equal(site, site0) and same_bits(dist, dist0)
    d0, _, _ = oracle_lib.query_esdf(sc.esdf_origin, sc.esdf_dims, sc.esdf_voxel, has0, dist0, sc.probes)
    assert summary[0] == env_id
    assert summary[1] == d0.min(), "summary: minimum probe distance"
    assert summary[2] == float((d0 < 0.02).sum()), "summary: near-contact count"
    assert summary[3] == float(mask0.sum()), "summary: seed count"


@pytest.mark.parametrize("lanes", [1, 3])
def test_batch_of_small_environments_matches_per_environment_oracle(oracle_lib, lanes):
    """Five small worlds (different surfaces, primitives) through ks_batch_update: plain enqueue, capture, two replays."""
    ids = [10, 11, 12, 13, 14]
    batch, scs = _make_batch(ids, lanes, scene_of=scenes.small_scene)
    assert batch.lanes == min(lanes, len(ids))
    for _ in range(3):  # first call: eager update + capture; then two replays
        batch.update(True)
    assert batch.graph_kernels() > 0
    reps, ereps, summ = batch.sync()
    assert all(r.status == 0 for r in reps) and all(e.has_sites and e.signs_recovered for e in ereps)
    for i, sc in enumerate(scs):
        _check_env(oracle_lib, sc, batch.tsdf[i], batch.esdf[i], summ[i], ids[i], updates=3)
    batch.close()


def test_batch_config5_environments_full_size(oracle_lib):
    """Four configs[4] environments (300 x 200 x 200) on two lanes, async enqueue + caller-side capture + replay."""
    ids = [5, 6, 7, 8]
    batch, scs = _make_batch(ids, lanes=2)
    batch.update_async(True)
    batch.sync()
    g = api.Graph(batch.stream)
    with g:
        batch.update_async(True)
    kernels, nodes = g.node_count()
    assert kernels >= 4 * 10
    g.launch()
    reps, ereps, summ = batch.sync()
    assert all(r.status == 0 for r in reps)
    for i in (0, 3):  # the oracle takes ~10 s per environment: first and last
        _check_env(oracle_lib, scs[i], batch.tsdf[i], batch.esdf[i], summ[i], ids[i], updates=2)
    assert [int(s[0]) for s in summ] == ids
    g.close()
    batch.close()


def test_batch_reports_the_failing_environment(oracle_lib):
    """Pool exhaustion in one environment is reported with its id; the others are untouched by it."""
    scs = [scenes.small_scene(0), scenes.small_scene(1)]
    cfg = api.make_tsdf_config(scs[0].tsdf_voxel)
    cfg.capacity = 8  # far too small for the depth frame
    batch = api.EnvBatch(2, cfg, esdf_config(scs[0]), lanes=2, first_env=40)
    for i, sc in enumerate(scs):
        batch.tsdf[i].stage_frame(frame_of(sc.frames[0]))
        batch.set_inputs(i, 1 if i == 1 else 0, [])
    batch.update_async(True)
    with pytest.raises(api.ValidationError, match=r"environment 41: tsdf: pool exhausted"):
        batch.sync()
    batch.close()


def test_batch_allgather_over_nccl_single_rank():
    """ks_batch_attach_nccl with world = 1: ncclCommInitRank + ncclAllGather run for real (as a node of the batch graph);
    the gathered rows equal the local summaries."""
    try:
        uid = api.nccl_unique_id()
    except api.ValidationError as err:
        pytest.skip(f"NCCL not loadable here: {err}")
    ids = [0, 1, 2]
    batch, scs = _make_batch(ids, lanes=2, scene_of=scenes.small_scene)
    batch.attach_nccl(uid, 1, 0, max_local_envs=4)  # one padding row
    for _ in range(2):
        batch.update(True)
    _, _, summ = batch.sync()
    all_rows = batch.gathered()
    assert all_rows.shape == (4, 4)
    assert same_bits(all_rows[:3], summ) and np.isnan(all_rows[3]).all()
    batch.close()
