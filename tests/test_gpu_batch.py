"""Batched stamps (ks_tsdf_stamp_batch): all primitives of an update in three launches must leave the world exactly
as the reference's sequential stamp_primitive calls do (sdf_world.hpp:394-444) -- pool indices, hash slot order, free
list, voxels -- including the call that runs out of pool entries (its message, and nothing after it applied)."""
import numpy as np
import pytest

from paper_2603_05493_b200 import api, scenes
from parity_util import assert_world_parity, esdf_config, frame_of

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _built():
    from paper_2603_05493_b200 import build
    build.build()
    assert api.load_library().ks_device_count() > 0, "GPU tests need a CUDA device"


def _prims(scene):
    return [api.Cuboid(c.R, c.t, c.half_extents) for c in scene.cuboids] + [api.SphereShape(s.center, s.radius) for s in scene.spheres]


def _cpu_sequential(cpu, prims):
    """The reference's behaviour for `for p in prims: stamp_primitive(world, p)`: returns the exception text, if any."""
    for p in prims:
        try:
            if isinstance(p, api.Cuboid):
                cpu.stamp_cuboid(p.pose_R, p.pose_t, p.half_extents)
            else:
                cpu.stamp_sphere(p.center, p.radius)
        except Exception as err:  # noqa: BLE001
            return str(err)
    return None


def _check_state(tsdf, cpu):
    assert_world_parity(tsdf, cpu, exact_pool=True)
    rep = tsdf.sync()
    assert rep.live_blocks == cpu.allocated_block_count() and rep.next_fresh == cpu.next_fresh()
    assert np.array_equal(tsdf.free_list(), cpu.free_list())


def test_config2_scene_with_batched_stamps(oracle_lib):
    scene = scenes.config2()
    cfg = api.make_tsdf_config(scene.tsdf_voxel)
    cfg.capacity = scene.capacity
    tsdf = api.make_tsdf(cfg)
    cpu = oracle_lib.make_tsdf(scene.tsdf_voxel, capacity=scene.capacity)
    f = scene.frames[0]
    assert api.integrate_depth(tsdf, frame_of(f)) == cpu.integrate_depth(f.depth, f.width, f.height, f.intr, f.R, f.t)
    prims = _prims(scene)
    api.stamp_primitives(tsdf, prims)
    assert _cpu_sequential(cpu, prims) is None
    _check_state(tsdf, cpu)
    api.stamp_primitives(tsdf, prims)  # idempotent, nothing new to allocate (the steady state of a control loop)
    _check_state(tsdf, cpu)
    e = api.build_esdf(tsdf, esdf_config(scene))
    site, dist, _ = e.download(d2=False)
    _, _, site0, dist0 = cpu.build_esdf(scene.esdf_origin, scene.esdf_dims, scene.esdf_voxel)
    assert np.array_equal(site, site0) and np.array_equal(dist, dist0)


@pytest.mark.parametrize("seed", [71, 72, 73])
def test_random_batches_with_overlap_recycling_and_exhaustion(oracle_lib, seed):
    """Random batches of 1-20 overlapping primitives into small pools, with integrates / decays / recycles in between
    (so free-list entries and tombstones exist): after every batch the world equals the sequential reference, and a
    batch that runs out of pool raises the reference's text for the primitive that failed."""
    rng = np.random.RandomState(seed)
    failures = batches = 0
    for world in range(12):
        sc = scenes.small_scene(int(rng.randint(1, 10**6)), dims=(24, 20, 18), n_cuboids=0, n_spheres=0)
        f = sc.frames[0]
        capacity = int(rng.choice([40, 90, 200, 800, 3000]))
        cfg = api.make_tsdf_config(sc.tsdf_voxel)
        cfg.capacity, cfg.weight_threshold, cfg.alpha_time = capacity, 40.0, 0.7
        tsdf = api.make_tsdf(cfg)
        cpu = oracle_lib.make_tsdf(sc.tsdf_voxel, capacity=capacity, weight_threshold=40.0, alpha_time=0.7)
        for step in range(int(rng.randint(3, 8))):
            op = rng.choice(["batch", "batch", "integrate", "decay+recycle"])
            if op == "integrate":
                fr = api.DepthFrame(f.width, f.height, *f.intr, f.R, f.t, f.depth + np.float32(0.05 * rng.randint(0, 4)))
                try:
                    want = cpu.integrate_depth(fr.depth, f.width, f.height, f.intr, f.R, f.t)
                except Exception as err:  # noqa: BLE001
                    with pytest.raises(api.ValidationError) as got:
                        api.integrate_depth(tsdf, fr)
                    assert str(got.value) in str(err)
                else:
                    assert api.integrate_depth(tsdf, fr) == want
            elif op == "decay+recycle":
                fr = api.DepthFrame(f.width, f.height, *f.intr, f.R, f.t, f.depth)
                for _ in range(3):
                    api.decay_weights(tsdf, fr)
                    cpu.decay_weights(f.width, f.height, f.intr, f.R, f.t)
                assert api.recycle_blocks(tsdf) == cpu.recycle_blocks()
            else:
                prims = []
                for _ in range(int(rng.choice([1, 2, 3, 5, 9, 20]))):
                    c = sc.esdf_origin + rng.random_sample(3) * 0.45
                    if rng.random_sample() < 0.5:
                        prims.append(api.SphereShape(c, 0.02 + 0.1 * rng.random_sample()))
                    else:
                        prims.append(api.Cuboid(scenes.rot_z(float(rng.random_sample() * 2.0)), c, 0.02 + 0.1 * rng.random_sample(3)))
                want = _cpu_sequential(cpu, prims)
                batches += 1
                if want is None:
                    api.stamp_primitives(tsdf, prims)
                else:
                    failures += 1
                    with pytest.raises(api.ValidationError) as got:
                        api.stamp_primitives(tsdf, prims)
                    assert str(got.value) in want, (str(got.value), want)
            _check_state(tsdf, cpu)
    assert batches > 10 and failures > 0


def test_batch_inside_a_captured_update(oracle_lib):
    """integrate + ONE batched stamp + ESDF build captured and replayed."""
    import ctypes as C
    scene = scenes.small_scene(74, dims=(40, 32, 28), n_cuboids=3, n_spheres=2)
    lib = api.load_library()
    stream = C.c_void_p()
    assert lib.ks_stream_create(C.byref(stream)) == 0
    cfg = api.make_tsdf_config(scene.tsdf_voxel)
    cfg.capacity = scene.capacity
    tsdf = api.make_tsdf(cfg, stream.value)
    e = api.DenseEsdf(esdf_config(scene), stream.value)
    prims = _prims(scene)

    def enqueue():
        tsdf.upload_frame_async()
        tsdf.integrate_async()
        tsdf.stamp_batch_async(prims)
        e.build_async(tsdf)

    tsdf.stage_frame(frame_of(scene.frames[0]))
    enqueue()
    tsdf.sync()
    g = api.Graph(stream.value)
    with g:
        enqueue()
    for _ in range(2):
        g.launch()
    tsdf.sync()
    cpu = oracle_lib.make_tsdf(scene.tsdf_voxel, capacity=scene.capacity)
    f = scene.frames[0]
    for _ in range(3):
        cpu.integrate_depth(f.depth, f.width, f.height, f.intr, f.R, f.t)
        assert _cpu_sequential(cpu, prims) is None
    _check_state(tsdf, cpu)
    site, dist, _ = e.download(d2=False)
    _, _, site0, dist0 = cpu.build_esdf(scene.esdf_origin, scene.esdf_dims, scene.esdf_voxel)
    assert np.array_equal(site, site0) and np.array_equal(dist, dist0)
    g.close()
