"""Handle-level behaviour on the GPU: several live ESDFs of different sizes, one ESDF rebuilt against worlds with
different pool sizes, builds and world updates on separate streams (round-1 advisor findings)."""
import numpy as np
import pytest

from paper_2603_05493_b200 import api, scenes
from parity_util import assert_world_parity, cpu_world, esdf_config, frame_of, gpu_world

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _built():
    from paper_2603_05493_b200 import build
    build.build()
    assert api.load_library().ks_device_count() > 0, "GPU tests need a CUDA device"


def _oracle_field(cpu, scene):
    _, _, site0, dist0 = cpu.build_esdf(scene.esdf_origin, scene.esdf_dims, scene.esdf_voxel)
    return site0, dist0


def test_two_esdfs_of_different_sizes_coexist(oracle_lib):
    """A long-row ESDF (x sweep tile > 48 KB of shared memory) stays usable after a small one is created: the
    dynamic-shared-memory attribute is per kernel, process-wide, and must never be lowered."""
    big = scenes.small_scene(61, dims=(400, 24, 16), tsdf_voxel=0.01)
    small = scenes.small_scene(62, dims=(20, 18, 16))
    t_big, _ = gpu_world(big)
    c_big, _ = cpu_world(oracle_lib, big)
    e_big = api.build_esdf(t_big, esdf_config(big))
    t_small, _ = gpu_world(small)
    c_small, _ = cpu_world(oracle_lib, small)
    e_small = api.build_esdf(t_small, esdf_config(small))
    e_big.profile(True)  # plain launches (no private graph): every kernel is configured again
    api.build_esdf(t_big, esdf_config(big), e_big)
    e_big.profile(False)
    api.build_esdf(t_big, esdf_config(big), e_big)  # and through a freshly captured private graph
    for e, cpu, sc in ((e_big, c_big, big), (e_small, c_small, small)):
        site, dist, _ = e.download(d2=False)
        site0, dist0 = _oracle_field(cpu, sc)
        assert np.array_equal(site, site0) and np.array_equal(dist, dist0)


def test_one_esdf_rebuilt_against_a_world_with_a_larger_pool(oracle_lib):
    """build_esdf(tsdf2, esdf) after build_esdf(tsdf1, esdf): same voxel size, 16x the pool (per-pool-entry scratch must grow)."""
    scene = scenes.small_scene(63, dims=(44, 40, 30))
    first, _ = gpu_world(scene, capacity=700)
    cfg = esdf_config(scene)
    e = api.build_esdf(first, cfg)
    big_scene = scenes.small_scene(64, dims=(44, 40, 30), n_cuboids=3, n_spheres=2, capacity=12000)
    second, _ = gpu_world(big_scene)
    for _ in range(3):  # push the second world's pool indices past the first world's capacity
        f = big_scene.frames[0]
        shifted = scenes.Frame(f.depth + np.float32(0.11), f.R, f.t + np.array([0.2, 0.1, 0.0]), f.width, f.height, f.intr)
        api.integrate_depth(second, frame_of(shifted))
        big_scene.frames.append(shifted)
    cpu, _ = cpu_world(oracle_lib, big_scene)
    assert_world_parity(second, cpu, exact_pool=False)
    api.build_esdf(second, cfg, e)
    site, dist, _ = e.download(d2=False)
    site0, dist0 = _oracle_field(cpu, big_scene)
    assert np.array_equal(site, site0) and np.array_equal(dist, dist0)
    # and the scatter path, which rebuilds the per-pool-entry flags too
    mask = api.seed_scatter(second, cfg, e)
    assert np.array_equal(mask, cpu.seed_scatter(big_scene.esdf_origin, big_scene.esdf_dims, big_scene.esdf_voxel))


def test_async_build_and_world_updates_on_separate_streams(oracle_lib):
    """ks_esdf_build_async on the ESDF's own stream, then mutating TSDF calls on the world's stream without any
    host synchronisation in between: the update must wait for the build that still reads the world."""
    scene = scenes.small_scene(65, dims=(64, 48, 40))
    tsdf, _ = gpu_world(scene)
    cpu, _ = cpu_world(oracle_lib, scene)
    e = api.DenseEsdf(esdf_config(scene))  # own stream, not the world's
    fields = []
    f = scene.frames[0]
    for k in range(4):
        e.build_async(tsdf)  # reads the world as it stands now
        fields.append(_oracle_field(cpu, scene))
        c = scene.esdf_origin + np.array([0.2 + 0.15 * k, 0.3, 0.25])
        tsdf.stamp_async(api.SphereShape(c, 0.07))  # enqueued right behind, on the world's stream
        cpu.stamp_sphere(c, 0.07)
        site, dist, _ = e.download(d2=False)  # the build enqueued BEFORE the stamp
        assert np.array_equal(site, fields[-1][0]) and np.array_equal(dist, fields[-1][1]), k
    tsdf.sync()
    assert_world_parity(tsdf, cpu)


def test_graph_captured_before_a_larger_frame_keeps_its_buffers(oracle_lib):
    """A graph captured with a small frame stays valid after a larger frame grew the staging slot and the op lists:
    the old buffers are retired, not freed, so replaying the old graph integrates the OLD frame again (the memory it
    was captured with) -- no use after free, and the world equals the oracle's for that sequence of frames."""
    import ctypes as C
    small = scenes.small_scene(71, width=48, height=36, n_cuboids=0, n_spheres=0)
    large = scenes.small_scene(72, width=160, height=120, n_cuboids=0, n_spheres=0)
    lib = api.load_library()
    stream = C.c_void_p()
    assert lib.ks_stream_create(C.byref(stream)) == 0
    cfg = api.make_tsdf_config(small.tsdf_voxel)
    cfg.capacity = 8192
    t = api.make_tsdf(cfg, stream.value)
    fs, fl = small.frames[0], large.frames[0]
    t.stage_frame(frame_of(fs))
    t.upload_frame_async()
    t.integrate_async()
    t.sync()
    g = api.Graph(stream.value)
    with g:
        t.upload_frame_async()
        t.integrate_async()
    g.launch()
    t.sync()
    t.stage_frame(frame_of(fl))  # 11x the pixels: slot and op lists grow
    t.upload_frame_async()
    t.integrate_async()
    rep = t.sync()
    assert rep.status == 0
    for _ in range(2):
        g.launch()  # the old graph: the small frame once more, from the retired buffers
    rep = t.sync()
    assert rep.status == 0
    cpu = oracle_lib.make_tsdf(small.tsdf_voxel, capacity=8192)
    for f in (fs, fs, fl, fs, fs):
        cpu.integrate_depth(f.depth, f.width, f.height, f.intr, f.R, f.t)
    assert assert_world_parity(t, cpu)
    g.close()
