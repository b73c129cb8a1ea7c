"""Run one synthetic scene through the CUDA path (C ABI) and through a CPU checker, for comparison."""
import numpy as np

from paper_2603_05493_b200 import api


def frame_of(f) -> api.DepthFrame:
    return api.DepthFrame(f.width, f.height, f.intr[0], f.intr[1], f.intr[2], f.intr[3], f.R, f.t, f.depth)


def gpu_world(scene, **cfg_overrides):
    cfg = api.make_tsdf_config(scene.tsdf_voxel)
    cfg.capacity = scene.capacity
    for k, v in cfg_overrides.items():
        setattr(cfg, k, v)
    tsdf = api.make_tsdf(cfg)
    touched = [api.integrate_depth(tsdf, frame_of(f)) for f in scene.frames]
    for c in scene.cuboids:
        api.stamp_primitive(tsdf, api.Cuboid(c.R, c.t, c.half_extents))
    for s in scene.spheres:
        api.stamp_primitive(tsdf, api.SphereShape(s.center, s.radius))
    for m in getattr(scene, "meshes", []):
        api.stamp_mesh(tsdf, api.TriangleMesh(m.vertices, m.triangles))
    return tsdf, touched


def cpu_world(lib, scene, **kw):
    t = lib.make_tsdf(scene.tsdf_voxel, capacity=scene.capacity, **kw)
    touched = [t.integrate_depth(f.depth, f.width, f.height, f.intr, f.R, f.t) for f in scene.frames]
    for c in scene.cuboids:
        t.stamp_cuboid(c.R, c.t, c.half_extents)
    for s in scene.spheres:
        t.stamp_sphere(s.center, s.radius)
    for m in getattr(scene, "meshes", []):  # restatement only: the reference build has no mesh stamping
        t.stamp_mesh(m.vertices, m.triangles)
    return t, touched


def esdf_config(scene, seeding="gather") -> api.EsdfConfig:
    return api.EsdfConfig(tuple(scene.esdf_origin), scene.esdf_dims[0], scene.esdf_dims[1], scene.esdf_dims[2],
                          scene.esdf_voxel, seeding)


def same_bits(a, b):
    a = np.ascontiguousarray(a, np.float64)
    b = np.ascontiguousarray(b, np.float64)
    return a.shape == b.shape and np.array_equal(a.view(np.uint64), b.view(np.uint64))


def assert_world_parity(gpu: api.SparseTsdf, cpu, exact_pool=True, rtol=1e-5):
    """Block allocation bit-exact (key set, and pool indices on no-recycle histories); TSDF channels
    within 1e-5 relative (the north-star tolerance) -- and we additionally record bit equality."""
    gk, gp = gpu.export_blocks()
    ck, cp = cpu.export_blocks()
    g = {tuple(k): int(p) for k, p in zip(gk.tolist(), gp.tolist())}
    c = {tuple(k): int(p) for k, p in zip(ck.tolist(), cp.tolist())}
    assert set(g) == set(c), "live key sets differ"
    if exact_pool:
        assert g == c, "key -> pool assignment differs"
        assert np.array_equal(gk, ck) and np.array_equal(gp, cp), "hash slot order differs from sequential insertion"
    keys = sorted(g)
    gs, gw, gg = gpu.download_blocks([g[k] for k in keys])
    bit_exact = True
    for i, k in enumerate(keys):
        cs, cw, cg = cpu.block_channels(c[k])
        assert np.array_equal(np.isinf(gg[i]), np.isinf(cg)), k
        fin = np.isfinite(cg)
        np.testing.assert_allclose(gs[i], cs, rtol=rtol, atol=1e-300)
        np.testing.assert_allclose(gw[i], cw, rtol=rtol, atol=1e-300)
        np.testing.assert_allclose(gg[i][fin], cg[fin], rtol=rtol, atol=1e-300)
        bit_exact &= same_bits(gs[i], cs) and same_bits(gw[i], cw) and same_bits(gg[i], cg)
    return bit_exact
