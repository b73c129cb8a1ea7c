"""The C oracle against the live reference build (only where /root/reference is mounted)."""
import numpy as np
import pytest

from paper_2603_05493_b200 import scenes


def _same_bits(a, b):
    return np.array_equal(np.ascontiguousarray(a).view(np.uint64), np.ascontiguousarray(b).view(np.uint64))


def _assert_same_world(a, b):
    ka, pa = a.export_blocks()
    kb, pb = b.export_blocks()
    assert np.array_equal(ka, kb) and np.array_equal(pa, pb)  # same slots, same pool indices
    assert np.array_equal(a.free_list(), b.free_list())
    assert a.next_fresh() == b.next_fresh() and a.available() == b.available()
    for p in pa:
        for x, y in zip(a.block_channels(int(p)), b.block_channels(int(p))):
            assert _same_bits(x, y)


@pytest.mark.parametrize("seed", [11, 12, 13])
def test_dynamic_scene_lifecycle_is_identical(oracle_lib, reference_lib, seed):
    """integrate / stamp / decay / recycle / re-integrate at a new pose, 6 rounds, tiny pool."""
    rng = np.random.RandomState(seed)
    sc = scenes.small_scene(seed, dims=(24, 20, 18), n_cuboids=0, n_spheres=0)
    worlds = [lib.make_tsdf(sc.tsdf_voxel, capacity=400, weight_threshold=40.0, alpha_time=0.7)
              for lib in (oracle_lib, reference_lib)]
    f = sc.frames[0]
    for rnd in range(6):
        t = f.t + np.array([0.25 * rnd, 0.0, 0.0])
        depth = f.depth + np.float32(0.05 * rnd)
        touched = []
        for w in worlds:
            try:
                touched.append(w.integrate_depth(depth, f.width, f.height, f.intr, f.R, t))
            except Exception as e:  # pool exhaustion must agree too, message included
                touched.append(str(e))
        assert touched[0] == touched[1]
        if rnd == 2:
            centre = sc.esdf_origin + rng.random_sample(3) * 0.3
            for w in worlds:
                w.stamp_sphere(centre, 0.07)
        for _ in range(3):
            for w in worlds:
                w.decay_weights(f.width, f.height, f.intr, f.R, t)
        assert worlds[0].recycle_blocks() == worlds[1].recycle_blocks()
        _assert_same_world(*worlds)


def test_pool_exhaustion_is_all_or_nothing(oracle_lib, reference_lib):
    sc = scenes.small_scene(5)
    f = sc.frames[0]
    for lib in (oracle_lib, reference_lib):
        w = lib.make_tsdf(sc.tsdf_voxel, capacity=8)
        with pytest.raises(Exception, match=r"tsdf: pool exhausted, frame requires \d+ new blocks but only 8 are available"):
            w.integrate_depth(f.depth, f.width, f.height, f.intr, f.R, f.t)
        assert w.allocated_block_count() == 0 and w.next_fresh() == 0


@pytest.mark.parametrize("seed,ratio,origin", [(21, 1.0, (0, 0, 0)), (22, 1.5, (0.013, -0.2, 0.4)), (23, 4.0, (0, 0, 0)),
                                               (24, 0.25, (-0.1, -0.1, -0.1))])
def test_esdf_stages_are_identical(oracle_lib, reference_lib, seed, ratio, origin):
    dims = (max(2, int(40 / ratio)), max(2, int(36 / ratio)), max(2, int(30 / ratio))) if ratio >= 1 else (50, 44, 38)
    sc = scenes.small_scene(seed, dims=dims, ratio=ratio, origin=origin)
    res = []
    for lib in (oracle_lib, reference_lib):
        w = lib.make_tsdf(sc.tsdf_voxel, capacity=sc.capacity)
        for f in sc.frames:
            w.integrate_depth(f.depth, f.width, f.height, f.intr, f.R, f.t)
        for c in sc.cuboids:
            w.stamp_cuboid(c.R, c.t, c.half_extents)
        for s in sc.spheres:
            w.stamp_sphere(s.center, s.radius)
        gather = w.seed_gather(sc.esdf_origin, sc.esdf_dims, sc.esdf_voxel)
        scatter = w.seed_scatter(sc.esdf_origin, sc.esdf_dims, sc.esdf_voxel)
        has, site, dist = lib.propagate(gather, sc.esdf_dims, sc.esdf_voxel)
        signed = w.recover_signs(sc.esdf_origin, sc.esdf_dims, sc.esdf_voxel, has, site, dist)
        rng = np.random.RandomState(seed)
        pts = sc.esdf_origin + (rng.random_sample((2000, 3)) * 1.4 - 0.2) * np.array(dims) * sc.esdf_voxel
        q = lib.query_esdf(sc.esdf_origin, sc.esdf_dims, sc.esdf_voxel, has, signed, pts)
        tq = w.query_tsdf(pts)
        tg = w.query_tsdf(pts, geom_only=True)
        res.append((gather, scatter, has, site, dist, signed, q, tq, tg))
    a, b = res
    assert gather.sum() > 0
    assert np.array_equal(a[0], b[0]) and np.array_equal(a[1], b[1]) and a[2] == b[2]
    assert np.array_equal(a[3], b[3]) and _same_bits(a[4], b[4]) and _same_bits(a[5], b[5])
    assert _same_bits(a[6][0], b[6][0]) and _same_bits(a[6][1], b[6][1]) and np.array_equal(a[6][2], b[6][2])
    for i in (7, 8):
        assert _same_bits(a[i][0], b[i][0]) and np.array_equal(a[i][1], b[i][1])


def test_propagate_random_grids_with_ties(oracle_lib, reference_lib):
    rng = np.random.RandomState(3)
    for trial in range(25):
        dims = tuple(int(v) for v in rng.randint(1, 40, 3))
        cells = dims[0] * dims[1] * dims[2]
        mask = (rng.random_sample(cells) < rng.choice([0.002, 0.02, 0.3])).astype(np.uint8)
        ha, sa, da = oracle_lib.propagate(mask, dims, 0.02)
        hb, sb, db = reference_lib.propagate(mask, dims, 0.02)
        assert ha == hb and np.array_equal(sa, sb) and _same_bits(da, db)


def _collision_case(lib, seed):
    sc = scenes.small_scene(seed, dims=(36, 30, 26))
    w = lib.make_tsdf(sc.tsdf_voxel, capacity=sc.capacity)
    for f in sc.frames:
        w.integrate_depth(f.depth, f.width, f.height, f.intr, f.R, f.t)
    for c in sc.cuboids:
        w.stamp_cuboid(c.R, c.t, c.half_extents)
    for s in sc.spheres:
        w.stamp_sphere(s.center, s.radius)
    _, has, _, dist = w.build_esdf(sc.esdf_origin, sc.esdf_dims, sc.esdf_voxel)
    rng = np.random.RandomState(seed)
    ext = np.array(sc.esdf_dims) * sc.esdf_voxel
    S, T = 40, 6
    centers = sc.esdf_origin + (rng.random_sample((T, S, 3)) * 1.1 - 0.05) * ext
    centers[1:] = centers[0] + np.cumsum(rng.normal(0, 0.05, (T - 1, S, 3)), 0)
    vel = rng.normal(0, 0.3, (T, S, 3))
    vel[2, :5] = 0.0
    radii = 0.02 + rng.random_sample(S) * 0.08
    static = lib.scene_collision_static(sc.esdf_origin, sc.esdf_dims, sc.esdf_voxel, has, dist, centers[0], radii)
    swept = lib.scene_collision_swept(sc.esdf_origin, sc.esdf_dims, sc.esdf_voxel, has, dist, centers, radii, vel, dt=0.1)
    return static, swept


@pytest.mark.parametrize("seed", [51, 52])
def test_scene_collision_is_identical(oracle_lib, reference_lib, seed):
    (a_static, a_swept), (b_static, b_swept) = _collision_case(oracle_lib, seed), _collision_case(reference_lib, seed)
    assert a_static[:3] == b_static[:3] and _same_bits(a_static[3], b_static[3])
    assert a_static[2] > 0 and a_static[1] >= 0          # the fixture does collide
    for x, y in zip(a_swept, b_swept):
        assert _same_bits(x, y)
    assert a_swept[0][:, 2].sum() > 0
