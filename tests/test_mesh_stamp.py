"""Triangle-mesh stamping.

The reference has no mesh implementation, so parity for this one function is UNPINNED: the
CUDA path is compared bit for bit with oracle/ks_oracle.c's restatement of this repo's own definition
(csrc/mesh.cuh), and the definition itself is anchored on the reference's analytic primitives -- a 12-triangle box
must reproduce sdf_cuboid / stamp_primitive(Cuboid) (sdf_world.hpp:224-229, :394-444) and an icosphere must
approach sdf_sphere (:231-233) within its chord error.
"""
from pathlib import Path

import numpy as np
import pytest

import cpu_checkers
from paper_2603_05493_b200 import scenes
from parity_util import assert_world_parity, cpu_world, esdf_config, gpu_world, same_bits


GOLD = Path(__file__).resolve().parent / "golden" / "mesh_restatement.npz"


@pytest.fixture(scope="module")
def oracle():
    return cpu_checkers.oracle()


def _cuboid_sdf(points, center, he, R):
    q = np.abs((points - center) @ R) - he
    return np.linalg.norm(np.maximum(q, 0.0), axis=1) + np.minimum(q.max(axis=1), 0.0)


# ---- the definition, on the CPU ---------------------------------------------------------------------------------
@pytest.mark.parametrize("yaw", [0.0, 0.4, 1.3])
def test_box_mesh_distance_is_the_cuboid_distance(oracle, yaw):
    rng = np.random.RandomState(3)
    c, he, R = np.array([0.3, 0.2, 0.5]), np.array([0.2, 0.1, 0.15]), scenes.rot_z(yaw)
    m = scenes.box_mesh(c, he, R)
    pts = c + (rng.random_sample((20000, 3)) - 0.5)
    d = oracle.mesh_sdf(m.vertices, m.triangles, pts)
    ref = _cuboid_sdf(pts, c, he, R)
    assert np.abs(d - ref).max() < 1e-12
    assert np.array_equal(d < 0, ref < 0)


def test_icosphere_distance_approaches_the_sphere_distance(oracle):
    rng = np.random.RandomState(4)
    c, r = np.array([0.1, -0.2, 0.3]), 0.2
    pts = c + (rng.random_sample((5000, 3)) - 0.5)
    ref = np.linalg.norm(pts - c, axis=1) - r
    worst = []
    for s in (1, 2, 3):
        m = scenes.icosphere(c, r, s)
        d = oracle.mesh_sdf(m.vertices, m.triangles, pts)
        worst.append(np.abs(d - ref).max())
        far = np.abs(ref) > worst[-1]
        assert np.array_equal(d[far] < 0, ref[far] < 0)
        assert (d >= ref - 1e-12).all()  # the inscribed polyhedron lies inside the sphere
    assert worst[0] > worst[1] > worst[2] and worst[2] < 1e-3


def test_points_on_the_surface_are_plus_zero_and_vertices_edges_sign_correctly(oracle):
    m = scenes.box_mesh((0.0, 0.0, 0.0), (1.0, 1.0, 1.0))
    on = np.array([[1.0, 0.0, 0.0], [1.0, 1.0, 0.0], [1.0, 1.0, 1.0], [0.25, -1.0, 0.5]])
    d = oracle.mesh_sdf(m.vertices, m.triangles, on)
    assert np.array_equal(d, np.zeros(4)) and not np.signbit(d).any()
    out = np.array([[2.0, 2.0, 2.0], [2.0, 2.0, 0.0], [0.9, 0.9, 0.9], [0.99, 0.99, 0.0]])
    d = oracle.mesh_sdf(m.vertices, m.triangles, out)
    np.testing.assert_allclose(d, [np.sqrt(3.0), np.sqrt(2.0), -0.1, -0.01], rtol=0, atol=1e-12)


def test_validation_messages(oracle):
    m = scenes.box_mesh((0.0, 0.0, 0.0), (1.0, 1.0, 1.0))
    t = oracle.make_tsdf(0.05, capacity=64)
    bad = m.vertices.copy()
    bad[3, 1] = np.nan
    for verts, tris, text in ((bad, m.triangles, "stamp: non-finite mesh"),
                              (m.vertices, m.triangles + 7, "stamp: mesh index out of range"),
                              (m.vertices, np.array([[0, 0, 1]], np.int32), "stamp: degenerate mesh triangle"),
                              (m.vertices, np.zeros((0, 3), np.int32), "stamp: empty mesh")):
        with pytest.raises(cpu_checkers.CheckerError, match=text):
            t.stamp_mesh(verts, tris)
    assert t.allocated_block_count() == 0


def test_box_mesh_stamp_allocates_and_fills_like_stamp_primitive(oracle):
    """Same candidate blocks, same pool order and the cuboid's distances (to rounding) as the reference's
    stamp_primitive(Cuboid) -- checked against the reference build when present, else the restatement."""
    ref = cpu_checkers.reference() if cpu_checkers.reference_available() else oracle
    c, he, R = np.array([0.31, 0.22, 0.18]), np.array([0.11, 0.07, 0.09]), scenes.rot_z(0.3)
    a = ref.make_tsdf(0.01, capacity=4096)
    a.stamp_cuboid(R, c, he)
    b = oracle.make_tsdf(0.01, capacity=4096)
    m = scenes.box_mesh(c, he, R)
    b.stamp_mesh(m.vertices, m.triangles)
    ak, ap = a.export_blocks()
    bk, bp = b.export_blocks()
    assert np.array_equal(ak, bk) and np.array_equal(ap, bp) and len(ap) > 50
    for pool in ap.tolist():
        ga, gb = a.block_channels(pool)[2], b.block_channels(pool)[2]
        np.testing.assert_allclose(gb, ga, rtol=0, atol=1e-12)


def test_restatement_matches_its_committed_vectors(oracle):
    """tests/golden/mesh_restatement.npz (made by make_mesh_golden.py from liboracle.so -- NOT reference output)."""
    from golden.make_mesh_golden import cases, stamped_world
    gold = np.load(GOLD)
    for name, (mesh, pts) in cases().items():
        assert same_bits(oracle.mesh_sdf(mesh.vertices, mesh.triangles, pts), gold[f"{name}_sdf"]), name
    keys, geom = stamped_world(oracle)
    assert np.array_equal(keys, gold["world_keys"]) and same_bits(geom, gold["world_geom"])


@pytest.mark.gpu
def test_gpu_matches_the_committed_vectors():
    from golden.make_mesh_golden import cases
    from paper_2603_05493_b200 import api
    gold = np.load(GOLD)
    cfg = api.make_tsdf_config(0.02)
    cfg.capacity = 4096
    t = api.make_tsdf(cfg)
    for mesh, _ in cases().values():
        api.stamp_mesh(t, api.TriangleMesh(mesh.vertices, mesh.triangles))
    keys, pool = t.export_blocks()
    order = np.lexsort((keys[:, 2], keys[:, 1], keys[:, 0]))
    assert np.array_equal(keys[order], gold["world_keys"])
    assert same_bits(t.download_blocks(pool[order].tolist())[2], gold["world_geom"])


# ---- the CUDA path against the restatement ------------------------------------------------------------------------
def _mesh_scene(seed, n_meshes=2, subdivisions=2, **kw):
    scene = scenes.small_scene(seed, **kw)
    rng = np.random.RandomState(100 + seed)
    extent = np.array(scene.esdf_dims) * scene.esdf_voxel
    for i in range(n_meshes):
        c = scene.esdf_origin + (0.2 + 0.6 * rng.random_sample(3)) * extent
        if i % 2 == 0:
            scene.meshes.append(scenes.icosphere(c, 0.08 + 0.1 * rng.random_sample(), subdivisions))
        else:
            scene.meshes.append(scenes.box_mesh(c, 0.05 + 0.1 * rng.random_sample(3), scenes.rot_z(rng.random_sample())))
    return scene


@pytest.mark.gpu
@pytest.mark.parametrize("seed", [1, 2, 3])
def test_gpu_mesh_stamp_is_bit_identical_to_the_restatement(oracle, seed):
    from paper_2603_05493_b200 import api
    scene = _mesh_scene(seed)
    tsdf, touched = gpu_world(scene)
    cpu, touched0 = cpu_world(oracle, scene)
    assert touched == touched0
    assert assert_world_parity(tsdf, cpu), "channels not bit-identical"
    esdf = api.build_esdf(tsdf, esdf_config(scene))
    site, dist, _ = esdf.download()
    _, _, site0, dist0 = cpu.build_esdf(scene.esdf_origin, scene.esdf_dims, scene.esdf_voxel)
    assert np.array_equal(site, site0) and same_bits(dist, dist0)
    assert (dist < 0).any() and (dist > 0).any()


@pytest.mark.gpu
def test_gpu_mesh_only_world_and_large_mesh(oracle):
    """5120 triangles (several shared-memory chunks of the stamping kernel), no depth frame, off-grid centre."""
    from paper_2603_05493_b200 import api
    scene = scenes.small_scene(5, n_cuboids=0, n_spheres=0)
    scene.frames.clear()
    scene.meshes.append(scenes.icosphere((0.41, 0.37, 0.33), 0.21, 4))
    tsdf, _ = gpu_world(scene)
    cpu, _ = cpu_world(oracle, scene)
    assert assert_world_parity(tsdf, cpu)
    pts = np.array([[0.41, 0.37, 0.33 + 0.21 - 0.03], [0.41, 0.37, 0.33 + 0.21 + 0.03]])
    sdf, valid = api.query_tsdf_geom(tsdf, pts)
    assert np.asarray(valid).all() and sdf[0] < 0 < sdf[1]


@pytest.mark.gpu
def test_gpu_box_mesh_matches_stamp_primitive_cuboid():
    """The mesh path reproduces the reference-pinned cuboid stamp: same blocks, distances to rounding."""
    from paper_2603_05493_b200 import api
    c, he, R = np.array([0.31, 0.22, 0.18]), np.array([0.11, 0.07, 0.09]), scenes.rot_z(0.3)
    worlds = []
    for as_mesh in (False, True):
        cfg = api.make_tsdf_config(0.01)
        cfg.capacity = 4096
        t = api.make_tsdf(cfg)
        if as_mesh:
            m = scenes.box_mesh(c, he, R)
            api.stamp_mesh(t, api.TriangleMesh(m.vertices, m.triangles))
        else:
            api.stamp_primitive(t, api.Cuboid(R, c, he))
        keys, pool = t.export_blocks()
        worlds.append((keys, pool, t.download_blocks(pool.tolist())[2]))
    assert np.array_equal(worlds[0][0], worlds[1][0]) and np.array_equal(worlds[0][1], worlds[1][1])
    np.testing.assert_allclose(worlds[1][2], worlds[0][2], rtol=0, atol=1e-12)


@pytest.mark.gpu
def test_gpu_mesh_validation_and_capture():
    from paper_2603_05493_b200 import api
    m = scenes.box_mesh((0.2, 0.2, 0.2), (0.1, 0.1, 0.1))
    for verts, tris, text in ((np.full_like(m.vertices, np.inf), m.triangles, "stamp: non-finite mesh"),
                              (m.vertices, m.triangles + 7, "stamp: mesh index out of range"),
                              (m.vertices, np.array([[0, 0, 1]], np.int32), "stamp: degenerate mesh triangle"),
                              (m.vertices, np.zeros((0, 3), np.int32), "stamp: empty mesh")):
        with pytest.raises(api.ValidationError, match=text):
            api.TriangleMesh(verts, tris)
    mesh = api.TriangleMesh(m.vertices, m.triangles)
    assert mesh.triangle_count() == 12
    # pool too small for the candidate blocks: all-or-nothing, as stamp_primitive (sdf_world.hpp:313-317)
    cfg = api.make_tsdf_config(0.01)
    cfg.capacity = 8
    t = api.make_tsdf(cfg)
    with pytest.raises(api.ValidationError, match="pool exhausted"):
        api.stamp_mesh(t, mesh)
    assert api.allocated_block_count(t) == 0


@pytest.mark.gpu
def test_config4_mixed_scene_full_size_against_the_restatement(oracle):
    """BASELINE configs[3] at full size: depth + 3 cuboids + sphere + 1280-triangle mesh into 400 x 200 x 200 cells,
    then one million batched distance + gradient queries (the restatement needs ~10 s)."""
    from paper_2603_05493_b200 import api
    scene, pts = scenes.config4()
    tsdf, touched = gpu_world(scene)
    cpu, touched0 = cpu_world(oracle, scene)
    assert touched == touched0
    assert assert_world_parity(tsdf, cpu)
    e = api.build_esdf(tsdf, esdf_config(scene))
    site, dist, _ = e.download()
    mask0, has0, site0, dist0 = cpu.build_esdf(scene.esdf_origin, scene.esdf_dims, scene.esdf_voxel)
    assert int(e.report().seed_count) == int(mask0.sum())
    assert np.array_equal(site, site0) and same_bits(dist, dist0)
    s = api.query(e, pts)
    d0, g0, i0 = oracle.query_esdf(scene.esdf_origin, scene.esdf_dims, scene.esdf_voxel, has0, dist0, pts)
    assert same_bits(s.distance, d0) and same_bits(s.gradient, g0) and np.array_equal(s.inside, i0)
    # inside the mesh the field is negative, just outside it is positive
    c = np.array([0.35, 0.8, 0.7])
    inside = api.query(e, np.array([c, c + [0.0, 0.0, 0.2]]))
    assert inside.distance[0] < 0 < inside.distance[1]


# ---- an independent checker on non-convex meshes (tests/mesh_independent.py: segment-clamp distance + winding-number sign) ----
def _nonconvex_cases():
    import mesh_independent as mi
    return {"torus": mi.torus((0.4, 0.4, 0.3), 0.2, 0.07), "l_prism": mi.l_prism((0.15, 0.2, 0.1))}


@pytest.mark.parametrize("name", ["torus", "l_prism"])
def test_restatement_agrees_with_the_independent_checker_on_nonconvex_meshes(oracle, name):
    """Different distance algorithm, different sign principle (tests/mesh_independent.py), same answer: magnitudes
    to 1e-12, signs everywhere except within 1e-9 of the surface."""
    import mesh_independent as mi
    verts, tris = _nonconvex_cases()[name]
    rng = np.random.RandomState(11)
    lo, hi = verts.min(axis=0) - 0.15, verts.max(axis=0) + 0.15
    pts = lo + rng.random_sample((6000, 3)) * (hi - lo)
    d = oracle.mesh_sdf(verts, tris, pts)
    ref, wind = mi.signed_distance(verts, tris, pts)
    assert np.abs(np.minimum(np.abs(wind - 1.0), np.abs(wind))).max() < 1e-6, "the test mesh is not closed / consistently oriented"
    np.testing.assert_allclose(np.abs(d), np.abs(ref), rtol=0, atol=1e-12)
    off = np.abs(ref) > 1e-9
    assert np.array_equal(d[off] < 0, ref[off] < 0)
    assert (ref < 0).sum() > 100 and (ref > 0).sum() > 100


@pytest.mark.gpu
@pytest.mark.parametrize("name", ["torus", "l_prism"])
def test_gpu_stamp_of_nonconvex_meshes_against_the_independent_checker(name):
    """ks_tsdf_stamp_mesh on a torus and an L-shaped prism: every stamped voxel's geometry value equals the independent
    signed distance at its centre (1e-12; sign included), blocks = those whose centre lies within truncation + block radius."""
    import mesh_independent as mi
    from paper_2603_05493_b200 import api
    verts, tris = _nonconvex_cases()[name]
    voxel = 0.01
    cfg = api.make_tsdf_config(voxel)
    cfg.capacity = 8192
    t = api.make_tsdf(cfg)
    api.stamp_mesh(t, api.TriangleMesh(verts, tris))
    keys, pools = t.export_blocks()
    assert len(keys) > 100
    _, _, geom = t.download_blocks(pools)
    idx = np.arange(512)
    local = np.stack([idx & 7, (idx >> 3) & 7, idx >> 6], axis=1)
    rng = np.random.RandomState(5)
    pick = rng.choice(len(keys), size=min(len(keys), 120), replace=False)
    centres = np.concatenate([((keys[k][None, :] * 8 + local) + 0.5) * voxel for k in pick])
    ref, _ = mi.signed_distance(verts, tris, centres)
    got = geom[pick].reshape(-1)
    np.testing.assert_allclose(got, ref, rtol=0, atol=1e-12)
    off = np.abs(ref) > 1e-9
    assert np.array_equal(np.signbit(got[off]), ref[off] < 0)
    # candidate rule (stamp_primitive's, sdf_world.hpp:425-431): |sdf(block centre)| <= truncation + half the block diagonal
    bc = (keys * 8 + 4.0) * voxel
    dref, _ = mi.signed_distance(verts, tris, bc)
    reach = cfg.truncation + 0.5 * 8 * voxel * np.sqrt(3.0)
    assert (np.abs(dref) <= reach + 1e-12).all()
