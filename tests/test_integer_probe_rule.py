"""The integer sign-probe rule of the x sweep (csrc/esdf.cu SignTable::negative, E.iprobe) against the reference's
fp64 arithmetic, on the CPU.

recover_signs (esdf.hpp:297-304) probes the geometry channel at  site_center + ve * delta.normalized()  and
query_tsdf_geom takes  floor(probe / v)  per axis (sdf_world.hpp:254-258).  When ve == v and the cell centres sit at
voxel centres, ks_b200 replaces that by: the probe's voxel = the site's voxel + sign(d_a) on every axis with
4 d_a^2 > |d|^2 (integers).  This test evaluates the reference's expressions in numpy fp64 -- same operand order, Eigen's
a0 + (a1 + a2) reduction -- for every offset up to 40 cells per axis and a few hundred thousand larger ones, on several
voxel sizes and grid origins, and expects the integer rule everywhere.
"""
import numpy as np
import pytest


def reference_offsets(site, d, v, origin):
    """voxel(probe) - voxel(site centre), the way the reference computes it; site, d: integer arrays [N, 3]."""
    site_c = origin + (site + 0.5) * v                     # EsdfConfig::cell_center (esdf.hpp:51-53)
    query_c = origin + (site + d + 0.5) * v
    delta = query_c - site_c
    n = np.sqrt(delta[:, 0] ** 2 + (delta[:, 1] ** 2 + delta[:, 2] ** 2))  # squaredNorm: a0 + (a1 + a2)
    probe = site_c + v * (delta / n[:, None])              # site_center + voxel_size * delta.normalized()
    return (np.floor(probe / v) - np.floor(site_c / v)).astype(np.int64)


def integer_rule(d):
    d2 = (d.astype(np.int64) ** 2).sum(axis=1, keepdims=True)
    return np.where(4 * d.astype(np.int64) ** 2 > d2, np.sign(d), 0)


@pytest.mark.parametrize("v,origin", [(0.005, (0.0, 0.0, 0.0)), (0.01, (0.0, 0.0, 0.0)), (0.002, (0.0, 0.0, 0.0)),
                                      (0.02, (-0.74, 0.5, 0.22)), (0.013, (1.3, -2.6, 0.013)), (0.005, (35.0, -12.0, 7.5))])
def test_every_offset_up_to_40_cells(v, origin):
    r = np.arange(-40, 41)
    d = np.stack(np.meshgrid(r, r, r, indexing="ij"), axis=-1).reshape(-1, 3)
    d = d[(d != 0).any(axis=1)]
    origin = np.asarray(origin, np.float64)
    # the rule needs the centres at voxel middles: true for these origins (multiples of v), as bind_tsdf checks per axis
    q = (origin + 0.5 * v) / v
    assert np.abs(q - np.floor(q) - 0.5).max() < 1e-9
    rng = np.random.RandomState(1)
    site = rng.randint(0, 400, size=d.shape)
    assert np.array_equal(reference_offsets(site, d, v, origin), integer_rule(d))


def test_large_offsets_and_near_misses():
    """Offsets up to 1023 per axis (d2 < 2^22), including the vectors that come closest to the 4 d_a^2 = |d|^2 boundary
    (|4 a^2 - d2| small): the margin 1 / (6 d2) is still five orders of magnitude above fp64 rounding."""
    rng = np.random.RandomState(2)
    d = rng.randint(-1023, 1024, size=(400_000, 3))
    # near misses: 3 a^2 close to b^2 + c^2 -> choose b, c then the nearest a
    b, c = rng.randint(1, 1000, size=(2, 200_000))
    a = np.rint(np.sqrt((b.astype(np.float64) ** 2 + c.astype(np.float64) ** 2) / 3.0)).astype(np.int64)
    near = np.stack([a * rng.choice([-1, 1], size=a.shape), b, c], axis=1)
    near = near[:, rng.permutation(3)]
    d = np.concatenate([d, near])
    d = d[(d != 0).any(axis=1)]
    assert (4 * d.astype(np.int64) ** 2 != (d.astype(np.int64) ** 2).sum(axis=1, keepdims=True)).all(), "3 a^2 = b^2 + c^2 has no integer solution"
    site = rng.randint(0, 1024, size=d.shape)
    for v, origin in ((0.005, np.zeros(3)), (0.002, np.array([0.4, -0.2, 1.0]))):
        assert np.array_equal(reference_offsets(site, d, v, origin), integer_rule(d))
