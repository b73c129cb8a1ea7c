"""Generate tests/golden/*.npz from the REFERENCE build (oracle/_ref/libks_ref.so).

Run in the build container, where /root/reference is mounted:
    python tests/golden/make_golden.py
The fixtures let the oracle (and through it the CUDA path) be pinned on boxes where the
reference tree does not exist.  Inputs are regenerated from seeds by the tests themselves
(paper_2603_05493_b200.scenes / numpy RandomState), only reference OUTPUTS are stored.
"""
import hashlib
import sys
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
sys.path.insert(0, str(HERE.parent))
sys.path.insert(0, str(HERE.parent.parent))

import cpu_checkers  # noqa: E402
from paper_2603_05493_b200 import scenes  # noqa: E402

EDT_CASES = [  # (seed, dims, n_seeds)
    (0, (1, 1, 1), 1), (1, (7, 1, 1), 2), (2, (1, 9, 1), 3), (3, (1, 1, 11), 2), (4, (17, 13, 9), 5),
    (5, (32, 32, 32), 100), (6, (33, 20, 41), 1), (7, (64, 64, 64), 500), (8, (40, 3, 25), 60),
    (9, (21, 34, 2), 400),
]


def edt_mask(seed, dims, n_seeds):
    rng = np.random.RandomState(seed)
    cells = dims[0] * dims[1] * dims[2]
    mask = np.zeros(cells, np.uint8)
    mask[rng.choice(cells, min(n_seeds, cells), replace=False)] = 1
    return mask


def d2_from_site(site, dims):
    nx, ny, nz = dims
    z, y, x = np.meshgrid(np.arange(nz), np.arange(ny), np.arange(nx), indexing="ij")
    cell = np.stack([x.ravel(), y.ravel(), z.ravel()], 1).astype(np.int64)
    d = cell - site.astype(np.int64)
    return (d * d).sum(1).astype(np.int32)


def run_scene(lib, scene):
    t = lib.make_tsdf(scene.tsdf_voxel, capacity=scene.capacity)
    touched = [t.integrate_depth(f.depth, f.width, f.height, f.intr, f.R, f.t) for f in scene.frames]
    for c in scene.cuboids:
        t.stamp_cuboid(c.R, c.t, c.half_extents)
    for s in scene.spheres:
        t.stamp_sphere(s.center, s.radius)
    keys, pool = t.export_blocks()
    order = np.lexsort((keys[:, 2], keys[:, 1], keys[:, 0]))
    keys, pool = keys[order], pool[order]
    chans = np.stack([np.stack(t.block_channels(int(p))) for p in pool])  # [L, 3, 512]
    mask, has, site, dist = t.build_esdf(scene.esdf_origin, scene.esdf_dims, scene.esdf_voxel)
    scatter = t.seed_scatter(scene.esdf_origin, scene.esdf_dims, scene.esdf_voxel)
    rng = np.random.RandomState(99)
    ext = np.array(scene.esdf_dims) * scene.esdf_voxel
    pts = scene.esdf_origin + (rng.random_sample((256, 3)) * 1.2 - 0.1) * ext
    qd, qg, qi = lib.query_esdf(scene.esdf_origin, scene.esdf_dims, scene.esdf_voxel, has, dist, pts)
    tq, tv = t.query_tsdf(pts)
    return dict(touched=np.array(touched, np.int32), keys=keys, pool=pool,
                chan_sha=np.frombuffer(hashlib.sha256(chans.tobytes()).digest(), np.uint8),
                chan_head=chans[:4], gather=np.packbits(mask), scatter=np.packbits(scatter),
                has=np.array([has]), site=site.astype(np.int16), dist=dist, q_pts=pts, q_dist=qd, q_grad=qg,
                q_inside=qi, tq=tq, tv=tv)


def main():
    cpu_checkers.build_checkers()
    ref = cpu_checkers.reference()
    out = {}
    for seed, dims, n in EDT_CASES:
        has, site, dist = ref.propagate(edt_mask(seed, dims, n), dims, 0.01)
        out[f"edt{seed}_site"] = site.astype(np.int16)
        out[f"edt{seed}_d2"] = d2_from_site(site, dims)
        out[f"edt{seed}_dist"] = dist
    np.savez_compressed(HERE / "edt_reference.npz", **out)
    for seed, kw in SCENE_CASES.items():
        res = run_scene(ref, scenes.small_scene(seed, **kw))
        np.savez_compressed(HERE / f"scene{seed}_reference.npz", **res)
    print("wrote", sorted(p.name for p in HERE.glob("*.npz")))


SCENE_CASES = {
    1: dict(),
    2: dict(ratio=2.0, dims=(30, 20, 25)),
    3: dict(ratio=0.5, dims=(60, 50, 40), origin=(-0.3, 0.1, -0.2)),
}

if __name__ == "__main__":
    main()
