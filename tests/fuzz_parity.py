"""Randomised parity run on the GPU box (not a pytest: minutes, not seconds).

    python tests/fuzz_parity.py [--seconds 300] [--seed 1]

Draws small mixed scenes with random grid shapes, ESDF/TSDF voxel ratios, off-grid origins and primitive counts,
runs the CUDA path and the CPU oracle on each, and compares block tables, seed masks, sites, signed distances and
queries exactly.  Stops at the first mismatch with the scene's parameters (reproducible from the printed seed).
"""
import argparse
import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent.parent
for p in (str(ROOT), str(ROOT / "tests")):
    if p not in sys.path:
        sys.path.insert(0, p)

import cpu_checkers  # noqa: E402
from paper_2603_05493_b200 import api, scenes  # noqa: E402
from parity_util import assert_world_parity, cpu_world, esdf_config, gpu_world, same_bits  # noqa: E402


def one_case(oracle, rng, index, meshes=False):
    ratio = float(rng.choice([1.0, 1.0, 1.0, 0.5, 0.75, 1.0 / 3.0, 0.4, 0.9, 1.25, 2.0]))
    tsdf_voxel = float(rng.choice([0.02, 0.025, 0.013]))
    dims = tuple(int(v) for v in rng.randint(5, 72, 3))
    if rng.random_sample() < 0.2:
        dims = (int(rng.choice([4, 8, 32, 64, 100])), dims[1], dims[2])  # nx % 4 == 0 (cp.async fill) and exact tiles
    aligned = rng.random_sample() < 0.5
    origin = (rng.randint(-40, 40, 3) * tsdf_voxel) if aligned else (rng.random_sample(3) - 0.5) * 1.7
    params = dict(dims=dims, tsdf_voxel=tsdf_voxel, ratio=ratio, origin=tuple(float(v) for v in origin),
                  n_cuboids=int(rng.randint(0, 4)), n_spheres=int(rng.randint(0, 3)))
    scene = scenes.small_scene(int(rng.randint(1, 10**6)), **params)
    n_meshes = int(rng.choice([0, 0, 1, 2])) if meshes else 0
    ext = np.array(scene.esdf_dims) * scene.esdf_voxel
    for _ in range(n_meshes):  # closed meshes: icospheres of 20..1280 triangles, rotated boxes; some poking out of the grid
        c = scene.esdf_origin + (rng.random_sample(3) * 1.2 - 0.1) * ext
        if rng.random_sample() < 0.5:
            scene.meshes.append(scenes.icosphere(c, 0.03 + rng.random_sample() * 0.2 * ext.min(), int(rng.randint(0, 4))))
        else:
            scene.meshes.append(scenes.box_mesh(c, 0.02 + rng.random_sample(3) * 0.2 * ext.min(), scenes.rot_z(rng.random_sample() * 3.0) @ scenes.rot_y(rng.random_sample())))
    params["n_meshes"] = n_meshes
    seeding = "gather" if rng.random_sample() < 0.85 else "scatter"
    tsdf, touched = gpu_world(scene)
    cpu, touched0 = cpu_world(oracle, scene)
    assert touched == touched0, ("touched", params)
    assert_world_parity(tsdf, cpu)
    cfg = esdf_config(scene, seeding)
    e = api.build_esdf(tsdf, cfg)
    site, dist, d2 = e.download()
    mask0, has0, site0, dist0 = cpu.build_esdf(scene.esdf_origin, scene.esdf_dims, scene.esdf_voxel, seeding)
    assert int(e.report().seed_count) == int(mask0.sum()), ("seed count", params, seeding)
    assert np.array_equal(site, site0), ("sites", params, seeding)
    assert np.array_equal(dist, dist0) and np.array_equal(np.signbit(dist), np.signbit(dist0)), ("signed distance", params, seeding)
    pts = scene.esdf_origin + (rng.random_sample((2000, 3)) * 1.2 - 0.1) * ext
    s = api.query(e, pts)
    d0, g0, i0 = oracle.query_esdf(scene.esdf_origin, scene.esdf_dims, scene.esdf_voxel, has0, dist0, pts)
    assert same_bits(s.distance, d0) and same_bits(s.gradient, g0) and np.array_equal(s.inside, i0), ("query", params)
    return params, seeding, int(mask0.sum())


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--seconds", type=float, default=300.0)
    ap.add_argument("--seed", type=int, default=1)
    ap.add_argument("--meshes", action="store_true", help="also stamp 0-2 random triangle meshes per scene")
    args = ap.parse_args()
    oracle = cpu_checkers.oracle()
    rng = np.random.RandomState(args.seed)
    t0 = time.time()
    n = 0
    ratios = {}
    while time.time() - t0 < args.seconds:
        params, seeding, seeds = one_case(oracle, rng, n, args.meshes)
        ratios[round(params["ratio"], 3)] = ratios.get(round(params["ratio"], 3), 0) + 1
        n += 1
        if n % 25 == 0:
            print(f"{n} scenes ok ({time.time() - t0:.0f} s), last: {params} {seeding} seeds={seeds}", flush=True)
    print(f"fuzz ok: {n} scenes, seed {args.seed}, by ratio {dict(sorted(ratios.items()))}")


if __name__ == "__main__":
    main()
