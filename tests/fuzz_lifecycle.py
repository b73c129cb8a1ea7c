"""Randomised world-model lifecycle on the GPU box: integrate / stamp / decay / recycle sequences with small pools
(exhaustion included), CUDA path vs oracle after every step: return values, exception texts, key -> pool
assignment, hash slot order, free list, channels.

    python tests/fuzz_lifecycle.py [--seconds 300] [--seed 1]
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
from parity_util import assert_world_parity, esdf_config, same_bits  # noqa: E402


def both(gpu_call, cpu_call, what):
    """Run the same operation on both sides; they must agree on the result or on the exception text."""
    try:
        want = cpu_call()
    except Exception as err:  # noqa: BLE001
        try:
            gpu_call()
        except api.ValidationError as got:
            assert str(got) == str(err) or str(got) in str(err), (what, str(got), str(err))
            return None
        raise AssertionError(f"{what}: the oracle raised {err!r}, the GPU path did not")
    got = gpu_call()
    assert got == want, (what, got, want)
    return got


def one_world(oracle, rng, esdf_every=0.5):
    sc = scenes.small_scene(int(rng.randint(1, 10**6)), dims=(24, 20, 18), n_cuboids=0, n_spheres=0)
    f = sc.frames[0]
    capacity = int(rng.choice([60, 150, 400, 2000]))
    wt, alpha = float(rng.choice([5.0, 40.0, 200.0])), float(rng.choice([0.5, 0.7, 0.95]))
    cfg = api.make_tsdf_config(sc.tsdf_voxel)
    cfg.capacity, cfg.weight_threshold, cfg.alpha_time = capacity, wt, alpha
    tsdf = api.make_tsdf(cfg)
    cpu = oracle.make_tsdf(sc.tsdf_voxel, capacity=capacity, weight_threshold=wt, alpha_time=alpha)
    steps = 0
    t = f.t.copy()
    # ONE DenseEsdf for the world's whole life, rebuilt into after some of the operations: its directory, planes, site
    # tables, double-buffered field and private graph must follow every allocation / recycling / stamp
    esdf = api.DenseEsdf(esdf_config(sc)) if esdf_every else None
    for _ in range(int(rng.randint(4, 12))):
        op = rng.choice(["integrate", "integrate", "sphere", "cuboid", "mesh", "decay", "recycle"])
        if op == "integrate":
            t = f.t + np.array([0.25 * rng.randint(0, 4), 0.1 * rng.randint(0, 3), 0.0])
            depth = f.depth + np.float32(0.05 * rng.randint(0, 5))
            fr = api.DepthFrame(f.width, f.height, *f.intr, f.R, t, depth)
            both(lambda: api.integrate_depth(tsdf, fr), lambda: cpu.integrate_depth(depth, f.width, f.height, f.intr, f.R, t), op)
        elif op == "sphere":
            c, r = sc.esdf_origin + rng.random_sample(3) * 0.4, 0.03 + 0.1 * rng.random_sample()
            both(lambda: api.stamp_primitive(tsdf, api.SphereShape(c, r)), lambda: cpu.stamp_sphere(c, r), op)
        elif op == "cuboid":
            c, he = sc.esdf_origin + rng.random_sample(3) * 0.4, 0.02 + 0.12 * rng.random_sample(3)
            R = scenes.rot_z(float(rng.random_sample()))
            both(lambda: api.stamp_primitive(tsdf, api.Cuboid(R, c, he)), lambda: cpu.stamp_cuboid(R, c, he), op)
        elif op == "mesh":  # icosphere or rotated box as triangles: allocation (and exhaustion) must behave like the primitives
            c = sc.esdf_origin + rng.random_sample(3) * 0.4
            m = (scenes.icosphere(c, 0.03 + 0.1 * rng.random_sample(), int(rng.randint(0, 3))) if rng.random_sample() < 0.5
                 else scenes.box_mesh(c, 0.02 + 0.12 * rng.random_sample(3), scenes.rot_z(float(rng.random_sample()))))
            dm = api.TriangleMesh(m.vertices, m.triangles)
            both(lambda: api.stamp_mesh(tsdf, dm), lambda: cpu.stamp_mesh(m.vertices, m.triangles), op)
        elif op == "decay":
            fr = api.DepthFrame(f.width, f.height, *f.intr, f.R, t, f.depth)
            for _ in range(int(rng.randint(1, 4))):
                api.decay_weights(tsdf, fr)
                cpu.decay_weights(f.width, f.height, f.intr, f.R, t)
        else:
            both(lambda: api.recycle_blocks(tsdf), lambda: cpu.recycle_blocks(), op)
        assert_world_parity(tsdf, cpu, exact_pool=True)
        rep = tsdf.sync()
        assert rep.live_blocks == cpu.allocated_block_count() and rep.next_fresh == cpu.next_fresh(), op
        assert np.array_equal(tsdf.free_list(), cpu.free_list()), op
        if esdf is not None and rng.random_sample() < esdf_every:
            api.build_esdf(tsdf, esdf.config, esdf)
            site, dist, _ = esdf.download(d2=False)
            mask0, has0, site0, dist0 = cpu.build_esdf(sc.esdf_origin, sc.esdf_dims, sc.esdf_voxel)
            assert esdf.has_sites == has0 and int(esdf.report().seed_count) == int(mask0.sum()), op
            assert np.array_equal(site, site0) and same_bits(dist, dist0), f"ESDF rebuilt after {op} differs"
        steps += 1
    return steps


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--seconds", type=float, default=300.0)
    ap.add_argument("--seed", type=int, default=1)
    args = ap.parse_args()
    oracle = cpu_checkers.oracle()
    rng = np.random.RandomState(args.seed)
    t0 = time.time()
    worlds = steps = 0
    while time.time() - t0 < args.seconds:
        steps += one_world(oracle, rng)
        worlds += 1
        if worlds % 50 == 0:
            print(f"{worlds} worlds, {steps} operations ok ({time.time() - t0:.0f} s)", flush=True)
    print(f"lifecycle fuzz ok: {worlds} worlds, {steps} operations, seed {args.seed}")


if __name__ == "__main__":
    main()
