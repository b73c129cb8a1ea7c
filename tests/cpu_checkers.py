"""ctypes bindings for the two CPU checkers (TEST INFRASTRUCTURE ONLY).

  oracle()     -> oracle/liboracle.so       prefix ko_  (C restatement, oracle/ks_oracle.c)
  reference()  -> oracle/_ref/libks_ref.so  prefix kr_  (the reference's own headers, unmodified)

Both export the interface declared in oracle/ks_oracle_api.h, so one wrapper class drives
either.  Only tests/, __graft_entry__.smoke() and bench.py's CPU-baseline legs import this.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent.parent
ORACLE_DIR = ROOT / "oracle"

_f64p = np.ctypeslib.ndpointer(np.float64, flags="C_CONTIGUOUS")
_f32p = np.ctypeslib.ndpointer(np.float32, flags="C_CONTIGUOUS")
_i32p = np.ctypeslib.ndpointer(np.int32, flags="C_CONTIGUOUS")
_u8p = np.ctypeslib.ndpointer(np.uint8, flags="C_CONTIGUOUS")


def _vec(a, n, dtype=np.float64):
    out = np.ascontiguousarray(np.asarray(a, dtype=dtype).reshape(-1))
    assert out.size == n, (out.size, n)
    return out


class CheckerError(RuntimeError):
    pass


class CpuChecker:
    """One loaded checker library (`ko_` or `kr_` prefix)."""

    def __init__(self, path: Path, prefix: str, kind: str):
        self.kind = kind
        self.path = Path(path)
        self.lib = C.CDLL(str(path))
        self.p = prefix
        L = self.lib
        VP = C.c_void_p

        def fn(name, restype, *argtypes):
            f = getattr(L, prefix + name)
            f.restype = restype
            f.argtypes = list(argtypes)
            return f

        self._last_error = fn("last_error", C.c_char_p)
        self._create = fn("tsdf_create", VP, _f64p, C.c_int, C.c_int)
        self._destroy = fn("tsdf_destroy", None, VP)
        self._integrate = fn("integrate_depth", C.c_int, VP, _f32p, C.c_int, C.c_int, _f64p, _f64p, _f64p)
        self._stamp_cuboid = fn("stamp_cuboid", C.c_int, VP, _f64p, _f64p, _f64p)
        self._stamp_sphere = fn("stamp_sphere", C.c_int, VP, _f64p, C.c_double)
        # mesh stamping exists in the restatement only (the reference has none: SPEC.md:8)
        self.has_mesh = hasattr(L, prefix + "stamp_mesh")
        if self.has_mesh:
            self._stamp_mesh = fn("stamp_mesh", C.c_int, VP, _f64p, C.c_int, _i32p, C.c_int)
            self._mesh_sdf = fn("mesh_sdf", C.c_int, _f64p, C.c_int, _i32p, C.c_int, _f64p, C.c_int64, _f64p)
        self._decay = fn("decay_weights", None, VP, C.c_int, C.c_int, _f64p, _f64p, _f64p)
        self._recycle = fn("recycle_blocks", C.c_int, VP)
        self._count = fn("allocated_block_count", C.c_int, VP)
        self._available = fn("available", C.c_int, VP)
        self._next_fresh = fn("next_fresh", C.c_int, VP)
        self._slot_count = fn("slot_count", C.c_int, VP)
        self._find = fn("find", C.c_int, VP, C.c_int, C.c_int, C.c_int)
        self._free_list = fn("free_list", C.c_int, VP, _i32p, C.c_int)
        self._export = fn("export_blocks", C.c_int, VP, _i32p, _i32p, C.c_int)
        self._channels = fn("block_channels", None, VP, C.c_int, _f64p, _f64p, _f64p)
        self._query_tsdf = fn("query_tsdf", None, VP, _f64p, C.c_int64, C.c_int, _f64p, _u8p)
        self._seed_gather = fn("seed_gather", None, VP, _f64p, _i32p, C.c_double, _u8p)
        self._seed_scatter = fn("seed_scatter", None, VP, _f64p, _i32p, C.c_double, _u8p)
        self._propagate = fn("propagate", C.c_int, _u8p, C.c_int64, _i32p, C.c_double, _i32p, _f64p)
        self._recover = fn("recover_signs", None, VP, _f64p, _i32p, C.c_double, C.c_int, _i32p, _f64p)
        self._query_esdf = fn("query_esdf", None, _f64p, _i32p, C.c_double, C.c_int, _f64p, _f64p,
                              C.c_int64, _f64p, _f64p, _u8p)

        self._timed_update = fn("timed_update", C.c_int64, VP, C.c_int, _f32p, C.c_int, C.c_int, _f64p, _f64p, _f64p,
                                C.c_int, _f64p, _f64p, _f64p, C.c_int, _f64p, _f64p, _f64p, _i32p, C.c_double,
                                _f64p, _f64p)

        self._coll_static = fn("scene_collision_static", None, _f64p, _i32p, C.c_double, C.c_int, _f64p, _f64p, _f64p,
                               C.c_int64, C.c_double, _f64p, _f64p)
        self._coll_swept = fn("scene_collision_swept", None, _f64p, _i32p, C.c_double, C.c_int, _f64p, _f64p, _f64p,
                              _f64p, C.c_int, C.c_int, C.c_double, C.c_double, C.c_int, _f64p, _f64p, _f64p, _f64p)

    def scene_collision_static(self, origin, dims, voxel_size, has_sites, distance, centers, radii, margin=0.025):
        """collision.hpp:130-152 -> (max_penetration, worst_sphere, cost, gradient[n,3])"""
        c = np.ascontiguousarray(centers, np.float64).reshape(-1, 3)
        r = np.ascontiguousarray(radii, np.float64).reshape(-1)
        rep = np.zeros(3, np.float64)
        grad = np.zeros((max(len(r), 1), 3), np.float64)
        self._coll_static(_vec(origin, 3), _vec(dims, 3, np.int32), float(voxel_size), int(has_sites),
                          np.ascontiguousarray(distance, np.float64), c, r, len(r), float(margin), rep, grad)
        return float(rep[0]), int(rep[1]), float(rep[2]), grad[:len(r)]

    def scene_collision_swept(self, origin, dims, voxel_size, has_sites, distance, centers, radii, velocities,
                              margin=0.025, dt=1.0, max_checks=10000):
        """collision.hpp:177-239 -> (reports[T,3], center_grad, next_grad, velocity_grad), each [T,S,3]"""
        c = np.ascontiguousarray(centers, np.float64)
        T, S = c.shape[0], c.shape[1]
        v = np.ascontiguousarray(velocities, np.float64).reshape(T, S, 3)
        r = np.ascontiguousarray(radii, np.float64).reshape(S)
        rep = np.zeros((T, 3), np.float64)
        g0, g1, g2 = (np.zeros((T, S, 3), np.float64) for _ in range(3))
        self._coll_swept(_vec(origin, 3), _vec(dims, 3, np.int32), float(voxel_size), int(has_sites),
                         np.ascontiguousarray(distance, np.float64), c.reshape(-1), r, v.reshape(-1), T, S, float(margin),
                         float(dt), int(max_checks), rep.reshape(-1), g0.reshape(-1), g1.reshape(-1), g2.reshape(-1))
        return rep, g0, g1, g2

    def timed_update(self, tsdf: "CheckerTsdf", scene, dims=None):
        """One full update of `scene` timed inside the library; returns (seconds per stage dict, seeds, checksum)."""
        frames = scene.frames
        f0 = frames[0]
        depth = np.ascontiguousarray(np.stack([f.depth.reshape(-1) for f in frames]).astype(np.float32).reshape(-1))
        R = np.ascontiguousarray(np.stack([np.asarray(f.R, np.float64).reshape(9) for f in frames]).reshape(-1))
        t = np.ascontiguousarray(np.stack([np.asarray(f.t, np.float64).reshape(3) for f in frames]).reshape(-1))
        z3, z9, z1 = np.zeros(3), np.zeros(9), np.zeros(1)
        cR = np.ascontiguousarray(np.concatenate([np.asarray(c.R, np.float64).reshape(9) for c in scene.cuboids] or [z9]))
        ct = np.ascontiguousarray(np.concatenate([np.asarray(c.t, np.float64).reshape(3) for c in scene.cuboids] or [z3]))
        che = np.ascontiguousarray(np.concatenate([np.asarray(c.half_extents, np.float64).reshape(3) for c in scene.cuboids] or [z3]))
        sc = np.ascontiguousarray(np.concatenate([np.asarray(s.center, np.float64).reshape(3) for s in scene.spheres] or [z3]))
        sr = np.ascontiguousarray(np.array([s.radius for s in scene.spheres] or [0.0], np.float64))
        times = np.zeros(5, np.float64)
        checksum = np.zeros(1, np.float64)
        dims = _vec(scene.esdf_dims if dims is None else dims, 3, np.int32)
        seeds = self._timed_update(tsdf.h, len(frames), depth, f0.width, f0.height, _vec(f0.intr, 4), R, t,
                                   len(scene.cuboids), cR, ct, che, len(scene.spheres), sc, sr,
                                   _vec(scene.esdf_origin, 3), dims, float(scene.esdf_voxel), times, checksum)
        if seeds < 0:
            raise CheckerError(self.last_error())
        return dict(zip(("integrate", "stamp", "seed", "propagate", "signs"), times.tolist())), int(seeds), float(checksum[0])

    def last_error(self) -> str:
        return (self._last_error() or b"").decode()

    # --- TSDF ---------------------------------------------------------------------------
    def make_tsdf(self, voxel_size=0.01, truncation=None, alpha_time=0.99, alpha_frustum=0.5,
                  weight_threshold=0.5, capacity=8192, slot_count=0) -> "CheckerTsdf":
        if truncation is None:
            truncation = 4.0 * voxel_size
        cfg = np.array([voxel_size, truncation, alpha_time, alpha_frustum, weight_threshold], np.float64)
        handle = self._create(cfg, int(capacity), int(slot_count))
        if not handle:
            raise CheckerError(self.last_error())
        return CheckerTsdf(self, handle, voxel_size, truncation, capacity)

    # --- ESDF (stateless) ----------------------------------------------------------------
    def mesh_sdf(self, vertices, triangles, points):
        """Signed distance of a closed triangle mesh at `points` (restatement only, see has_mesh)."""
        v = np.ascontiguousarray(vertices, np.float64).reshape(-1)
        t = np.ascontiguousarray(triangles, np.int32).reshape(-1)
        pts = np.ascontiguousarray(points, np.float64).reshape(-1, 3)
        out = np.empty(len(pts), np.float64)
        if self._mesh_sdf(v, v.size // 3, t, t.size // 3, pts.reshape(-1), len(pts), out) != 0:
            raise CheckerError(self.last_error())
        return out

    def propagate(self, mask, dims, voxel_size):
        dims = _vec(dims, 3, np.int32)
        mask = np.ascontiguousarray(mask, np.uint8).reshape(-1)
        cells = int(dims[0]) * int(dims[1]) * int(dims[2])
        site = np.empty((max(cells, 1), 3), np.int32)
        dist = np.empty(max(cells, 1), np.float64)
        has = self._propagate(mask, mask.size, dims, float(voxel_size), site, dist)
        if has < 0:
            raise CheckerError(self.last_error())
        return bool(has), site[:cells], dist[:cells]

    def query_esdf(self, origin, dims, voxel_size, has_sites, distance, points):
        pts = np.ascontiguousarray(points, np.float64).reshape(-1, 3)
        n = pts.shape[0]
        d = np.empty(n, np.float64)
        g = np.empty((n, 3), np.float64)
        inside = np.empty(n, np.uint8)
        self._query_esdf(_vec(origin, 3), _vec(dims, 3, np.int32), float(voxel_size), int(has_sites),
                         np.ascontiguousarray(distance, np.float64), pts, n, d, g, inside)
        return d, g, inside.astype(bool)


class CheckerTsdf:
    def __init__(self, lib: CpuChecker, handle, voxel_size, truncation, capacity):
        self.lib = lib
        self.h = handle
        self.voxel_size = voxel_size
        self.truncation = truncation
        self.capacity = capacity

    def close(self):
        if self.h:
            self.lib._destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def integrate_depth(self, depth, width, height, intr, pose_R, pose_t) -> int:
        depth = np.ascontiguousarray(depth, np.float32).reshape(-1)
        assert depth.size == width * height
        k = self.lib._integrate(self.h, depth, width, height, _vec(intr, 4), _vec(pose_R, 9), _vec(pose_t, 3))
        if k < 0:
            raise CheckerError(self.lib.last_error())
        return k

    def stamp_cuboid(self, pose_R, pose_t, half_extents):
        if self.lib._stamp_cuboid(self.h, _vec(pose_R, 9), _vec(pose_t, 3), _vec(half_extents, 3)) != 0:
            raise CheckerError(self.lib.last_error())

    def stamp_sphere(self, center, radius):
        if self.lib._stamp_sphere(self.h, _vec(center, 3), float(radius)) != 0:
            raise CheckerError(self.lib.last_error())

    def stamp_mesh(self, vertices, triangles):
        v = np.ascontiguousarray(vertices, np.float64).reshape(-1)
        t = np.ascontiguousarray(triangles, np.int32).reshape(-1)
        if self.lib._stamp_mesh(self.h, v, v.size // 3, t, t.size // 3) != 0:
            raise CheckerError(self.lib.last_error())

    def decay_weights(self, width, height, intr, pose_R, pose_t):
        self.lib._decay(self.h, width, height, _vec(intr, 4), _vec(pose_R, 9), _vec(pose_t, 3))

    def recycle_blocks(self) -> int:
        return self.lib._recycle(self.h)

    def allocated_block_count(self) -> int:
        return self.lib._count(self.h)

    def available(self) -> int:
        return self.lib._available(self.h)

    def next_fresh(self) -> int:
        return self.lib._next_fresh(self.h)

    def slot_count(self) -> int:
        return self.lib._slot_count(self.h)

    def find(self, key) -> int:
        return self.lib._find(self.h, int(key[0]), int(key[1]), int(key[2]))

    def free_list(self):
        out = np.empty(max(self.capacity, 1), np.int32)
        n = self.lib._free_list(self.h, out, out.size)
        return out[:n].copy()

    def export_blocks(self):
        """(keys[L,3], pool[L]) of live blocks in slot order."""
        n = self.allocated_block_count()
        keys = np.empty((max(n, 1), 3), np.int32)
        pool = np.empty(max(n, 1), np.int32)
        self.lib._export(self.h, keys, pool, n)
        return keys[:n], pool[:n]

    def block_channels(self, pool: int):
        s = np.empty(512, np.float64)
        w = np.empty(512, np.float64)
        g = np.empty(512, np.float64)
        self.lib._channels(self.h, int(pool), s, w, g)
        return s, w, g

    def blocks_by_key(self):
        """dict key(tuple) -> (pool, sum, wt, geom), the by-key parity view."""
        keys, pool = self.export_blocks()
        return {tuple(int(c) for c in k): (int(p),) + self.block_channels(int(p)) for k, p in zip(keys, pool)}

    def query_tsdf(self, points, geom_only=False):
        pts = np.ascontiguousarray(points, np.float64).reshape(-1, 3)
        n = pts.shape[0]
        out = np.empty(n, np.float64)
        valid = np.empty(n, np.uint8)
        self.lib._query_tsdf(self.h, pts, n, int(geom_only), out, valid)
        return out, valid.astype(bool)

    def seed_gather(self, origin, dims, voxel_size):
        dims = _vec(dims, 3, np.int32)
        mask = np.empty(int(dims[0]) * int(dims[1]) * int(dims[2]), np.uint8)
        self.lib._seed_gather(self.h, _vec(origin, 3), dims, float(voxel_size), mask)
        return mask

    def seed_scatter(self, origin, dims, voxel_size):
        dims = _vec(dims, 3, np.int32)
        mask = np.empty(int(dims[0]) * int(dims[1]) * int(dims[2]), np.uint8)
        self.lib._seed_scatter(self.h, _vec(origin, 3), dims, float(voxel_size), mask)
        return mask

    def recover_signs(self, origin, dims, voxel_size, has_sites, site, distance):
        out = np.array(distance, np.float64, copy=True).reshape(-1)
        self.lib._recover(self.h, _vec(origin, 3), _vec(dims, 3, np.int32), float(voxel_size), int(has_sites),
                          np.ascontiguousarray(site, np.int32).reshape(-1), out)
        return out

    def build_esdf(self, origin, dims, voxel_size, seeding="gather"):
        """seed -> propagate -> recover_signs (esdf.hpp:323-327)."""
        mask = (self.seed_gather if seeding == "gather" else self.seed_scatter)(origin, dims, voxel_size)
        has, site, dist = self.lib.propagate(mask, dims, voxel_size)
        dist = self.recover_signs(origin, dims, voxel_size, has, site, dist)
        return mask, has, site, dist


def build_checkers(quiet=True):
    """(Re)build liboracle.so and, when /root/reference is mounted, _ref/libks_ref.so."""
    subprocess.run(["make", "-C", str(ORACLE_DIR), "all"], check=True,
                   stdout=subprocess.DEVNULL if quiet else None)


_cache = {}


def oracle() -> CpuChecker:
    if "o" not in _cache:
        path = ORACLE_DIR / "liboracle.so"
        if not path.exists():
            build_checkers()
        _cache["o"] = CpuChecker(path, "ko_", "port")
    return _cache["o"]


def reference_available() -> bool:
    return (ORACLE_DIR / "_ref" / "libks_ref.so").exists()


def reference() -> CpuChecker:
    if "r" not in _cache:
        path = ORACLE_DIR / "_ref" / "libks_ref.so"
        if not path.exists() and os.path.isdir("/root/reference"):
            build_checkers()
        _cache["r"] = CpuChecker(path, "kr_", "reference")
    return _cache["r"]
