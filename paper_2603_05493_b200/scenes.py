"""Synthetic scenes for the BASELINE.json configurations.

Everything is generated once on the host with numpy and handed, as the same buffers, to the
CUDA path and to the CPU checkers, so no device-side transcendental can make the two disagree.
Camera: 640x480 pinhole, fx = fy = 525, cx = 319.5, cy = 239.5.
"""
from __future__ import annotations

from dataclasses import dataclass, field
from typing import List, Tuple

import numpy as np

WIDTH, HEIGHT = 640, 480
INTRINSICS = (525.0, 525.0, 319.5, 239.5)  # fx, fy, cx, cy


@dataclass
class Frame:
    depth: np.ndarray  # float32 [H, W], range along the optical axis; 0/NaN/inf/negative invalid
    R: np.ndarray      # float64 [3, 3] camera-to-world rotation
    t: np.ndarray      # float64 [3]    camera-to-world translation
    width: int = WIDTH
    height: int = HEIGHT
    intr: Tuple[float, float, float, float] = INTRINSICS


@dataclass
class Cuboid:
    R: np.ndarray
    t: np.ndarray
    half_extents: np.ndarray


@dataclass
class Sphere:
    center: np.ndarray
    radius: float


@dataclass
class Mesh:
    """Closed indexed triangle mesh in the world frame, outward counter-clockwise triangles."""
    vertices: np.ndarray   # float64 [V, 3]
    triangles: np.ndarray  # int32 [T, 3]


@dataclass
class Scene:
    name: str
    tsdf_voxel: float
    capacity: int
    esdf_origin: np.ndarray
    esdf_dims: Tuple[int, int, int]
    esdf_voxel: float
    frames: List[Frame] = field(default_factory=list)
    cuboids: List[Cuboid] = field(default_factory=list)
    spheres: List[Sphere] = field(default_factory=list)
    meshes: List[Mesh] = field(default_factory=list)

    @property
    def truncation(self) -> float:
        return 4.0 * self.tsdf_voxel

    @property
    def cells(self) -> int:
        return int(self.esdf_dims[0]) * int(self.esdf_dims[1]) * int(self.esdf_dims[2])


def rot_z(a: float) -> np.ndarray:
    c, s = np.cos(a), np.sin(a)
    return np.array([[c, -s, 0.0], [s, c, 0.0], [0.0, 0.0, 1.0]])


def rot_y(a: float) -> np.ndarray:
    c, s = np.cos(a), np.sin(a)
    return np.array([[c, 0.0, s], [0.0, 1.0, 0.0], [-s, 0.0, c]])


def _pixel_grid(width=WIDTH, height=HEIGHT):
    px = np.arange(width, dtype=np.float32)[None, :]
    py = np.arange(height, dtype=np.float32)[:, None]
    return px, py


def wavy_depth(base: float, amp: float, phase: float = 0.0, width=WIDTH, height=HEIGHT) -> np.ndarray:
    """base + amp * sin(0.02 px + phase) * cos(0.03 py), all in float32."""
    px, py = _pixel_grid(width, height)
    d = np.float32(base) + np.float32(amp) * np.sin(np.float32(0.02) * px + np.float32(phase)) * np.cos(
        np.float32(0.03) * py)
    return np.ascontiguousarray(d.astype(np.float32))


def punch_invalid(depth: np.ndarray, fraction=0.05, seed=11) -> np.ndarray:
    """Set a seeded fraction of pixels to the invalid encodings (0, NaN, -1, +inf)."""
    rng = np.random.RandomState(seed)
    out = depth.copy().reshape(-1)
    idx = rng.choice(out.size, int(out.size * fraction), replace=False)
    codes = np.array([0.0, np.nan, -1.0, np.inf], np.float32)
    out[idx] = codes[rng.randint(0, 4, idx.size)]
    return out.reshape(depth.shape)


def _cuboid(center, half_extents, yaw=0.0) -> Cuboid:
    return Cuboid(rot_z(yaw), np.asarray(center, np.float64), np.asarray(half_extents, np.float64))


def box_mesh(center, half_extents, R=None) -> Mesh:
    """The 12-triangle surface of a cuboid (corner k = signs (k&1, k&2, k&4), as stamp_primitive enumerates them)."""
    he = np.asarray(half_extents, np.float64)
    R = np.eye(3) if R is None else np.asarray(R, np.float64)
    corners = np.array([[(1 if k & 1 else -1), (1 if k & 2 else -1), (1 if k & 4 else -1)] for k in range(8)], np.float64)
    verts = (corners * he) @ R.T + np.asarray(center, np.float64)
    quads = [(0, 4, 6, 2), (1, 3, 7, 5), (0, 1, 5, 4), (2, 6, 7, 3), (0, 2, 3, 1), (4, 5, 7, 6)]  # -x +x -y +y -z +z
    tris = [t for a, b, c, d in quads for t in ((a, b, c), (a, c, d))]
    return Mesh(np.ascontiguousarray(verts), np.array(tris, np.int32))


def icosphere(center, radius: float, subdivisions: int = 2) -> Mesh:
    """Icosahedron subdivided `subdivisions` times and pushed onto the sphere: 20 * 4^s triangles."""
    g = (1.0 + np.sqrt(5.0)) / 2.0
    verts = [(-1, g, 0), (1, g, 0), (-1, -g, 0), (1, -g, 0), (0, -1, g), (0, 1, g), (0, -1, -g), (0, 1, -g),
             (g, 0, -1), (g, 0, 1), (-g, 0, -1), (-g, 0, 1)]
    verts = [np.asarray(v, np.float64) / np.sqrt(1.0 + g * g) for v in verts]
    tris = [(0, 11, 5), (0, 5, 1), (0, 1, 7), (0, 7, 10), (0, 10, 11), (1, 5, 9), (5, 11, 4), (11, 10, 2), (10, 7, 6),
            (7, 1, 8), (3, 9, 4), (3, 4, 2), (3, 2, 6), (3, 6, 8), (3, 8, 9), (4, 9, 5), (2, 4, 11), (6, 2, 10),
            (8, 6, 7), (9, 8, 1)]
    for _ in range(subdivisions):
        mid, out = {}, []

        def midpoint(i, j):
            key = (min(i, j), max(i, j))
            if key not in mid:
                m = verts[i] + verts[j]
                verts.append(m / np.sqrt(m @ m))
                mid[key] = len(verts) - 1
            return mid[key]

        for a, b, c in tris:
            ab, bc, ca = midpoint(a, b), midpoint(b, c), midpoint(c, a)
            out += [(a, ab, ca), (b, bc, ab), (c, ca, bc), (ab, bc, ca)]
        tris = out
    v = np.asarray(verts, np.float64) * float(radius) + np.asarray(center, np.float64)
    return Mesh(np.ascontiguousarray(v), np.array(tris, np.int32))


def config1(variant: str = "flat", invalid: bool = False) -> Scene:
    """640x480 frame into a 1 m^3 workspace at 1 cm (CPU-runnable oracle case)."""
    depth = np.full((HEIGHT, WIDTH), 1.0, np.float32) if variant == "flat" else wavy_depth(1.0, 0.05)
    if invalid:
        depth = punch_invalid(depth)
    scene = Scene("cfg1-" + variant, 0.01, 65536, np.zeros(3), (100, 100, 100), 0.01)
    scene.frames.append(Frame(depth, np.eye(3), np.array([0.5, 0.5, -0.2])))
    return scene


def config2(dims=(400, 200, 200)) -> Scene:
    """2 m^3 (2 x 1 x 1 m) workspace at 5 mm, one depth camera + three cuboids."""
    scene = Scene("cfg2", 0.005, 131072, np.zeros(3), tuple(dims), 0.005)
    scene.frames.append(Frame(wavy_depth(1.2, 0.1), np.eye(3), np.array([1.0, 0.5, -0.3])))
    scene.cuboids += [
        _cuboid((0.5, 0.5, 0.3), (0.15, 0.1, 0.2)),
        _cuboid((1.4, 0.3, 0.5), (0.1, 0.2, 0.1)),
        _cuboid((1.0, 0.7, 0.2), (0.3, 0.05, 0.15), yaw=0.5),
    ]
    return scene


def config3(dims=(500, 500, 500)) -> Scene:
    """1 m^3 manipulation workspace at 2 mm, four depth cameras + two cuboids."""
    scene = Scene("cfg3", 0.002, 262144, np.zeros(3), tuple(dims), 0.002)
    centre = np.array([0.5, 0.5, 0.5])
    for k in range(4):
        R = rot_y(k * np.pi / 2.0)
        fwd = R @ np.array([0.0, 0.0, 1.0])
        scene.frames.append(Frame(wavy_depth(0.7, 0.05, phase=float(k)), R, centre - 0.9 * fwd))
    scene.cuboids += [
        _cuboid((0.5, 0.1, 0.5), (0.4, 0.02, 0.4)),
        _cuboid((0.5, 0.4, 0.5), (0.05, 0.08, 0.05), yaw=0.3),
    ]
    return scene


def config4(n_queries=1_000_000) -> Tuple[Scene, np.ndarray]:
    """config2 + a sphere + a 1280-triangle mesh (mesh + cuboid + depth mixed scene), with Q uniform query points."""
    scene = config2()
    scene.name = "cfg4"
    scene.spheres.append(Sphere(np.array([1.6, 0.7, 0.6]), 0.12))
    scene.meshes.append(icosphere((0.35, 0.8, 0.7), 0.14, 3))
    rng = np.random.RandomState(7)
    extent = np.array(scene.esdf_dims, np.float64) * scene.esdf_voxel
    points = scene.esdf_origin + rng.random_sample((n_queries, 3)) * extent
    return scene, np.ascontiguousarray(points)


def config5_env(env: int, dims=(300, 200, 200)) -> Scene:
    """One of 128 independent environments: 1.5 x 1 x 1 m at 5 mm, jittered cuboids."""
    rng = np.random.RandomState(1000 + env)
    scene = Scene(f"cfg5-env{env}", 0.005, 16384, np.zeros(3), tuple(dims), 0.005)
    scene.frames.append(Frame(wavy_depth(1.2, 0.1, phase=0.1 * (env % 16)), np.eye(3), np.array([0.75, 0.5, -0.3])))
    base = [((0.4, 0.5, 0.3), (0.15, 0.1, 0.2), 0.0), ((1.1, 0.3, 0.5), (0.1, 0.2, 0.1), 0.0),
            ((0.75, 0.7, 0.2), (0.3, 0.05, 0.15), 0.5)]
    for centre, he, yaw in base:
        jitter = (rng.random_sample(3) - 0.5) * 0.1
        scene.cuboids.append(_cuboid(np.asarray(centre) + jitter, he, yaw + (rng.random_sample() - 0.5) * 0.4))
    return scene


def small_scene(seed: int, dims=(48, 40, 36), tsdf_voxel=0.02, ratio=1.0, origin=(0.0, 0.0, 0.0),
                width=96, height=72, n_cuboids=2, n_spheres=1, capacity=4096) -> Scene:
    """Seeded small mixed scene (depth + cuboids + spheres) for parity tests that finish in seconds."""
    rng = np.random.RandomState(seed)
    ve = tsdf_voxel * ratio
    extent = np.array(dims, np.float64) * ve
    origin = np.asarray(origin, np.float64)
    scene = Scene(f"small-{seed}", tsdf_voxel, capacity, origin, tuple(dims), ve)
    fx = fy = 0.82 * width
    intr = (fx, fy, (width - 1) / 2.0, (height - 1) / 2.0)
    px, py = _pixel_grid(width, height)
    base = 0.6 * extent[2] + 0.35
    depth = (np.float32(base) + np.float32(0.08) * np.sin(np.float32(0.11) * px + np.float32(seed)) * np.cos(
        np.float32(0.07) * py)).astype(np.float32)
    depth = punch_invalid(depth, 0.03, seed + 5)
    yaw = (rng.random_sample() - 0.5) * 0.3
    cam_t = origin + np.array([0.5 * extent[0], 0.5 * extent[1], -0.3])
    scene.frames.append(Frame(depth, rot_y(yaw), cam_t, width, height, intr))
    for _ in range(n_cuboids):
        c = origin + rng.random_sample(3) * extent
        he = 0.04 + rng.random_sample(3) * 0.15 * extent.min()
        scene.cuboids.append(_cuboid(c, he, yaw=(rng.random_sample() - 0.5) * 2.0))
    for _ in range(n_spheres):
        c = origin + rng.random_sample(3) * extent
        scene.spheres.append(Sphere(c, 0.05 + rng.random_sample() * 0.12 * extent.min()))
    return scene
