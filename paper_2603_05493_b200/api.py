"""Host-side mirror of the reference's ks:: perception API over the ks_b200 C ABI.

Function names, argument meaning and error behaviour follow
/root/reference/proj/include/ks/sdf_world.hpp and esdf.hpp:

    make_tsdf_config, make_tsdf, integrate_depth, stamp_primitive, decay_weights, recycle_blocks,
    query_tsdf, query_tsdf_geom, allocated_block_count, seed_gather, seed_scatter, propagate,
    recover_signs, build_esdf, query

Everything here is a thin ctypes call into libks_b200.so (include/ks_b200.h).  There is no CPU
implementation: loading fails loudly when the library is missing, and every compute call fails with
KS_ERR_CUDA when no device is present.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field
from pathlib import Path
from typing import Optional, Sequence, Tuple

import numpy as np

PKG = Path(__file__).resolve().parent
LIB_PATH = PKG / "libks_b200.so"

KS_OK, KS_ERR_INVALID, KS_ERR_POOL_EXHAUSTED, KS_ERR_TABLE_FULL, KS_ERR_CUDA, KS_ERR_RANGE, KS_ERR_UNSUPPORTED = range(7)


class ValidationError(RuntimeError):
    """ks::ValidationError (core.hpp:36-39)."""


class CudaError(RuntimeError):
    pass


class TsdfConfigC(C.Structure):
    _fields_ = [("voxel_size", C.c_double), ("truncation", C.c_double), ("alpha_time", C.c_double),
                ("alpha_frustum", C.c_double), ("weight_threshold", C.c_double), ("capacity", C.c_int32),
                ("slot_count", C.c_int32)]


class CameraC(C.Structure):
    _fields_ = [("width", C.c_int32), ("height", C.c_int32), ("fx", C.c_double), ("fy", C.c_double),
                ("cx", C.c_double), ("cy", C.c_double), ("pose_R", C.c_double * 9), ("pose_t", C.c_double * 3)]


class EsdfConfigC(C.Structure):
    _fields_ = [("origin", C.c_double * 3), ("nx", C.c_int32), ("ny", C.c_int32), ("nz", C.c_int32),
                ("voxel_size", C.c_double), ("seeding", C.c_int32)]


class PrimitiveC(C.Structure):  # ks_primitive
    _fields_ = [("kind", C.c_int32), ("reserved", C.c_int32), ("pose_R", C.c_double * 9), ("pose_t", C.c_double * 3),
                ("half_extents", C.c_double * 3), ("center", C.c_double * 3), ("radius", C.c_double)]


class TsdfReportC(C.Structure):
    _fields_ = [(n, C.c_int32) for n in ("status", "blocks_touched", "required", "available", "live_blocks",
                                          "next_fresh", "free_count", "recycled")]


class CollisionReportC(C.Structure):
    _fields_ = [("max_penetration", C.c_double), ("cost", C.c_double), ("worst_sphere", C.c_int32), ("reserved", C.c_int32)]


class EsdfReportC(C.Structure):
    _fields_ = [("status", C.c_int32), ("has_sites", C.c_int32), ("signs_recovered", C.c_int32),
                ("seed_count", C.c_int64)]


_lib = None

# every symbol include/ks_b200.h declares (tests check the .so exports exactly these)
ABI_SYMBOLS = [
    "ks_last_error", "ks_version", "ks_device_count", "ks_kernel_launch_count", "ks_stream_create",
    "ks_stream_destroy", "ks_stream_sync", "ks_graph_begin_capture", "ks_graph_end_capture", "ks_graph_launch",
    "ks_graph_node_count", "ks_graph_destroy", "ks_tsdf_config_init", "ks_tsdf_create", "ks_tsdf_destroy",
    "ks_tsdf_set_stream", "ks_tsdf_get_stream", "ks_tsdf_integrate_depth", "ks_tsdf_stage_frame",
    "ks_tsdf_upload_frame_async", "ks_tsdf_integrate_async", "ks_tsdf_stage_frame_slot", "ks_tsdf_frame_buffer", "ks_host_alloc", "ks_host_free",
    "ks_tsdf_upload_frame_slot_async", "ks_tsdf_integrate_slot_async", "ks_tsdf_stamp_cuboid", "ks_tsdf_stamp_sphere",
    "ks_tsdf_stamp_cuboid_async", "ks_tsdf_stamp_sphere_async", "ks_mesh_create", "ks_mesh_destroy",
    "ks_mesh_triangle_count", "ks_tsdf_stamp_mesh", "ks_tsdf_stamp_mesh_async", "ks_tsdf_decay_weights",
    "ks_tsdf_decay_weights_async", "ks_tsdf_recycle_blocks", "ks_tsdf_sync", "ks_tsdf_query",
    "ks_tsdf_allocated_block_count", "ks_tsdf_find", "ks_tsdf_export_blocks", "ks_tsdf_download_blocks",
    "ks_tsdf_free_list", "ks_tsdf_profile", "ks_tsdf_stage_ms", "ks_esdf_profile", "ks_esdf_stage_ms", "ks_esdf_create", "ks_esdf_destroy", "ks_esdf_set_stream", "ks_esdf_build",
    "ks_esdf_build_async", "ks_esdf_seed", "ks_esdf_propagate", "ks_esdf_recover_signs", "ks_esdf_sync", "ks_esdf_last_report", "ks_esdf_probe_summary_device_async",
    "ks_esdf_download", "ks_esdf_query", "ks_esdf_query_device_async", "ks_esdf_scene_collision_static",
    "ks_esdf_scene_collision_swept", "ks_tsdf_export_slots", "ks_tsdf_generation", "ks_esdf_generation",
    "ks_tsdf_stamp_batch", "ks_tsdf_stamp_batch_async",
    "ks_batch_create", "ks_batch_destroy", "ks_batch_size", "ks_batch_lanes", "ks_batch_tsdf", "ks_batch_esdf", "ks_batch_stream",
    "ks_batch_set_inputs", "ks_batch_set_probes", "ks_batch_set_first_env", "ks_batch_update_async", "ks_batch_update",
    "ks_batch_graph_kernels", "ks_batch_sync", "ks_batch_summary_device", "ks_partition_envs", "ks_nccl_unique_id",
    "ks_batch_attach_nccl", "ks_batch_attach_nccl_comm", "ks_batch_gathered_device", "ks_batch_gathered_rows", "ks_batch_gathered",
]


def load_library() -> C.CDLL:
    """Load libks_b200.so.  Fails loudly: there is no fallback implementation."""
    global _lib
    if _lib is not None:
        return _lib
    if not LIB_PATH.exists():
        raise ImportError(f"{LIB_PATH} is missing: run `python -m paper_2603_05493_b200.build` "
                          "(the perception path has no CPU implementation)")
    lib = C.CDLL(str(LIB_PATH))
    VP, I32, I64, D = C.c_void_p, C.c_int32, C.c_int64, C.c_double
    P = C.POINTER
    sig = {
        "ks_last_error": (C.c_char_p, []),
        "ks_version": (C.c_char_p, []),
        "ks_device_count": (C.c_int, []),
        "ks_kernel_launch_count": (I64, []),
        "ks_stream_create": (C.c_int, [P(VP)]),
        "ks_stream_destroy": (C.c_int, [VP]),
        "ks_stream_sync": (C.c_int, [VP]),
        "ks_graph_begin_capture": (C.c_int, [VP]),
        "ks_graph_end_capture": (C.c_int, [VP, P(VP)]),
        "ks_graph_launch": (C.c_int, [VP, VP]),
        "ks_graph_node_count": (C.c_int, [VP, P(I64), P(I64)]),
        "ks_graph_destroy": (None, [VP]),
        "ks_tsdf_config_init": (C.c_int, [D, P(TsdfConfigC)]),
        "ks_tsdf_create": (C.c_int, [P(TsdfConfigC), P(VP)]),
        "ks_tsdf_destroy": (None, [VP]),
        "ks_tsdf_set_stream": (C.c_int, [VP, VP]),
        "ks_tsdf_get_stream": (VP, [VP]),
        "ks_tsdf_integrate_depth": (C.c_int, [VP, P(CameraC), VP, P(I32)]),
        "ks_tsdf_stage_frame": (C.c_int, [VP, P(CameraC), VP]),
        "ks_tsdf_upload_frame_async": (C.c_int, [VP]),
        "ks_tsdf_stage_frame_slot": (C.c_int, [VP, I32, P(CameraC), VP]),
        "ks_tsdf_frame_buffer": (C.c_int, [VP, I32, I32, I32, P(VP)]),
        "ks_host_alloc": (C.c_int, [C.c_size_t, P(VP)]),
        "ks_host_free": (None, [VP]),
        "ks_tsdf_upload_frame_slot_async": (C.c_int, [VP, I32]),
        "ks_tsdf_integrate_slot_async": (C.c_int, [VP, I32]),
        "ks_tsdf_integrate_async": (C.c_int, [VP]),
        "ks_tsdf_stamp_cuboid": (C.c_int, [VP, VP, VP, VP]),
        "ks_tsdf_stamp_sphere": (C.c_int, [VP, VP, D]),
        "ks_tsdf_stamp_cuboid_async": (C.c_int, [VP, VP, VP, VP]),
        "ks_tsdf_stamp_sphere_async": (C.c_int, [VP, VP, D]),
        "ks_mesh_create": (C.c_int, [VP, I32, VP, I32, P(VP)]),
        "ks_mesh_destroy": (None, [VP]),
        "ks_mesh_triangle_count": (I32, [VP]),
        "ks_tsdf_stamp_mesh": (C.c_int, [VP, VP]),
        "ks_tsdf_stamp_mesh_async": (C.c_int, [VP, VP]),
        "ks_tsdf_decay_weights": (C.c_int, [VP, P(CameraC)]),
        "ks_tsdf_decay_weights_async": (C.c_int, [VP, P(CameraC)]),
        "ks_tsdf_recycle_blocks": (C.c_int, [VP, P(I32)]),
        "ks_tsdf_sync": (C.c_int, [VP, P(TsdfReportC)]),
        "ks_tsdf_query": (C.c_int, [VP, VP, I64, I32, VP, VP]),
        "ks_tsdf_allocated_block_count": (C.c_int, [VP, P(I32)]),
        "ks_tsdf_find": (C.c_int, [VP, VP, P(I32)]),
        "ks_tsdf_export_blocks": (C.c_int, [VP, VP, VP, I32, P(I32)]),
        "ks_tsdf_download_blocks": (C.c_int, [VP, VP, I32, VP, VP, VP]),
        "ks_tsdf_free_list": (C.c_int, [VP, VP, I32, P(I32)]),
        "ks_tsdf_profile": (C.c_int, [VP, I32]),
        "ks_tsdf_stage_ms": (C.c_int, [VP, P(C.c_float)]),
        "ks_esdf_profile": (C.c_int, [VP, I32]),
        "ks_esdf_stage_ms": (C.c_int, [VP, P(C.c_float)]),
        "ks_esdf_create": (C.c_int, [P(EsdfConfigC), P(VP)]),
        "ks_esdf_destroy": (None, [VP]),
        "ks_esdf_set_stream": (C.c_int, [VP, VP]),
        "ks_esdf_build": (C.c_int, [VP, VP]),
        "ks_esdf_build_async": (C.c_int, [VP, VP]),
        "ks_esdf_seed": (C.c_int, [VP, VP, I32, VP]),
        "ks_esdf_propagate": (C.c_int, [VP, VP, I64]),
        "ks_esdf_recover_signs": (C.c_int, [VP, VP]),
        "ks_esdf_sync": (C.c_int, [VP, P(EsdfReportC)]),
        "ks_esdf_last_report": (C.c_int, [VP, P(EsdfReportC)]),
        "ks_esdf_probe_summary_device_async": (C.c_int, [VP, VP, C.c_int64, C.c_double, C.c_double, VP]),
        "ks_esdf_download": (C.c_int, [VP, VP, VP, VP]),
        "ks_esdf_query": (C.c_int, [VP, VP, I64, VP, VP, VP]),
        "ks_esdf_query_device_async": (C.c_int, [VP, VP, I64, VP, VP, VP]),
        "ks_esdf_scene_collision_static": (C.c_int, [VP, VP, VP, I64, D, P(CollisionReportC), VP]),
        "ks_esdf_scene_collision_swept": (C.c_int, [VP, VP, VP, VP, I32, I32, D, D, I32, P(CollisionReportC), VP, VP, VP]),
        "ks_tsdf_export_slots": (C.c_int, [VP, VP, VP, VP, I32, P(I32)]),
        "ks_tsdf_generation": (C.c_uint64, [VP]),
        "ks_esdf_generation": (C.c_uint64, [VP]),
        "ks_tsdf_stamp_batch": (C.c_int, [VP, P(PrimitiveC), I32]),
        "ks_tsdf_stamp_batch_async": (C.c_int, [VP, P(PrimitiveC), I32]),
        "ks_batch_create": (C.c_int, [I32, P(TsdfConfigC), P(EsdfConfigC), I32, P(VP)]),
        "ks_batch_destroy": (None, [VP]),
        "ks_batch_size": (I32, [VP]),
        "ks_batch_lanes": (I32, [VP]),
        "ks_batch_tsdf": (VP, [VP, I32]),
        "ks_batch_esdf": (VP, [VP, I32]),
        "ks_batch_stream": (VP, [VP]),
        "ks_batch_set_inputs": (C.c_int, [VP, I32, I32, P(PrimitiveC), I32, P(VP), I32]),
        "ks_batch_set_probes": (C.c_int, [VP, I32, VP, I64, D]),
        "ks_batch_set_first_env": (C.c_int, [VP, I32]),
        "ks_batch_update_async": (C.c_int, [VP, I32]),
        "ks_batch_update": (C.c_int, [VP, I32]),
        "ks_batch_graph_kernels": (I64, [VP]),
        "ks_batch_sync": (C.c_int, [VP, P(TsdfReportC), P(EsdfReportC), VP]),
        "ks_batch_summary_device": (VP, [VP]),
        "ks_partition_envs": (C.c_int, [I32, I32, I32, P(I32), P(I32)]),
        "ks_nccl_unique_id": (C.c_int, [VP]),
        "ks_batch_attach_nccl": (C.c_int, [VP, VP, I32, I32, I32]),
        "ks_batch_attach_nccl_comm": (C.c_int, [VP, VP, I32, I32, I32]),
        "ks_batch_gathered_device": (VP, [VP]),
        "ks_batch_gathered_rows": (I32, [VP]),
        "ks_batch_gathered": (C.c_int, [VP, VP]),
    }
    assert sorted(sig) == sorted(ABI_SYMBOLS)
    for name, (res, args) in sig.items():
        f = getattr(lib, name)
        f.restype = res
        f.argtypes = args
    _lib = lib
    return lib


def last_error() -> str:
    return (load_library().ks_last_error() or b"").decode()


def _check(rc: int):
    if rc == KS_OK:
        return
    msg = last_error()
    if rc == KS_ERR_CUDA:
        raise CudaError(msg)
    raise ValidationError(msg)


def _ptr(a: Optional[np.ndarray]):
    return None if a is None else a.ctypes.data_as(C.c_void_p)


def _f64(a, n=None) -> np.ndarray:
    out = np.ascontiguousarray(np.asarray(a, np.float64).reshape(-1))
    if n is not None:
        assert out.size == n
    return out


def kernel_launch_count() -> int:
    return int(load_library().ks_kernel_launch_count())


# ---- value types mirroring the reference structs --------------------------------------------------

@dataclass
class TsdfConfig:  # sdf_world.hpp:38-54
    voxel_size: float = 0.01
    truncation: float = 0.04
    alpha_time: float = 0.99
    alpha_frustum: float = 0.5
    weight_threshold: float = 0.5
    capacity: int = 8192
    slot_count: int = 0


def make_tsdf_config(voxel_size: float) -> TsdfConfig:  # sdf_world.hpp:56-61
    return TsdfConfig(voxel_size=voxel_size, truncation=4.0 * voxel_size)


@dataclass
class DepthFrame:  # sdf_world.hpp:191-204
    width: int
    height: int
    fx: float
    fy: float
    cx: float
    cy: float
    pose_R: np.ndarray = field(default_factory=lambda: np.eye(3))
    pose_t: np.ndarray = field(default_factory=lambda: np.zeros(3))
    depth: Optional[np.ndarray] = None

    def camera(self) -> CameraC:
        cam = CameraC(int(self.width), int(self.height), float(self.fx), float(self.fy), float(self.cx), float(self.cy))
        cam.pose_R[:] = list(_f64(self.pose_R, 9))
        cam.pose_t[:] = list(_f64(self.pose_t, 3))
        return cam


@dataclass
class Cuboid:  # sdf_world.hpp:212-215
    pose_R: np.ndarray
    pose_t: np.ndarray
    half_extents: np.ndarray


@dataclass
class SphereShape:  # sdf_world.hpp:217-220
    center: np.ndarray
    radius: float


class TriangleMesh:
    """A closed, outward-oriented indexed triangle mesh (world frame) resident on the device.  No reference
    counterpart: see include/ks_b200.h "Triangle-mesh stamping"."""

    def __init__(self, vertices, triangles):
        self.lib = load_library()
        self.vertices = np.ascontiguousarray(vertices, np.float64).reshape(-1, 3)
        self.triangles = np.ascontiguousarray(triangles, np.int32).reshape(-1, 3)
        h = C.c_void_p()
        _check(self.lib.ks_mesh_create(_ptr(self.vertices), len(self.vertices), _ptr(self.triangles), len(self.triangles),
                                       C.byref(h)))
        self.h = h

    def triangle_count(self) -> int:
        return int(self.lib.ks_mesh_triangle_count(self.h))

    def close(self):
        if getattr(self, "h", None):
            self.lib.ks_mesh_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


@dataclass
class EsdfConfig:  # esdf.hpp:35-54
    origin: Sequence[float] = (0.0, 0.0, 0.0)
    nx: int = 1
    ny: int = 1
    nz: int = 1
    voxel_size: float = 0.01
    seeding: str = "gather"

    def cell_count(self) -> int:
        return int(self.nx) * int(self.ny) * int(self.nz)


@dataclass
class EsdfSample:  # esdf.hpp:329-333 (batched)
    distance: np.ndarray
    gradient: np.ndarray
    inside: np.ndarray


# ---- handles -------------------------------------------------------------------------------------

class SparseTsdf:
    """ks::SparseTsdf (sdf_world.hpp:206-210) living in HBM."""

    def __init__(self, config: TsdfConfig, stream: Optional[int] = None):
        self.lib = load_library()
        self.config = config
        c = TsdfConfigC(config.voxel_size, config.truncation, config.alpha_time, config.alpha_frustum,
                        config.weight_threshold, int(config.capacity), int(config.slot_count))
        h = C.c_void_p()
        _check(self.lib.ks_tsdf_create(C.byref(c), C.byref(h)))
        self.h = h
        if stream is not None:
            _check(self.lib.ks_tsdf_set_stream(self.h, C.c_void_p(stream)))

    @classmethod
    def _borrowed(cls, handle, config: "TsdfConfig", owner) -> "SparseTsdf":
        """A view of a world owned by something else (an EnvBatch): same methods, never destroyed from here."""
        self = cls.__new__(cls)
        self.lib, self.config, self.h, self._owner = load_library(), config, C.c_void_p(handle), owner
        return self

    def close(self):
        if getattr(self, "h", None):
            if getattr(self, "_owner", None) is None:
                self.lib.ks_tsdf_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def frame_buffer(self, width: int, height: int, slot: int = 0) -> np.ndarray:
        """The slot's page-locked staging area as a (height, width) float32 array: pixels written here and staged
        with this very array skip the staging copy."""
        out = C.c_void_p()
        _check(self.lib.ks_tsdf_frame_buffer(self.h, slot, width, height, C.byref(out)))
        buf = (C.c_float * (width * height)).from_address(out.value)
        return np.frombuffer(buf, dtype=np.float32).reshape(height, width)

    # capturable pieces
    def stage_frame(self, frame: DepthFrame, slot: int = 0):
        depth = np.ascontiguousarray(frame.depth, np.float32).reshape(-1)
        if depth.size != frame.width * frame.height:
            raise ValidationError("depth frame: depth buffer size mismatch")  # sdf_world.hpp:200-201
        cam = frame.camera()
        _check(self.lib.ks_tsdf_stage_frame_slot(self.h, slot, C.byref(cam), _ptr(depth)))

    def upload_frame_async(self, slot: int = 0):
        _check(self.lib.ks_tsdf_upload_frame_slot_async(self.h, slot))

    def integrate_async(self, slot: int = 0):
        _check(self.lib.ks_tsdf_integrate_slot_async(self.h, slot))

    def stamp_async(self, primitive):
        if isinstance(primitive, TriangleMesh):
            _check(self.lib.ks_tsdf_stamp_mesh_async(self.h, primitive.h))
        elif isinstance(primitive, Cuboid):
            R, t, he = _f64(primitive.pose_R, 9), _f64(primitive.pose_t, 3), _f64(primitive.half_extents, 3)
            _check(self.lib.ks_tsdf_stamp_cuboid_async(self.h, _ptr(R), _ptr(t), _ptr(he)))
        else:
            c = _f64(primitive.center, 3)
            _check(self.lib.ks_tsdf_stamp_sphere_async(self.h, _ptr(c), float(primitive.radius)))

    def stamp_batch_async(self, primitives):
        """All cuboids / spheres of an update in three launches (ks_tsdf_stamp_batch_async): same world as the calls one by one."""
        arr = _primitive_array(primitives)
        _check(self.lib.ks_tsdf_stamp_batch_async(self.h, arr, len(primitives)))

    def sync(self) -> TsdfReportC:
        rep = TsdfReportC()
        _check(self.lib.ks_tsdf_sync(self.h, C.byref(rep)))
        return rep

    def profile(self, enable=True):
        _check(self.lib.ks_tsdf_profile(self.h, int(enable)))

    def stage_ms(self):
        """{discover, allocate, integrate} of the last integrate, {candidates+allocate, stamp} of the last stamp."""
        out = (C.c_float * 5)()
        _check(self.lib.ks_tsdf_stage_ms(self.h, out))
        return dict(zip(("discover", "allocate", "integrate", "stamp_candidates", "stamp_blocks"), list(out)))

    # parity views
    def export_blocks(self) -> Tuple[np.ndarray, np.ndarray]:
        n = C.c_int32()
        _check(self.lib.ks_tsdf_export_blocks(self.h, None, None, 0, C.byref(n)))
        keys = np.empty((max(n.value, 1), 3), np.int32)
        pool = np.empty(max(n.value, 1), np.int32)
        _check(self.lib.ks_tsdf_export_blocks(self.h, _ptr(keys), _ptr(pool), n.value, C.byref(n)))
        return keys[:n.value], pool[:n.value]

    def download_blocks(self, pools) -> Tuple[np.ndarray, np.ndarray, np.ndarray]:
        pools = np.ascontiguousarray(pools, np.int32)
        n = pools.size
        s, w, g = (np.empty((max(n, 1), 512), np.float64) for _ in range(3))
        _check(self.lib.ks_tsdf_download_blocks(self.h, _ptr(pools), n, _ptr(s), _ptr(w), _ptr(g)))
        return s[:n], w[:n], g[:n]

    def find(self, key) -> int:
        k = np.ascontiguousarray(key, np.int32)
        out = C.c_int32()
        _check(self.lib.ks_tsdf_find(self.h, _ptr(k), C.byref(out)))
        return out.value

    def free_list(self) -> np.ndarray:
        out = np.empty(max(self.config.capacity, 1), np.int32)
        n = C.c_int32()
        _check(self.lib.ks_tsdf_free_list(self.h, _ptr(out), out.size, C.byref(n)))
        return out[:n.value].copy()


class DenseEsdf:
    """ks::DenseEsdf (esdf.hpp:58-64) living in HBM; site/distance are downloaded on demand."""

    def __init__(self, config: EsdfConfig, stream: Optional[int] = None):
        self.lib = load_library()
        self.config = config
        c = EsdfConfigC()
        c.origin[:] = [float(v) for v in config.origin]
        c.nx, c.ny, c.nz = int(config.nx), int(config.ny), int(config.nz)
        c.voxel_size = float(config.voxel_size)
        c.seeding = 1 if config.seeding == "gather" else 0
        h = C.c_void_p()
        _check(self.lib.ks_esdf_create(C.byref(c), C.byref(h)))
        self.h = h
        if stream is not None:
            _check(self.lib.ks_esdf_set_stream(self.h, C.c_void_p(stream)))

    @classmethod
    def _borrowed(cls, handle, config: "EsdfConfig", owner) -> "DenseEsdf":
        self = cls.__new__(cls)
        self.lib, self.config, self.h, self._owner = load_library(), config, C.c_void_p(handle), owner
        return self

    def close(self):
        if getattr(self, "h", None):
            if getattr(self, "_owner", None) is None:
                self.lib.ks_esdf_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def build_async(self, tsdf: SparseTsdf):
        _check(self.lib.ks_esdf_build_async(self.h, tsdf.h))

    def profile(self, enable=True):
        _check(self.lib.ks_esdf_profile(self.h, int(enable)))

    def stage_ms(self):
        out = (C.c_float * 6)()
        _check(self.lib.ks_esdf_stage_ms(self.h, out))
        return dict(zip(("directory", "seed", "flood_z", "sweep_y", "sweep_x", "signs"), list(out)))

    def report(self) -> EsdfReportC:
        rep = EsdfReportC()
        _check(self.lib.ks_esdf_sync(self.h, C.byref(rep)))
        return rep

    def last_report(self) -> EsdfReportC:
        """What the last blocking call (build_esdf, propagate, report ...) saw; does not wait for the device."""
        rep = EsdfReportC()
        _check(self.lib.ks_esdf_last_report(self.h, C.byref(rep)))
        return rep

    @property
    def has_sites(self) -> bool:
        return bool(self.report().has_sites)

    @property
    def signs_recovered(self) -> bool:
        return bool(self.report().signs_recovered)

    def download(self, site=True, distance=True, d2=True):
        n = self.config.cell_count()
        s = np.empty((n, 3), np.int32) if site else None
        d = np.empty(n, np.float64) if distance else None
        q = np.empty(n, np.int32) if d2 else None
        _check(self.lib.ks_esdf_download(self.h, _ptr(s), _ptr(d), _ptr(q)))
        return s, d, q

    @property
    def site(self) -> np.ndarray:
        return self.download(True, False, False)[0]

    @property
    def distance(self) -> np.ndarray:
        return self.download(False, True, False)[1]


# ---- the reference's free functions ------------------------------------------------------------------

class PinnedArray:
    """A page-locked float32 host array (ks_host_alloc): integrate_depth uploads such a frame in place."""

    def __init__(self, shape):
        self.lib = load_library()
        n = int(np.prod(shape))
        self.ptr = C.c_void_p()
        _check(self.lib.ks_host_alloc(n * 4, C.byref(self.ptr)))
        self.array = np.frombuffer((C.c_float * n).from_address(self.ptr.value), dtype=np.float32).reshape(shape)

    def close(self):
        if self.ptr:
            self.array = None
            self.lib.ks_host_free(self.ptr)
            self.ptr = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def make_tsdf(config: TsdfConfig, stream: Optional[int] = None) -> SparseTsdf:  # sdf_world.hpp:327-334
    return SparseTsdf(config, stream)


def integrate_depth(tsdf: SparseTsdf, frame: DepthFrame) -> int:  # sdf_world.hpp:340-389
    depth = np.ascontiguousarray(frame.depth, np.float32).reshape(-1)
    if depth.size != frame.width * frame.height and frame.width > 0 and frame.height > 0 and frame.fx > 0 and frame.fy > 0:
        raise ValidationError("depth frame: depth buffer size mismatch")
    cam = frame.camera()
    touched = C.c_int32()
    _check(tsdf.lib.ks_tsdf_integrate_depth(tsdf.h, C.byref(cam), _ptr(depth), C.byref(touched)))
    return touched.value


def stamp_primitive(tsdf: SparseTsdf, primitive) -> None:  # sdf_world.hpp:394-444
    if isinstance(primitive, Cuboid):
        R, t, he = _f64(primitive.pose_R, 9), _f64(primitive.pose_t, 3), _f64(primitive.half_extents, 3)
        _check(tsdf.lib.ks_tsdf_stamp_cuboid(tsdf.h, _ptr(R), _ptr(t), _ptr(he)))
    else:
        c = _f64(primitive.center, 3)
        _check(tsdf.lib.ks_tsdf_stamp_sphere(tsdf.h, _ptr(c), float(primitive.radius)))


def _primitive_array(primitives):
    arr = (PrimitiveC * max(1, len(primitives)))()
    for out, p in zip(arr, primitives):
        if isinstance(p, Cuboid):
            out.kind = 0
            out.pose_R[:] = _f64(p.pose_R, 9).tolist()
            out.pose_t[:] = _f64(p.pose_t, 3).tolist()
            out.half_extents[:] = _f64(p.half_extents, 3).tolist()
        else:
            out.kind = 1
            out.center[:] = _f64(p.center, 3).tolist()
            out.radius = float(p.radius)
    return arr


def stamp_primitives(tsdf: SparseTsdf, primitives) -> None:
    """stamp_primitive (sdf_world.hpp:394-444) over a list, in order, stopping at the first that raises -- as one batch."""
    _check(tsdf.lib.ks_tsdf_stamp_batch(tsdf.h, _primitive_array(primitives), len(primitives)))


def stamp_mesh(tsdf: SparseTsdf, mesh: TriangleMesh) -> None:  # flow of sdf_world.hpp:418-443, distance from csrc/mesh.cuh
    _check(tsdf.lib.ks_tsdf_stamp_mesh(tsdf.h, mesh.h))


def decay_weights(tsdf: SparseTsdf, camera: DepthFrame) -> None:  # sdf_world.hpp:449-457
    cam = camera.camera()
    _check(tsdf.lib.ks_tsdf_decay_weights(tsdf.h, C.byref(cam)))


def recycle_blocks(tsdf: SparseTsdf) -> int:  # sdf_world.hpp:462-475
    n = C.c_int32()
    _check(tsdf.lib.ks_tsdf_recycle_blocks(tsdf.h, C.byref(n)))
    return n.value


def _query_tsdf(tsdf: SparseTsdf, points, geom_only: bool):
    pts = np.ascontiguousarray(points, np.float64).reshape(-1, 3)
    n = pts.shape[0]
    out = np.empty(max(n, 1), np.float64)
    valid = np.empty(max(n, 1), np.uint8)
    _check(tsdf.lib.ks_tsdf_query(tsdf.h, _ptr(pts), n, int(geom_only), _ptr(out), _ptr(valid)))
    return out[:n], valid[:n].astype(bool)


def query_tsdf(tsdf: SparseTsdf, points):  # sdf_world.hpp:500-502 (batched: value, has_value)
    return _query_tsdf(tsdf, points, False)


def query_tsdf_geom(tsdf: SparseTsdf, points):  # sdf_world.hpp:505-507
    return _query_tsdf(tsdf, points, True)


def allocated_block_count(tsdf: SparseTsdf) -> int:  # sdf_world.hpp:509
    n = C.c_int32()
    _check(tsdf.lib.ks_tsdf_allocated_block_count(tsdf.h, C.byref(n)))
    return n.value


def _seed(tsdf: SparseTsdf, config: EsdfConfig, mode: int, esdf: Optional[DenseEsdf]):
    e = esdf or DenseEsdf(config)
    mask = np.empty(config.cell_count(), np.uint8)
    _check(e.lib.ks_esdf_seed(e.h, tsdf.h, mode, _ptr(mask)))
    return mask


def seed_gather(tsdf: SparseTsdf, config: EsdfConfig, esdf: Optional[DenseEsdf] = None) -> np.ndarray:  # esdf.hpp:102-122
    return _seed(tsdf, config, 1, esdf)


def seed_scatter(tsdf: SparseTsdf, config: EsdfConfig, esdf: Optional[DenseEsdf] = None) -> np.ndarray:  # esdf.hpp:73-98
    return _seed(tsdf, config, 0, esdf)


def propagate(seeds: np.ndarray, config: EsdfConfig, esdf: Optional[DenseEsdf] = None) -> DenseEsdf:  # esdf.hpp:193-282
    e = esdf or DenseEsdf(config)
    mask = np.ascontiguousarray(seeds, np.uint8).reshape(-1)
    _check(e.lib.ks_esdf_propagate(e.h, _ptr(mask), mask.size))
    return e


def recover_signs(esdf: DenseEsdf, tsdf: SparseTsdf) -> DenseEsdf:  # esdf.hpp:288-320
    _check(esdf.lib.ks_esdf_recover_signs(esdf.h, tsdf.h))
    return esdf


def build_esdf(tsdf: SparseTsdf, config: EsdfConfig, esdf: Optional[DenseEsdf] = None) -> DenseEsdf:  # esdf.hpp:323-327
    e = esdf or DenseEsdf(config)
    _check(e.lib.ks_esdf_build(e.h, tsdf.h))
    return e


class QueryBuffers:
    """Page-locked host buffers for a batch of n queries (points in, distance / gradient / inside out): with these the
    copies of `query` run at PCIe speed and no fresh host pages are touched per call."""

    def __init__(self, n: int):
        self.lib = load_library()
        self.n = int(n)
        self._ptrs = []

        def pinned(count, ctype, dtype, shape):
            ptr = C.c_void_p()
            _check(self.lib.ks_host_alloc(count * C.sizeof(ctype), C.byref(ptr)))
            self._ptrs.append(ptr)
            return np.frombuffer((ctype * count).from_address(ptr.value), dtype=dtype).reshape(shape)

        m = max(self.n, 1)
        self.points = pinned(3 * m, C.c_double, np.float64, (m, 3))
        self.distance = pinned(m, C.c_double, np.float64, (m,))
        self.gradient = pinned(3 * m, C.c_double, np.float64, (m, 3))
        self.inside = pinned(m, C.c_uint8, np.uint8, (m,))

    def close(self):
        self.points = self.distance = self.gradient = self.inside = None
        for ptr in self._ptrs:
            self.lib.ks_host_free(ptr)
        self._ptrs = []

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def query(esdf: DenseEsdf, points, buffers: Optional[QueryBuffers] = None) -> EsdfSample:  # esdf.hpp:337-387, batched over points
    """`buffers` (optional): results land in its page-locked arrays (views are returned, `inside` as uint8); pass
    `buffers.points` itself as `points` to skip the host-side copy of the inputs too."""
    pts = np.ascontiguousarray(points, np.float64).reshape(-1, 3)
    n = pts.shape[0]
    if buffers is not None:
        if n > buffers.n:
            raise ValidationError("query: more points than the buffers hold")
        if pts.ctypes.data != buffers.points.ctypes.data:
            buffers.points[:n] = pts
        _check(esdf.lib.ks_esdf_query(esdf.h, _ptr(buffers.points), n, _ptr(buffers.distance), _ptr(buffers.gradient), _ptr(buffers.inside)))
        return EsdfSample(buffers.distance[:n], buffers.gradient[:n], buffers.inside[:n])
    d = np.empty(max(n, 1), np.float64)
    g = np.empty((max(n, 1), 3), np.float64)
    inside = np.empty(max(n, 1), np.uint8)
    _check(esdf.lib.ks_esdf_query(esdf.h, _ptr(pts), n, _ptr(d), _ptr(g), _ptr(inside)))
    return EsdfSample(d[:n], g[:n], inside[:n].astype(bool))


@dataclass
class CollisionReport:  # collision.hpp:46-52 (scene part)
    max_penetration: float
    worst_first: int
    cost: float
    gradient: np.ndarray


def scene_collision_static(esdf: DenseEsdf, centers, radii, activation_margin: float = 0.025) -> CollisionReport:
    """collision.hpp:130-152"""
    c = np.ascontiguousarray(centers, np.float64).reshape(-1, 3)
    r = np.ascontiguousarray(radii, np.float64).reshape(-1)
    if c.shape[0] != r.size:
        raise ValidationError("scene_collision: center/radius count mismatch")
    rep = CollisionReportC()
    grad = np.zeros((max(r.size, 1), 3), np.float64)
    _check(esdf.lib.ks_esdf_scene_collision_static(esdf.h, _ptr(c), _ptr(r), r.size, float(activation_margin), C.byref(rep), _ptr(grad)))
    return CollisionReport(rep.max_penetration, rep.worst_sphere, rep.cost, grad[:r.size])


def scene_collision(esdf: DenseEsdf, centers, radii, velocities, activation_margin=0.025, dt=1.0, max_checks=10000):
    """collision.hpp:177-239 -> (reports[T] as (max_penetration, worst_sphere, cost) array, center, next, velocity gradients)"""
    c = np.ascontiguousarray(centers, np.float64)
    v = np.ascontiguousarray(velocities, np.float64)
    if c.shape[0] != v.shape[0]:
        raise ValidationError("scene_collision: centers/velocities timestep mismatch")
    T, S = c.shape[0], c.shape[1]
    r = np.ascontiguousarray(radii, np.float64).reshape(-1)
    if r.size != S or v.shape[1] != S:
        raise ValidationError("scene_collision: sphere count mismatch at timestep")
    reps = (CollisionReportC * T)()
    g0, g1, g2 = (np.zeros((T, S, 3), np.float64) for _ in range(3))
    _check(esdf.lib.ks_esdf_scene_collision_swept(esdf.h, _ptr(c), _ptr(r), _ptr(v), T, S, float(activation_margin), float(dt),
                                                  int(max_checks), reps, _ptr(g0), _ptr(g1), _ptr(g2)))
    out = np.array([[x.max_penetration, x.worst_sphere, x.cost] for x in reps], np.float64)
    return out, g0, g1, g2


# ---- CUDA graph helper ----------------------------------------------------------------------------

class Graph:
    """Capture a sequence of *_async calls issued on `stream` into one replayable CUDA graph."""

    def __init__(self, stream: int):
        self.lib = load_library()
        self.stream = C.c_void_p(stream)
        self.h = C.c_void_p()

    def __enter__(self):
        _check(self.lib.ks_graph_begin_capture(self.stream))
        return self

    def __exit__(self, exc_type, exc, tb):
        rc = self.lib.ks_graph_end_capture(self.stream, C.byref(self.h))
        if exc_type is None:
            _check(rc)
        return False

    def launch(self):
        _check(self.lib.ks_graph_launch(self.h, self.stream))

    def node_count(self) -> Tuple[int, int]:
        k, a = C.c_int64(), C.c_int64()
        _check(self.lib.ks_graph_node_count(self.h, C.byref(k), C.byref(a)))
        return k.value, a.value

    def close(self):
        if self.h:
            self.lib.ks_graph_destroy(self.h)
            self.h = C.c_void_p()


# ---- batched environments (BASELINE configs[4]; include/ks_b200.h "batched environments") ---------------------------------

SUMMARY_FIELDS = ("env", "min_distance", "colliding", "seeds")  # 4 x float64 per environment


def partition_envs(n_envs: int, world: int, rank: int) -> Tuple[int, int]:
    """ks_partition_envs: the contiguous range [lo, hi) of environments `rank` owns (earlier ranks take the remainder)."""
    lo, hi = C.c_int32(), C.c_int32()
    if load_library().ks_partition_envs(n_envs, world, rank, C.byref(lo), C.byref(hi)) != KS_OK:
        raise ValueError(last_error())
    return lo.value, hi.value


def nccl_unique_id() -> bytes:
    buf = (C.c_char * 128)()
    _check(load_library().ks_nccl_unique_id(buf))
    return bytes(buf)


class EnvBatch:
    """ks_batch: n independent (SparseTsdf, DenseEsdf) pairs of one configuration updated by one enqueue / one graph."""

    def __init__(self, n_envs: int, tsdf_config: TsdfConfig, esdf_config: EsdfConfig, lanes: int = 2, first_env: int = 0):
        self.lib = load_library()
        tc = TsdfConfigC(tsdf_config.voxel_size, tsdf_config.truncation, tsdf_config.alpha_time, tsdf_config.alpha_frustum,
                         tsdf_config.weight_threshold, int(tsdf_config.capacity), int(tsdf_config.slot_count))
        ec = EsdfConfigC()
        ec.origin[:] = [float(v) for v in esdf_config.origin]
        ec.nx, ec.ny, ec.nz = int(esdf_config.nx), int(esdf_config.ny), int(esdf_config.nz)
        ec.voxel_size = float(esdf_config.voxel_size)
        ec.seeding = 1 if esdf_config.seeding == "gather" else 0
        h = C.c_void_p()
        _check(self.lib.ks_batch_create(n_envs, C.byref(tc), C.byref(ec), lanes, C.byref(h)))
        self.h = h
        self.n = n_envs
        self.first_env = first_env
        _check(self.lib.ks_batch_set_first_env(self.h, first_env))
        self.tsdf = [SparseTsdf._borrowed(self.lib.ks_batch_tsdf(self.h, i), tsdf_config, self) for i in range(n_envs)]
        self.esdf = [DenseEsdf._borrowed(self.lib.ks_batch_esdf(self.h, i), esdf_config, self) for i in range(n_envs)]
        self._meshes = {}

    @property
    def stream(self) -> int:
        return int(self.lib.ks_batch_stream(self.h) or 0)

    @property
    def lanes(self) -> int:
        return int(self.lib.ks_batch_lanes(self.h))

    def set_inputs(self, env: int, n_cameras: int, primitives=(), meshes=()):
        prims = [p for p in primitives]
        arr = _primitive_array(prims)
        self._meshes[env] = list(meshes)  # borrowed by the library: keep them alive
        marr = (C.c_void_p * max(1, len(meshes)))(*[m.h for m in meshes])
        _check(self.lib.ks_batch_set_inputs(self.h, env, n_cameras, arr, len(prims), marr, len(meshes)))

    def set_probes(self, env: int, points, near_distance: float):
        pts = np.ascontiguousarray(np.asarray(points, np.float64).reshape(-1, 3))
        _check(self.lib.ks_batch_set_probes(self.h, env, _ptr(pts), pts.shape[0], float(near_distance)))

    def update_async(self, upload_frames: bool = True):
        _check(self.lib.ks_batch_update_async(self.h, int(upload_frames)))

    def update(self, upload_frames: bool = True):
        _check(self.lib.ks_batch_update(self.h, int(upload_frames)))

    def graph_kernels(self) -> int:
        return int(self.lib.ks_batch_graph_kernels(self.h))

    def sync(self):
        """(tsdf reports, esdf reports, summaries [n, 4]) after waiting for the batch stream."""
        reps = (TsdfReportC * self.n)()
        ereps = (EsdfReportC * self.n)()
        summ = np.empty((self.n, 4), np.float64)
        _check(self.lib.ks_batch_sync(self.h, reps, ereps, _ptr(summ)))
        return list(reps), list(ereps), summ

    def attach_nccl(self, unique_id: bytes, world: int, rank: int, max_local_envs: int):
        buf = (C.c_char * 128).from_buffer_copy(unique_id)
        _check(self.lib.ks_batch_attach_nccl(self.h, buf, world, rank, max_local_envs))

    def gathered(self) -> np.ndarray:
        rows = int(self.lib.ks_batch_gathered_rows(self.h))
        out = np.empty((rows, 4), np.float64)
        _check(self.lib.ks_batch_gathered(self.h, _ptr(out)))
        return out

    def close(self):
        if getattr(self, "h", None):
            for w in self.tsdf + self.esdf:
                w.h = None
            self.lib.ks_batch_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass
