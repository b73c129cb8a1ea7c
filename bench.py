#!/usr/bin/env python
"""ESDF-update benchmark for the perception hot path (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--workload cfg2|cfg1|cfg3|cfg5env]

One step = one full update of the workload scene: integrate the depth frame(s) + stamp the cuboids +
gather seeding + exact EDT + sign recovery (the ESDF is left queryable in HBM).  Default workload is
BASELINE.json configs[1]: 2 x 1 x 1 m workspace at 5 mm (400 x 200 x 200 = 16 M cells), one 640x480
camera, three cuboids.

  value  : ESDF cells per second, CUDA-graph replay, inputs resident in HBM (CUDA events, L2 flushed
           between steps, max over ranks; N ranks run N independent environments -> weak scaling)
  e2e    : the same metric through the blocking ks:: drop-in calls with HOST buffers
           (pinned staging + H2D of the frame, D2H of the reports inside the timed region)
  roofline     : the slowest kernel stage, algorithmic bytes / its CUDA-event time / measured HBM peak
  cpu_baseline : the reference's CPU implementation of the same update on this box's host, 1 core

--impl reference times only the CPU implementation (oracle/_ref = the reference's own headers when
built, else the oracle port).  The reference is single-threaded by construction, so cores = 1.
"""
from __future__ import annotations

import argparse
import ctypes as C
import json
import os
import statistics
import subprocess
import sys
import threading
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

METRIC = "esdf_update_voxels_per_s"
UNIT = "voxels/s"


# ---- workloads ------------------------------------------------------------------------------------------
def make_scene(workload: str, env: int = 0):
    from paper_2603_05493_b200 import scenes
    if workload == "cfg1":
        sc = scenes.config1("wavy")
    elif workload == "cfg2":
        sc = scenes.config2()
    elif workload == "cfg3":
        sc = scenes.config3()
    elif workload == "cfg4":
        sc = scenes.config4()[0]
    elif workload == "cfg5env":
        sc = scenes.config5_env(env)
    else:
        raise SystemExit(f"unknown workload {workload}")
    if env and workload != "cfg5env":  # independent environments: same layout, different surface
        for i, f in enumerate(sc.frames):
            f.depth = scenes.wavy_depth(float(f.depth.mean()), 0.1 if workload == "cfg2" else 0.05, phase=0.37 * env + i)
    return sc


WORKLOAD_DESC = {
    "cfg1": "configs[0]: 640x480 depth frame into 1 m^3 at 1 cm (100^3 cells)",
    "cfg2": "configs[1]: 2 m^3 (2x1x1 m) workspace at 5 mm, 400x200x200 cells, one 640x480 depth camera + 3 cuboids, full ESDF every frame",
    "cfg3": "configs[2]: 1 m^3 at 2 mm, 500^3 cells, 4 depth cameras + 2 cuboids",
    "cfg4": "configs[3]: configs[1] scene + sphere + 1280-triangle mesh, 1 M batched distance+gradient queries per update",
    "cfg5env": "configs[4]: independent 1.5x1x1 m environments at 5 mm (300x200x200 cells), --envs-per-gpu per rank",
}


def config_of(workload: str, scene, world: int, envs_per_gpu: int, queries: int):
    """The workload both arms report (identical keys and values in `--impl ours` and `--impl reference`)."""
    nx, ny, nz = scene.esdf_dims
    return {"workload": WORKLOAD_DESC[workload], "cells": nx * ny * nz, "dims": [nx, ny, nz], "tsdf_voxel_m": scene.tsdf_voxel,
            "esdf_voxel_m": scene.esdf_voxel, "cameras": len(scene.frames), "cuboids": len(scene.cuboids), "spheres": len(scene.spheres),
            "meshes": len(getattr(scene, "meshes", [])), "environments": world * envs_per_gpu, "environments_per_gpu": envs_per_gpu,
            "queries_per_update": queries}


def resolve_workload(args):
    """Default workload: configs[1] on one GPU; on N > 1 GPUs BASELINE.json's batched case, configs[4] = 128 environments."""
    world = int(os.environ.get("WORLD_SIZE", "1"))
    if args.workload is None:
        args.workload = "cfg5env" if world > 1 else "cfg2"
    if args.envs_per_gpu is None:
        args.envs_per_gpu = max(1, 128 // world) if (args.workload == "cfg5env" and world > 1) else 1
    return args


# ---- clocks ---------------------------------------------------------------------------------------------
class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled while the GPU is under this benchmark's load."""

    QUERY = ("timestamp,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
             "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.rows = []
        self.proc = None

    def start(self, wait_s: float = 5.0):
        """Start nvidia-smi and wait until its first sample has arrived (its start-up alone can take a second)."""
        try:
            self.proc = subprocess.Popen(["nvidia-smi", f"--id={self.index}", f"--query-gpu={self.QUERY}",
                                          "--format=csv,noheader,nounits", "-lms", "20"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            threading.Thread(target=self._pump, daemon=True).start()
        except OSError:
            self.proc = None
            return
        deadline = time.time() + wait_s
        while not self.rows and time.time() < deadline:
            time.sleep(0.01)

    def _pump(self):
        for line in self.proc.stdout:
            self.rows.append((time.time(), [c.strip() for c in line.split(",")]))

    def stop(self, t_begin: float, t_end: float, t_load: float = None):
        """Summarise the samples that arrived inside [t_begin, t_end] (the timed region); when that region is shorter
        than ~10 sampling periods, the window is widened backwards over the uninterrupted load that led into it
        (t_load: since when the GPU has been replaying the same update back to back)."""
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        time.sleep(0.05)
        self.proc.terminate()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]

        def summarise(rows):
            sm, mx, reasons = [], [], set()
            for _, r in rows:
                if len(r) < 8:
                    continue
                try:
                    sm.append(float(r[1]))
                    mx.append(float(r[2]))
                except ValueError:
                    continue
                for name, flag in zip(names, r[4:8]):
                    if flag.lower().startswith("active"):
                        reasons.add(name)
            return sm, mx, reasons

        inside = [row for row in self.rows if t_begin <= row[0] <= t_end]
        sm, mx, reasons = summarise(inside)
        window = "timed region"
        if len(sm) < 10 and t_load is not None:  # a short region: add the back-to-back replays that ran right before it
            sm, mx, reasons = summarise([row for row in self.rows if t_load <= row[0] <= t_end])
            window = "timed region + the %.1f s of uninterrupted replay before it (%d samples inside the region itself)" % (
                t_begin - t_load, len(inside))
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": sorted(reasons), "samples": len(sm), "window": window}


# ---- CPU legs -------------------------------------------------------------------------------------------
def cpu_checker():
    sys.path.insert(0, str(ROOT / "tests"))
    import cpu_checkers
    if cpu_checkers.reference_available():
        return cpu_checkers.reference()
    return cpu_checkers.oracle()


def cpu_update_seconds(lib, scene, dims):
    """One full update on a fresh world, timed inside the C/C++ library; returns (seconds, stage dict)."""
    world = lib.make_tsdf(scene.tsdf_voxel, capacity=scene.capacity)
    stages, seeds, checksum = lib.timed_update(world, scene, dims)
    world.close()
    return sum(stages.values()), stages, seeds, checksum


def host_cpu_model():
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    scene = make_scene(args.workload)
    lib = cpu_checker()
    nx, ny, nz = scene.esdf_dims
    # bounded sample: full TSDF update + ESDF over the first `zs` z-slices, sized so W+K steps take ~2.5 min
    per_cell_s = 3.6e-7  # ~2.8 M cells/s measured for this path on one core
    budget = 150.0 / max(1, args.steps + args.warmup)
    zs = int(max(4, min(nz, budget / (per_cell_s * nx * ny))))
    dims = (nx, ny, zs)
    cells = nx * ny * zs
    for _ in range(args.warmup):
        cpu_update_seconds(lib, scene, dims)
    t0 = time.perf_counter()
    inner = []
    for _ in range(args.steps):
        inner.append(cpu_update_seconds(lib, scene, dims)[0])
    wall = time.perf_counter() - t0
    secs = sum(inner)
    value = cells * args.steps / secs
    sample = (f"{args.workload} scene, full TSDF update + ESDF over {nx}x{ny}x{zs} of {nx}x{ny}x{nz} cells per step "
              f"(z-slab sample), timed inside the library; wall {wall:.1f}s; host {host_cpu_model()}")
    if getattr(scene, "meshes", None):  # the reference has no mesh stamping: its arm runs the scene without them
        sample += f"; the scene's {len(scene.meshes)} triangle mesh(es) are NOT stamped by the reference (no such function)"
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": 1e3 * secs / args.steps, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": config_of(args.workload, scene, int(os.environ.get("WORLD_SIZE", "1")), args.envs_per_gpu,
                            1_000_000 if args.workload == "cfg4" else 0),
        "sample_cells_per_step": cells,
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": 1, "kind": lib.kind, "sample": sample},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line))


# ---- our arm --------------------------------------------------------------------------------------------
def algorithmic_bytes(stage: str, C_: int, P: int, K: int, Kp: int, L: int, dcount: int) -> float:
    """Compulsory HBM bytes of each stage for the device formats in DESIGN.md."""
    return {
        "discover": 4.0 * P + 20.0 * K,
        "allocate": 12.0 * K,
        "integrate": 4.0 * P + K * (512 * (16 + 16 + 8) + 320),
        "stamp_blocks": Kp * (512 * (8 + 8 + 16) + 320),
        "directory": 4.0 * dcount + 8.0 * L,
        "seed": 3.0 * C_ / 8.0 + 6.0 * C_ / 8.0 + 2.0 * C_ / 8.0 + 128.0 * L + 5.0 * dcount,  # 3 resampled planes out; 5 rows + near row in, seed + near planes out; digest rows + directory in
        "flood_z": 2.0 * C_ / 8.0 + 3.0 * C_ / 8.0,                   # seed + table bit planes in; column bit strings (seeds, tables) + per-word info out
        "sweep_y": 3.0 * C_ / 8.0 + 6.0 * C_,                         # column words + info in; tile images out: candidate u32 + payload u16
        "sweep_x": 4.0 * C_ + 4.0 * C_ + C_ / 8.0,                    # candidate image in (u32; the u16 payload image is only touched next to stamped geometry), field word u32 out, own-sign plane
        "signs": 0.0,                                                 # fused into sweep_x
    }[stage]


def run_ours(args):
    import torch
    import torch.distributed as dist

    from paper_2603_05493_b200 import api, build
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    # the library normally travels prebuilt; if it is missing exactly one rank per node compiles it
    if not build.LIB.exists():
        if local == 0:
            build.build(force=True)
        else:
            deadline = time.time() + 300
            while not build.LIB.exists() and time.time() < deadline:
                time.sleep(1.0)
            time.sleep(2.0)
    if not torch.cuda.is_available():
        raise SystemExit("bench.py needs a CUDA device: the perception path has no CPU implementation")
    # KS_BENCH_SHARE_GPU=1 (tests only): every rank uses device 0 and the collective runs on gloo, so the
    # N > 1 control flow can be exercised on a one-GPU box.  The real multi-GPU run is NCCL, one rank per GPU.
    share_gpu = os.environ.get("KS_BENCH_SHARE_GPU") == "1"
    if share_gpu:
        local = 0
    torch.cuda.set_device(local)
    if world > 1:
        if share_gpu:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))

    def all_reduce_max(t):
        if share_gpu:
            c = t.cpu()
            dist.all_reduce(c, op=dist.ReduceOp.MAX)
            t.copy_(c)
        else:
            dist.all_reduce(t, op=dist.ReduceOp.MAX)

    stream = torch.cuda.Stream()
    E_local = max(1, args.envs_per_gpu)
    n_envs = world * E_local
    env_lo, env_hi = api.partition_envs(n_envs, world, rank)

    class Environment:
        """One independent scene: its own TSDF + ESDF handles, all on this rank's stream."""

        def __init__(self, env_id, handles=None):
            self.env_id = env_id
            queries = None
            if args.workload == "cfg4":
                from paper_2603_05493_b200 import scenes as _scenes
                self.scene, queries = _scenes.config4()
            else:
                self.scene = make_scene(args.workload, env=env_id)
            sc = self.scene
            self.dims = sc.esdf_dims
            # the "camera driver" writes its frames into page-locked host memory: the blocking calls upload them in place
            self.pinned = [api.PinnedArray((f.height, f.width)) for f in sc.frames]
            for pin, f in zip(self.pinned, sc.frames):
                pin.array[...] = np.asarray(f.depth, np.float32).reshape(f.height, f.width)
            self.frames = [api.DepthFrame(f.width, f.height, *f.intr, f.R, f.t, pin.array) for pin, f in zip(self.pinned, sc.frames)]
            self.staged_frames = None  # the same frames living in the handle's own staging slots (graph path)
            self.prims = [api.Cuboid(c.R, c.t, c.half_extents) for c in sc.cuboids] + \
                         [api.SphereShape(s.center, s.radius) for s in sc.spheres]
            self.meshes = [api.TriangleMesh(m.vertices, m.triangles) for m in sc.meshes]  # uploaded once (static geometry)
            cfg = api.make_tsdf_config(sc.tsdf_voxel)
            cfg.capacity = sc.capacity
            self.tcfg = cfg
            self.ecfg = api.EsdfConfig(tuple(sc.esdf_origin), *sc.esdf_dims, sc.esdf_voxel, "gather")
            if handles is None:
                self.tsdf = api.make_tsdf(cfg, stream.cuda_stream)
                self.esdf = api.DenseEsdf(self.ecfg, stream.cuda_stream)
            else:  # worlds owned by the C-ABI batch (ks_batch_*)
                self.tsdf, self.esdf = handles
            ext = np.array(sc.esdf_dims) * sc.esdf_voxel
            self.probes_host = np.ascontiguousarray(sc.esdf_origin + np.random.RandomState(3 + env_id).random_sample((4096, 3)) * ext)
            self.queries = None
            self.q_events = None  # (start, end) CUDA events around the query kernel while stage times are taken
            if queries is not None:  # configs[3]: 1 M batched distance + gradient queries per update
                self.query_buffers = api.QueryBuffers(len(queries))   # page-locked: the "planner" writes its points here
                self.query_buffers.points[...] = queries
                self.queries_host = self.query_buffers.points
                self.queries = torch.from_numpy(queries).cuda()
                self.q_dist = torch.empty(len(queries), dtype=torch.float64, device="cuda")
                self.q_grad = torch.empty((len(queries), 3), dtype=torch.float64, device="cuda")
                self.q_inside = torch.empty(len(queries), dtype=torch.uint8, device="cuda")

        def stage(self):
            if self.staged_frames is None:  # once: the frames move into the slots' pinned staging areas
                self.staged_frames = []
                for slot, f in enumerate(self.frames):
                    buf = self.tsdf.frame_buffer(f.width, f.height, slot)
                    buf[...] = np.asarray(f.depth, np.float32).reshape(f.height, f.width)
                    self.staged_frames.append(api.DepthFrame(f.width, f.height, f.fx, f.fy, f.cx, f.cy, f.pose_R, f.pose_t, buf))
            for slot, f in enumerate(self.staged_frames):
                self.tsdf.stage_frame(f, slot)  # camera parameters only: the pixels are already in place

        def enqueue_update(self, upload):
            for slot in range(len(self.frames)):  # one staging slot per camera
                if upload:
                    self.tsdf.upload_frame_async(slot)
                self.tsdf.integrate_async(slot)
            if self.prims:  # every cuboid / sphere of the update as one batch (three launches), meshes one by one
                self.tsdf.stamp_batch_async(self.prims)
            for m in self.meshes:
                self.tsdf.stamp_async(m)
            self.esdf.build_async(self.tsdf)
            if self.queries is not None:
                if self.q_events is not None:
                    self.q_events[0].record()
                api._check(self.esdf.lib.ks_esdf_query_device_async(
                    self.esdf.h, C.c_void_p(self.queries.data_ptr()), self.queries.shape[0], C.c_void_p(self.q_dist.data_ptr()),
                    C.c_void_p(self.q_grad.data_ptr()), C.c_void_p(self.q_inside.data_ptr())))
                if self.q_events is not None:
                    self.q_events[1].record()

        def blocking_update(self):
            k = 0
            for f in self.frames:
                k = api.integrate_depth(self.tsdf, f)          # H2D from the page-locked frame + 4 phases + D2H report
            if self.prims:
                api.stamp_primitives(self.tsdf, self.prims)
            for m in self.meshes:
                api.stamp_mesh(self.tsdf, m)
            api.build_esdf(self.tsdf, self.ecfg, self.esdf)
            r = self.esdf.last_report()                         # has_sites / seed count, read back by build_esdf (D2H)
            if self.queries is not None:
                api.query(self.esdf, self.queries_host, self.query_buffers)  # H2D points, D2H distance + gradient + inside (page-locked)
            return k, r.seed_count

    # Several environments (configs[4]) go through the C-ABI batch: ks_batch_create owns the worlds, one update of all of
    # them is one enqueue / one private graph, the per-environment summaries are written by the update itself and
    # all-gathered by ncclAllGather as the last node of that graph.
    exchange = world > 1 or E_local > 1
    batch = None
    if exchange:
        sc0 = make_scene(args.workload, env=env_lo)
        cfg0 = api.make_tsdf_config(sc0.tsdf_voxel)
        cfg0.capacity = sc0.capacity
        ecfg0 = api.EsdfConfig(tuple(sc0.esdf_origin), *sc0.esdf_dims, sc0.esdf_voxel, "gather")
        batch = api.EnvBatch(env_hi - env_lo, cfg0, ecfg0, lanes=args.lanes, first_env=env_lo)
        stream = torch.cuda.ExternalStream(batch.stream)
        envs = [Environment(e, (batch.tsdf[e - env_lo], batch.esdf[e - env_lo])) for e in range(env_lo, env_hi)]
        for i, env in enumerate(envs):
            batch.set_inputs(i, len(env.frames), env.prims, env.meshes)
            batch.set_probes(i, env.probes_host, 0.02)
        if world > 1 and not share_gpu:  # the batch's own communicator: 128-byte id from rank 0, ncclCommInitRank on every rank
            uid = [api.nccl_unique_id() if rank == 0 else None]
            dist.broadcast_object_list(uid, src=0)
            batch.attach_nccl(uid[0], world, rank, E_local)
    else:
        envs = [Environment(e) for e in range(env_lo, env_hi)]
    scene = envs[0].scene
    nx, ny, nz = scene.esdf_dims
    cells = nx * ny * nz
    frames, prims = envs[0].frames, envs[0].prims
    tsdf, esdf, ecfg = envs[0].tsdf, envs[0].esdf, envs[0].ecfg
    pixels = sum(f.width * f.height for f in frames)
    n_queries = 0 if envs[0].queries is None else int(envs[0].queries.shape[0])

    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")

    def enqueue_update(upload: bool):
        if batch is not None:
            batch.update_async(upload)
        else:
            envs[0].enqueue_update(upload)

    def gather_summaries_shared_gpu():
        """test mode only (KS_BENCH_SHARE_GPU=1, every rank on device 0, NCCL impossible): the summaries the update
        wrote are exchanged through gloo from the host.  The real multi-GPU run gathers inside the batch graph."""
        _, _, mine = batch.sync()
        pad = np.full((E_local, 4), np.nan)
        pad[:mine.shape[0]] = mine
        host_all = torch.empty((world * E_local, 4), dtype=torch.float64)
        dist.all_gather_into_tensor(host_all, torch.from_numpy(pad))
        return host_all.numpy()

    with torch.cuda.stream(stream):
        # ---- eager warm-up (allocates blocks, binds the directory), then stage timings ---------------
        for env in envs:
            env.stage()
        enqueue_update(upload=True)
        rep = tsdf.sync()
        touched_last, live = rep.blocks_touched, rep.live_blocks
        tsdf.profile(True)
        esdf.profile(True)
        stage_acc = {}
        if envs[0].queries is not None:
            envs[0].q_events = (torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
        for i in range(args.warmup + min(args.steps, 20)):
            flush.zero_()
            envs[0].enqueue_update(False)
            st = {**tsdf.stage_ms(), **esdf.stage_ms()}
            if envs[0].q_events is not None:
                stream.synchronize()
                st["query"] = envs[0].q_events[0].elapsed_time(envs[0].q_events[1])
            if i >= args.warmup:
                for k, v in st.items():
                    stage_acc.setdefault(k, []).append(v)
        envs[0].q_events = None
        stage_ms = {k: float(np.mean(v)) for k, v in stage_acc.items()}

        # ---- cold frame: the first update of a FRESH world (every block still to be allocated), plain launches -----------
        cold_ms = []
        for _ in range(3):
            cfg_cold = api.make_tsdf_config(scene.tsdf_voxel)
            cfg_cold.capacity = scene.capacity
            cold = api.make_tsdf(cfg_cold, stream.cuda_stream)
            for slot, f in enumerate(envs[0].frames):
                cold.stage_frame(f, slot)  # staging buffers and op lists are set up here, outside the timed part
                cold.upload_frame_async(slot)
            cold.sync()
            flush.zero_()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            for slot in range(len(envs[0].frames)):
                cold.integrate_async(slot)
            if envs[0].prims:
                cold.stamp_batch_async(envs[0].prims)
            for m in envs[0].meshes:
                cold.stamp_async(m)
            esdf.build_async(cold)
            e1.record()
            rep_cold = cold.sync()
            assert rep_cold.status == 0
            cold_ms.append(e0.elapsed_time(e1))
            cold.close()
        esdf.build_async(tsdf)  # back on the benchmark's own world
        tsdf.profile(False)
        esdf.profile(False)

        # ---- graph capture (inputs resident in HBM; multi-camera workloads re-upload inside the graph) --
        if batch is not None:  # the batch's private graph (ks_batch_update): first call captures, later calls replay
            class _BatchGraph:
                def launch(self):
                    batch.update(False)
            graph = _BatchGraph()
            graph.launch()
            kernel_nodes = all_nodes = batch.graph_kernels()
        else:
            graph = api.Graph(stream.cuda_stream)
            with graph:
                enqueue_update(upload=False)
            kernel_nodes, all_nodes = graph.node_count()
        sampler = ClockSampler(local)
        sampler.start()
        t_load = time.time()
        replays = 0
        while replays < max(args.warmup, 50) or time.time() - t_load < 1.2:  # >= 1.2 s of the same load the timed steps apply
            for _ in range(25):
                flush.zero_()
                graph.launch()
            replays += 25
            stream.synchronize()
        if world > 1:
            dist.barrier()
        starts = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
        ends = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
        torch.cuda.synchronize()
        t_begin = time.time()
        for i in range(args.steps):
            flush.zero_()  # L2 flush between timed iterations (outside the event pair)
            starts[i].record(stream)
            graph.launch()
            ends[i].record(stream)
        torch.cuda.synchronize()
        t_end = time.time()
        if world > 1:
            dist.barrier()
        clocks = sampler.stop(t_begin, t_end, t_load)
        per_step = [s.elapsed_time(e) for s, e in zip(starts, ends)]
        total_ms = torch.tensor([sum(per_step)], dtype=torch.float64, device="cuda")
        if world > 1:
            all_reduce_max(total_ms)
        total_ms = float(total_ms.item())
        rep = tsdf.sync()
        erep = esdf.report()
        assert rep.status == 0 and erep.has_sites

        # ---- e2e: blocking drop-in calls with host buffers ------------------------------------------------
        def blocking_update():
            if batch is None:
                envs[0].blocking_update()
                return
            # batch: every camera's pixels are written into its slot's page-locked staging area (zero-copy staging),
            # the update graph uploads them (H2D inside the timed region), sync reads back reports + summaries (D2H)
            for env in envs:
                env.stage()
            batch.update(True)
            batch.sync()

        for _ in range(args.warmup):
            blocking_update()
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        t0 = time.perf_counter()
        for _ in range(args.steps):
            blocking_update()
        torch.cuda.synchronize()
        e2e_s = torch.tensor([time.perf_counter() - t0], dtype=torch.float64, device="cuda")
        if world > 1:
            all_reduce_max(e2e_s)
        e2e_s = float(e2e_s.item())

        # ---- e2e through the graph API (stage + upload + replay + report), informational ----------------
        t0 = time.perf_counter()
        for _ in range(args.steps):
            if batch is not None:
                blocking_update()
                continue
            for env in envs:
                env.stage()
                for slot in range(len(env.frames)):
                    env.tsdf.upload_frame_async(slot)
            graph.launch()
            for env in envs:
                env.tsdf.sync()
                env.esdf.report()
        e2e_graph_s = time.perf_counter() - t0

        # ---- the exchanged summaries: every environment of every rank must be there -----------------------------------
        gathered_rows = None
        if batch is not None:
            rows = gather_summaries_shared_gpu() if (world > 1 and share_gpu) else batch.gathered()
            ids = sorted(int(r[0]) for r in rows if not np.isnan(r[0]))
            assert ids == list(range(n_envs)), f"summary exchange incomplete: {ids}"
            assert all(r[3] > 0 for r in rows if not np.isnan(r[0])), "an environment reported no seeds"
            gathered_rows = len(ids)

    if rank != 0:
        if world > 1:
            dist.destroy_process_group()
        return

    # ---- roofline of the slowest stage ------------------------------------------------------------------
    peaks_path = ROOT / "MEASURED_PEAKS.json"
    if peaks_path.exists():
        peak, peak_src = float(json.loads(peaks_path.read_text())["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    else:
        peak, peak_src = 6650.0, "fallback (B200_PROFILING.md)"
    K = touched_last if touched_last > 0 else 0
    dcount = 0
    kernel_stages = ["discover", "allocate", "integrate", "stamp_blocks", "directory", "seed", "flood_z", "sweep_y", "sweep_x", "signs"]
    dominant = max(kernel_stages, key=lambda s: stage_ms.get(s, 0.0))
    stage_bytes = {s: algorithmic_bytes(s, cells, pixels, K, max(live - K, 0), live, dcount) for s in kernel_stages}
    achieved = stage_bytes[dominant] / (stage_ms[dominant] * 1e-3) / 1e9
    traffic, traffic_all = None, {}
    traffic_path = ROOT / "profiles" / "dram_traffic.json"
    if traffic_path.exists():  # per-launch DRAM bytes from committed ncu captures of the same command (not measurable without ncu)
        traffic_all = json.loads(traffic_path.read_text()).get(args.workload, {})
        traffic = traffic_all.get(dominant)
    update_bytes = sum(stage_bytes[s] * (len(frames) if s in ("discover", "allocate", "integrate") else 1) for s in kernel_stages)
    survey_bytes = (len(frames) * 4.0 * (pixels / max(1, len(frames))) + 2 * 16 * 512 * K * len(frames) + 2 * 8 * 512 * max(live - K, 0)
                    + 30.0 * cells + 16384.0 * live + 20.0 * 2 * scene.capacity)
    stage_bytes["stamp_candidates"] = 0.0
    if n_queries:
        stage_bytes["query"] = 89.0 * n_queries  # 24 B in + 33 B out + 8 gathers of 4 B
    stage_table = []
    for name in ["discover", "allocate", "integrate", "stamp_candidates", "stamp_blocks", "directory", "seed", "flood_z", "sweep_y", "sweep_x", "query"]:
        if name not in stage_ms:
            continue
        ms = stage_ms[name]
        gbs = stage_bytes.get(name, 0.0) / (ms * 1e-3) / 1e9 if ms > 0 else 0.0
        stage_table.append({"stage": name, "ms": round(ms, 5), "algorithmic_bytes": stage_bytes.get(name, 0.0), "GB/s": round(gbs, 1),
                            "frac_of_hbm_peak": round(gbs / peak, 4), "dram_traffic_bytes": traffic_all.get(name)})
    ms_per_step = total_ms / args.steps
    value = n_envs * cells * args.steps / (total_ms * 1e-3)

    cpu_base = None
    if world == 1 and not args.no_cpu_baseline:
        lib = cpu_checker()
        sample_dims = scene.esdf_dims if cells <= 20_000_000 else (nx, ny, max(4, int(20_000_000 / (nx * ny))))
        runs = [cpu_update_seconds(lib, scene, sample_dims) for _ in range(2)]
        secs = min(r[0] for r in runs)
        sample_cells = sample_dims[0] * sample_dims[1] * sample_dims[2]
        cpu_base = {"value": sample_cells / secs, "unit": UNIT, "cores": 1, "kind": lib.kind,
                    "sample": f"2 full {args.workload} updates ({sample_dims[0]}x{sample_dims[1]}x{sample_dims[2]} cells each) on a fresh world, "
                              f"best of 2, timed inside the library; stages s = "
                              f"{ {k: round(v, 3) for k, v in runs[0][1].items()} }; host {host_cpu_model()}",
                    "seconds_per_update": secs}
        if getattr(scene, "meshes", None):
            cpu_base["sample"] += f"; the scene's {len(scene.meshes)} triangle mesh(es) are not stamped on the CPU side (the reference has no mesh stamping)"

    h2d = E_local * (sum(f.width * f.height * 4 + 248 for f in frames) + 24 * n_queries)
    d2h = E_local * (48 * (len(frames) + len(prims)) + 16 + 33 * n_queries)
    if batch is not None:  # per environment: the control block (ks_tsdf_sync), the ESDF report, its 32-byte summary row
        d2h = E_local * (48 + 16 + 32)
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": ms_per_step, "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic",
        "config": config_of(args.workload, scene, world, E_local, n_queries),
        "run": {"blocks_touched": touched_last, "live_blocks": live, "seeds": int(erep.seed_count), "execution": "cuda-graph replay",
                "l2": "flushed between timed steps (256 MiB memset outside the event pairs); per-step working set ~18 B/cell > 126 MB L2",
                "collective": "none" if not exchange else
                              ("ncclAllGather of 32-byte per-environment summaries, last node of the batch graph (ks_batch_attach_nccl)" if world > 1 and not share_gpu
                               else "ncclAllGather path not taken on one rank: summaries written by the update, read from the batch buffer"
                               if world == 1 else "test mode (ranks share one GPU): summaries exchanged through gloo; the multi-GPU run uses ncclAllGather inside the batch graph"),
                "summary_rows_gathered": gathered_rows, "lanes": None if batch is None else batch.lanes,
                "state": "steady state: the world's blocks exist (allocated by the warm-up); cold_frame_ms is the first update of a fresh world"},
        "clocks": clocks,
        "e2e": {"value": n_envs * cells * args.steps / e2e_s, "unit": UNIT, "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
                "ms_per_step": 1e3 * e2e_s / args.steps, "path": ("blocking ks:: calls: integrate_depth(page-locked host frame, uploaded in place) + stamp_primitive x%d + build_esdf + report" % len(prims))
                        if batch is None else "ks_batch: stage every frame in its pinned slot + ks_batch_update(upload) [H2D inside the graph] + ks_batch_sync (reports + summaries D2H)"},
        "e2e_graph": {"value": E_local * cells * args.steps / e2e_graph_s, "unit": UNIT, "ms_per_step": 1e3 * e2e_graph_s / args.steps,
                      "path": "stage_frame (frame written in the slot's pinned staging area) + upload_frame_async + graph replay + sync/report"},
        "gpu_launches": int(kernel_nodes * args.steps),
        "graph": {"kernel_nodes": int(kernel_nodes), "all_nodes": int(all_nodes)},
        "stage_ms": {k: round(v, 5) for k, v in stage_ms.items()},
        "stages": stage_table,
        "cold_frame_ms": {"value": float(np.median(cold_ms)), "runs": [round(v, 4) for v in cold_ms],
                          "what": "first update of a fresh world (all blocks allocated by this update), plain stream launches, inputs resident in HBM"},
        "roofline": {"bound": "hbm", "kernel": dominant, "achieved": achieved, "peak": peak, "unit": "GB/s",
                     "frac": achieved / peak, "traffic": traffic, "peak_source": peak_src,
                     "algorithmic_bytes_per_launch": stage_bytes[dominant],
                     "update_bytes": update_bytes, "update_frac_of_peak": update_bytes / (ms_per_step * 1e-3) / 1e9 / peak,
                     # SURVEY.md 8(d)'s formulas with ITS assumed formats (byte mask, 4-byte site + f32 distance fields, 21 B/cell of propagate passes):
                     "survey_update_bytes": survey_bytes, "survey_update_frac_of_peak": survey_bytes / (ms_per_step * 1e-3) / 1e9 / peak,
                     "note": "HBM is the nominal roof of every stage (no contraction on this path), but the sweeps are "
                             "instruction-issue bound: see profiles/README.md and profiles/r2/e_ncu_cfg2_k_sweep_x_dc.txt. The device formats move fewer bytes "
                             "than SURVEY 8(d) assumed (bit-packed masks, 4-byte field, phase 1 as bit strings), so frac is quoted on the smaller figure"},
        "cpu_baseline": cpu_base,
    }
    print(json.dumps(line))
    if world > 1:
        dist.destroy_process_group()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--workload", default=None, choices=sorted(WORKLOAD_DESC),
                    help="default: cfg2 on one GPU; cfg5env (BASELINE configs[4]) under torchrun with N > 1")
    ap.add_argument("--envs-per-gpu", type=int, default=None, help="independent environments per rank (cfg5env on N > 1 GPUs: 128 / N)")
    ap.add_argument("--lanes", type=int, default=2, help="streams a batch of environments is dealt onto (ks_batch_create)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    args = ap.parse_args()
    args = resolve_workload(args)
    args.warmup = max(args.warmup, 3) if args.impl == "ours" else args.warmup
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
