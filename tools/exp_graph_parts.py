"""How much of a replayed update each part costs: the same cfg2 world, graphs with parts left out (CUDA events, 300 replays each)."""
import sys, time
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
sys.path.insert(0, str(Path(__file__).resolve().parent.parent / "tests"))
import numpy as np, torch
from paper_2603_05493_b200 import api, scenes
from parity_util import frame_of, esdf_config

sc = scenes.config2()
stream = torch.cuda.Stream()
cfg = api.make_tsdf_config(sc.tsdf_voxel); cfg.capacity = sc.capacity
t = api.make_tsdf(cfg, stream.cuda_stream)
e = api.DenseEsdf(esdf_config(sc), stream.cuda_stream)
prims = [api.Cuboid(c.R, c.t, c.half_extents) for c in sc.cuboids]
t.stage_frame(frame_of(sc.frames[0]))
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")

def enqueue(integrate, stamp, build):
    if integrate: t.integrate_async()
    if stamp: t.stamp_batch_async(prims)
    if build: e.build_async(t)

with torch.cuda.stream(stream):
    t.upload_frame_async(); enqueue(True, True, True); t.sync()
    for name, parts in [("full", (1, 1, 1)), ("no integrate", (0, 1, 1)), ("no stamps", (1, 0, 1)), ("build only", (0, 0, 1)), ("integrate only", (1, 0, 0)), ("stamps only", (0, 1, 0)), ("tsdf only", (1, 1, 0))]:
        g = api.Graph(stream.cuda_stream)
        with g: enqueue(*parts)
        for _ in range(20): g.launch()
        stream.synchronize()
        ts = []
        for _ in range(100):
            flush.zero_()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(stream); g.launch(); b.record(stream); b.synchronize()
            ts.append(a.elapsed_time(b))
        print(f"{name:15s} {np.median(ts)*1e3:8.1f} us   kernels {g.node_count()[0]}")
        g.close()
