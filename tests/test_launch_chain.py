"""Programmatic dependent launch (csrc/common.cuh launch_kernel / pdl_enter) must not change a single bit: the same
update with KS_B200_NO_PDL=1 (plain stream-ordered launches) and with the default launches, plain and as a captured
CUDA graph, compared through hashes of the exported world and field."""
import hashlib
import json
import os
import subprocess
import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parent.parent

SCRIPT = r"""
import hashlib, json, sys
sys.path.insert(0, {root!r}); sys.path.insert(0, {root!r} + "/tests")
import numpy as np
from paper_2603_05493_b200 import api, scenes
from parity_util import esdf_config, frame_of, gpu_world

def digest(*arrays):
    h = hashlib.sha256()
    for a in arrays:
        h.update(np.ascontiguousarray(a).tobytes())
    return h.hexdigest()

out = {{}}
scene = scenes.small_scene(4)
scene.meshes.append(scenes.icosphere(scene.esdf_origin + 0.4 * np.array(scene.esdf_dims) * scene.esdf_voxel, 0.15, 2))
tsdf, touched = gpu_world(scene)
keys, pool = tsdf.export_blocks()
esdf = api.build_esdf(tsdf, esdf_config(scene))
site, dist, d2 = esdf.download()
out["plain"] = digest(keys, pool, *tsdf.download_blocks(pool.tolist()), site, dist, d2)
# the same update again as ONE captured graph on a fresh world, replayed twice
import torch
stream = torch.cuda.Stream()
cfg = api.make_tsdf_config(scene.tsdf_voxel); cfg.capacity = scene.capacity
t2 = api.make_tsdf(cfg, stream.cuda_stream)
e2 = api.DenseEsdf(esdf_config(scene), stream.cuda_stream)
mesh = api.TriangleMesh(scene.meshes[0].vertices, scene.meshes[0].triangles)
for slot, f in enumerate(scene.frames):
    t2.stage_frame(frame_of(f), slot)
def enqueue():
    for slot in range(len(scene.frames)):
        t2.upload_frame_async(slot); t2.integrate_async(slot)
    for c in scene.cuboids: t2.stamp_async(api.Cuboid(c.R, c.t, c.half_extents))
    for s in scene.spheres: t2.stamp_async(api.SphereShape(s.center, s.radius))
    t2.stamp_async(mesh)
    e2.build_async(t2)
enqueue(); t2.sync(); e2.report()         # first pass allocates; the graph below re-integrates into the same blocks
g = api.Graph(stream.cuda_stream)
with g:
    enqueue()
out["graph_nodes"] = list(g.node_count())
g.launch(); g.launch(); t2.sync(); e2.report()
site2, dist2, d22 = e2.download()
out["graph"] = digest(site2, d22, np.signbit(dist2))
print("RESULT " + json.dumps(out))
"""


def _run(no_pdl: bool):
    env = dict(os.environ)
    env.pop("KS_B200_NO_PDL", None)
    if no_pdl:
        env["KS_B200_NO_PDL"] = "1"
    proc = subprocess.run([sys.executable, "-c", SCRIPT.format(root=str(ROOT))], env=env, capture_output=True, text=True, timeout=600)
    assert proc.returncode == 0, proc.stderr[-2000:]
    line = [l for l in proc.stdout.splitlines() if l.startswith("RESULT ")][-1]
    return json.loads(line[len("RESULT "):])


@pytest.mark.gpu
def test_programmatic_launch_changes_nothing():
    with_pdl, without = _run(False), _run(True)
    assert with_pdl["plain"] == without["plain"]
    assert with_pdl["graph"] == without["graph"]
    assert with_pdl["graph_nodes"] == without["graph_nodes"] and with_pdl["graph_nodes"][0] > 10
