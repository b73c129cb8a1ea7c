"""Generate tests/golden/mesh_restatement.npz from oracle/liboracle.so.

NOT reference output: the reference has no mesh implementation, so this fixture pins this repo's
own definition (oracle/ks_oracle.c "triangle mesh stamping", csrc/mesh.cuh) against silent change -- a regression
vector for the restatement and, through tests/test_mesh_stamp.py, for the CUDA path.
    python tests/golden/make_mesh_golden.py
"""
import sys
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
sys.path.insert(0, str(HERE.parent))
sys.path.insert(0, str(HERE.parent.parent))

import cpu_checkers  # noqa: E402
from paper_2603_05493_b200 import scenes  # noqa: E402


def cases():
    """name -> (mesh, query points)"""
    rng = np.random.RandomState(21)
    out = {}
    for name, mesh in (("box", scenes.box_mesh((0.3, 0.2, 0.5), (0.2, 0.1, 0.15), scenes.rot_z(0.4) @ scenes.rot_y(0.2))),
                       ("ico2", scenes.icosphere((0.1, -0.2, 0.3), 0.2, 2))):
        c = mesh.vertices.mean(axis=0)
        out[name] = (mesh, c + (rng.random_sample((4096, 3)) - 0.5) * 0.9)
    return out


def stamped_world(lib):
    """A world with both meshes stamped: sorted keys and their geometry channels."""
    t = lib.make_tsdf(0.02, capacity=4096)
    for mesh, _ in cases().values():
        t.stamp_mesh(mesh.vertices, mesh.triangles)
    keys, pool = t.export_blocks()
    order = np.lexsort((keys[:, 2], keys[:, 1], keys[:, 0]))
    geom = np.stack([t.block_channels(int(p))[2] for p in pool[order]])
    return keys[order], geom


def main():
    lib = cpu_checkers.oracle()
    out = {}
    for name, (mesh, pts) in cases().items():
        out[f"{name}_sdf"] = lib.mesh_sdf(mesh.vertices, mesh.triangles, pts)
    out["world_keys"], out["world_geom"] = stamped_world(lib)
    np.savez_compressed(HERE / "mesh_restatement.npz", **out)
    print({k: v.shape for k, v in out.items()})


if __name__ == "__main__":
    main()
