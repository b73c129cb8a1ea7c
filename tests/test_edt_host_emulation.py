"""The sweep code of the CUDA kernels (csrc/edt_dc.cuh: monotone divide and conquer; csrc/edt_core.cuh: banded
stacks, the fallback for very large grids; both __host__ __device__) run on the CPU, stage by stage, against
the oracle.  This validates the level / merge / colour logic where no GPU exists; the product never executes
this emulation."""
import ctypes as C
import subprocess
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent.parent


def test_banded_sweeps_match_oracle_sites(oracle_lib, tmp_path):
    so = tmp_path / "libedt_emul.so"
    subprocess.run(["g++", "-O2", "-shared", "-fPIC", "-o", str(so), str(ROOT / "tests" / "host_emul" / "edt_emul.cpp")], check=True)
    lib = C.CDLL(str(so))
    rng = np.random.RandomState(0)
    for trial in range(120):
        dims = tuple(int(v) for v in rng.randint(1, 60, 3))
        if trial % 7 == 0:
            dims = (int(rng.randint(1, 200)), int(rng.randint(1, 5)), int(rng.randint(1, 5)))
        cells = dims[0] * dims[1] * dims[2]
        mask = (rng.random_sample(cells) < rng.choice([0.0005, 0.003, 0.02, 0.3, 0.9])).astype(np.uint8)
        if mask.sum() == 0:
            mask[rng.randint(cells)] = 1
        band_y, band_x = int(rng.choice([1, 2, 3, 5, 8, 16, 64])), int(rng.choice([1, 2, 3, 5, 8, 16, 64]))
        site = np.empty((cells, 3), np.int32)
        d2 = np.empty(cells, np.int32)
        lib.emul_propagate(mask.ctypes.data_as(C.c_void_p), dims[0], dims[1], dims[2], band_y, band_x,
                           site.ctypes.data_as(C.c_void_p), d2.ctypes.data_as(C.c_void_p))
        _, site0, _ = oracle_lib.propagate(mask, dims, 1.0)
        assert np.array_equal(site, site0), (dims, band_y, band_x)


def _emul_lib(tmp_path):
    so = tmp_path / "libedt_emul.so"
    subprocess.run(["g++", "-O2", "-shared", "-fPIC", "-o", str(so), str(ROOT / "tests" / "host_emul" / "edt_emul.cpp")], check=True)
    return C.CDLL(str(so))


def _run_dc(lib, mask, dims, warps_log2, fuzz=0):
    cells = mask.size
    site = np.empty((cells, 3), np.int32)
    d2 = np.empty(cells, np.int32)
    stats = (C.c_longlong * 4)()
    rc = lib.emul_propagate_dc(mask.ctypes.data_as(C.c_void_p), dims[0], dims[1], dims[2], warps_log2, fuzz,
                               site.ctypes.data_as(C.c_void_p), d2.ctypes.data_as(C.c_void_p), stats)
    assert rc == 0
    return site, d2, list(stats)


def test_divide_and_conquer_sweeps_match_oracle_sites(oracle_lib, tmp_path):
    lib = _emul_lib(tmp_path)
    rng = np.random.RandomState(1)
    for trial in range(150):
        dims = tuple(int(v) for v in rng.randint(1, 60, 3))
        if trial % 7 == 0:
            dims = (int(rng.randint(1, 300)), int(rng.randint(1, 5)), int(rng.randint(1, 5)))
        if trial % 11 == 0:
            dims = (int(rng.randint(1, 5)), int(rng.randint(1, 300)), int(rng.randint(1, 40)))
        cells = dims[0] * dims[1] * dims[2]
        mask = (rng.random_sample(cells) < rng.choice([0.0005, 0.003, 0.02, 0.3, 0.9])).astype(np.uint8)
        if mask.sum() == 0:
            mask[rng.randint(cells)] = 1
        warps_log2 = int(rng.choice([0, 1, 2, 3, 4]))
        site, d2, _ = _run_dc(lib, mask, dims, warps_log2, fuzz=int(rng.choice([0, 0, 1, 3, 40])))
        _, site0, dist0 = oracle_lib.propagate(mask, dims, 1.0)
        assert np.array_equal(site, site0), (dims, warps_log2)
        assert np.array_equal(np.sqrt(d2.astype(np.float64)), dist0), (dims, warps_log2)


def test_divide_and_conquer_edge_cases(oracle_lib, tmp_path):
    lib = _emul_lib(tmp_path)
    # rows with no seed at all, a single seed in a corner, fully seeded, and the tie rule (earlier site wins)
    for dims, seeds in [((9, 7, 5), [(8, 6, 4)]), ((9, 7, 5), [(0, 0, 0), (8, 0, 0)]), ((33, 2, 1), [(0, 0, 0), (32, 1, 0)]),
                        ((5, 5, 5), [(0, 2, 2), (4, 2, 2), (2, 0, 2), (2, 4, 2), (2, 2, 0), (2, 2, 4)]), ((64, 1, 1), [(31, 0, 0)])]:
        mask = np.zeros(dims[0] * dims[1] * dims[2], np.uint8)
        for (x, y, z) in seeds:
            mask[x + dims[0] * (y + dims[1] * z)] = 1
        for warps_log2 in (0, 2, 4):
            site, _, _ = _run_dc(lib, mask, dims, warps_log2)
            _, site0, _ = oracle_lib.propagate(mask, dims, 1.0)
            assert np.array_equal(site, site0), (dims, seeds, warps_log2)
    full = np.ones(6 * 5 * 4, np.uint8)
    site, d2, _ = _run_dc(lib, full, (6, 5, 4), 3)
    assert not d2.any()
    # key range: the library must fall back to the stack sweeps exactly when a key could overflow
    assert lib.emul_dc_fits(400, 200, 200) == 1 and lib.emul_dc_fits(500, 500, 500) == 1
    assert lib.emul_dc_fits(1024, 600, 600) == 1 and lib.emul_dc_fits(1024, 1024, 1024) == 0
