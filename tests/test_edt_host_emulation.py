"""The banded lower-envelope code of the CUDA sweeps (csrc/edt_core.cuh is __host__ __device__) run on the
CPU, stage by stage, against the oracle.  This validates the merge/colour logic where no GPU exists; the
product never executes this emulation."""
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
