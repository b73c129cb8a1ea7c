"""Pin the C oracle (oracle/ks_oracle.c) to vectors produced by the reference build
(tests/golden/make_golden.py ran oracle/_ref/libks_ref.so = the reference's own headers)."""
import hashlib
from pathlib import Path

import numpy as np
import pytest

from golden.make_golden import EDT_CASES, SCENE_CASES, d2_from_site, edt_mask, run_scene
from paper_2603_05493_b200 import scenes

GOLD = Path(__file__).resolve().parent / "golden"


@pytest.mark.parametrize("seed,dims,n", EDT_CASES)
def test_edt_matches_reference_vectors(oracle_lib, seed, dims, n):
    gold = np.load(GOLD / "edt_reference.npz")
    has, site, dist = oracle_lib.propagate(edt_mask(seed, dims, n), dims, 0.01)
    assert has
    assert np.array_equal(site.astype(np.int16), gold[f"edt{seed}_site"])
    assert np.array_equal(d2_from_site(site, dims), gold[f"edt{seed}_d2"])
    assert np.array_equal(dist.view(np.uint64), gold[f"edt{seed}_dist"].view(np.uint64))


@pytest.mark.parametrize("seed", sorted(SCENE_CASES))
def test_scene_pipeline_matches_reference_vectors(oracle_lib, seed):
    gold = np.load(GOLD / f"scene{seed}_reference.npz")
    got = run_scene(oracle_lib, scenes.small_scene(seed, **SCENE_CASES[seed]))
    for name in gold.files:
        a, b = got[name], gold[name]
        if a.dtype.kind == "f":  # bitwise, so that -0.0 and inf are pinned too
            assert np.array_equal(np.ascontiguousarray(a).view(np.uint64), b.view(np.uint64)), name
        else:
            assert np.array_equal(a, b), name
