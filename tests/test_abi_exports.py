"""CPU-side checks of the drop-in boundary: the library loads and exports exactly the symbols that
include/ks_b200.h declares; compute calls fail loudly without a device (no CPU fallback)."""
import ctypes
import re
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parent.parent


@pytest.fixture(scope="module")
def lib():
    from paper_2603_05493_b200 import build
    build.build()
    from paper_2603_05493_b200 import api
    return api.load_library()


def declared_symbols():
    text = (ROOT / "include" / "ks_b200.h").read_text()
    return sorted(set(re.findall(r"KS_API\s+[\w\s\*]+?\b(ks_\w+)\s*\(", text)))


def test_header_and_binding_agree(lib):
    from paper_2603_05493_b200 import api
    assert declared_symbols() == sorted(api.ABI_SYMBOLS)


def test_every_declared_symbol_is_exported(lib):
    for name in declared_symbols():
        assert hasattr(lib, name), name


def test_no_torch_or_oracle_in_the_product_library():
    import subprocess
    out = subprocess.run(["ldd", str(ROOT / "paper_2603_05493_b200" / "libks_b200.so")], capture_output=True, text=True).stdout
    assert "torch" not in out and "oracle" not in out and "ks_ref" not in out
    for src in (ROOT / "paper_2603_05493_b200").rglob("*"):
        if src.suffix in {".py", ".cu", ".cuh", ".h", ".hpp"}:
            body = src.read_text()
            assert "liboracle" not in body and "cpu_checkers" not in body and "ks_oracle" not in body, src


def test_compute_fails_loudly_without_a_device(lib):
    from paper_2603_05493_b200 import api
    if lib.ks_device_count() > 0:
        pytest.skip("a CUDA device is present")
    with pytest.raises(api.CudaError, match="no CUDA device"):
        api.make_tsdf(api.make_tsdf_config(0.01))
    with pytest.raises(api.CudaError, match="no CUDA device"):
        api.DenseEsdf(api.EsdfConfig(nx=4, ny=4, nz=4))


def test_batch_fails_loudly_without_a_device_and_partitions_on_the_host(lib):
    """ks_batch_create has no CPU path either; ks_partition_envs is host code (the N > 1 launcher calls it before any GPU work)."""
    from paper_2603_05493_b200 import api
    assert [api.partition_envs(128, 8, r) for r in (0, 7)] == [(0, 16), (112, 128)]
    assert [api.partition_envs(5, 3, r) for r in range(3)] == [(0, 2), (2, 4), (4, 5)]
    with pytest.raises(ValueError, match="bad partition arguments"):
        api.partition_envs(4, 2, 2)
    if lib.ks_device_count() > 0:
        pytest.skip("a CUDA device is present")
    with pytest.raises(api.CudaError):
        api.EnvBatch(2, api.make_tsdf_config(0.01), api.EsdfConfig(nx=4, ny=4, nz=4))


def test_validation_messages_match_the_reference(lib):
    from paper_2603_05493_b200 import api
    cases = [
        (dict(voxel_size=0.0), "tsdf: voxel_size must be > 0"),
        (dict(voxel_size=0.01, truncation=0.001), "tsdf: truncation must be >= voxel_size"),
        (dict(alpha_time=0.0), r"tsdf: decay factors must lie in \(0, 1\]"),
        (dict(capacity=0), "tsdf: capacity must be >= 1"),
    ]
    for kw, msg in cases:  # validation happens before any device work (sdf_world.hpp:47-53)
        with pytest.raises(api.ValidationError, match=msg):
            api.make_tsdf(api.TsdfConfig(**kw))
    with pytest.raises(api.ValidationError, match="esdf: dims must be >= 1"):
        api.DenseEsdf(api.EsdfConfig(nx=0, ny=4, nz=4))
    with pytest.raises(api.ValidationError, match="esdf: voxel_size must be > 0"):
        api.DenseEsdf(api.EsdfConfig(nx=2, ny=2, nz=2, voxel_size=-1.0))
