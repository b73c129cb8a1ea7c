"""The C++ drop-in header (include/ks_b200/ks.hpp): one program written against the reference's ks:: API,
built against the reference (golden output, generated where /root/reference is mounted) and against ks_b200."""
import os
import subprocess
import sysconfig
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parent.parent
SRC = ROOT / "tests" / "cpp" / "dropin_program.cpp"
GOLD = ROOT / "tests" / "golden" / "dropin_expected.txt"
STANDIN = ROOT / "oracle" / "eigen_standin"  # Eigen is not installed in this image


def build_b200_variant(out: Path):
    from paper_2603_05493_b200 import build
    build.build()
    lib_dir = ROOT / "paper_2603_05493_b200"
    subprocess.run(["g++", "-std=c++20", "-O2", f"-I{ROOT / 'include'}", f"-I{STANDIN}", str(SRC), "-o", str(out),
                    f"-L{lib_dir}", "-lks_b200", f"-Wl,-rpath,{lib_dir}"], check=True)


def test_program_compiles_against_ks_b200(tmp_path):
    build_b200_variant(tmp_path / "dropin_b200")


def test_golden_output_is_what_the_reference_prints(tmp_path):
    if not os.path.isdir("/root/reference/proj/include"):
        pytest.skip("reference tree not mounted")
    json_inc = Path(sysconfig.get_paths()["purelib"]) / "include" / "cudnn_frontend" / "thirdparty" / "nlohmann"
    exe = tmp_path / "dropin_ref"
    subprocess.run(["g++", "-std=c++20", "-O2", "-ffp-contract=off", "-DUSE_REFERENCE", "-I/root/reference/proj/include",
                    f"-I{STANDIN}", f"-I{json_inc}", str(SRC), "-o", str(exe)], check=True)
    out = subprocess.run([str(exe)], check=True, capture_output=True, text=True).stdout
    assert out == GOLD.read_text()


@pytest.mark.gpu
def test_program_prints_the_reference_output_on_the_gpu(tmp_path):
    exe = tmp_path / "dropin_b200"
    build_b200_variant(exe)
    out = subprocess.run([str(exe)], check=True, capture_output=True, text=True).stdout
    assert out == GOLD.read_text()
