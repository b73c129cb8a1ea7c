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
    subprocess.run(["g++", "-std=c++20", "-O2", f"-I{ROOT / 'include' / 'ks_b200' / 'overlay'}", f"-I{ROOT / 'include'}", f"-I{STANDIN}",
                    str(SRC), "-o", str(out), f"-L{lib_dir}", "-lks_b200", f"-Wl,-rpath,{lib_dir}"], check=True)


def test_program_compiles_against_ks_b200(tmp_path):
    build_b200_variant(tmp_path / "dropin_b200")


def test_golden_output_is_what_the_reference_prints(tmp_path):
    if not os.path.isdir("/root/reference/proj/include"):
        pytest.skip("reference tree not mounted")
    json_inc = Path(sysconfig.get_paths()["purelib"]) / "include" / "cudnn_frontend" / "thirdparty" / "nlohmann"
    exe = tmp_path / "dropin_ref"
    subprocess.run(["g++", "-std=c++20", "-O2", "-ffp-contract=off", "-DUSE_REFERENCE", f"-I{ROOT / 'oracle' / 'ref_stubs'}",
                    "-I/root/reference/proj/include", f"-I{STANDIN}", f"-I{json_inc}", str(SRC), "-o", str(exe)], check=True)
    out = subprocess.run([str(exe), str(tmp_path)], check=True, capture_output=True, text=True).stdout
    assert out == GOLD.read_text()


@pytest.mark.gpu
def test_program_prints_the_reference_output_on_the_gpu(tmp_path):
    exe = tmp_path / "dropin_b200"
    build_b200_variant(exe)
    out = subprocess.run([str(exe), str(tmp_path)], check=True, capture_output=True, text=True).stdout
    assert out == GOLD.read_text()


# ---- KSDEPTH1 / KSESDF1 files: host-only, so checked on the CPU too -------------------------------------
FILEIO = ROOT / "tests" / "cpp" / "fileio_program.cpp"
G = ROOT / "tests" / "golden"


def _build_fileio(out: Path, reference: bool):
    if reference:
        json_inc = Path(sysconfig.get_paths()["purelib"]) / "include" / "cudnn_frontend" / "thirdparty" / "nlohmann"
        cmd = ["g++", "-std=c++20", "-O2", "-ffp-contract=off", "-DUSE_REFERENCE", "-I/root/reference/proj/include",
               f"-I{STANDIN}", f"-I{json_inc}", str(FILEIO), "-o", str(out)]
    else:
        from paper_2603_05493_b200 import build
        build.build()
        lib_dir = ROOT / "paper_2603_05493_b200"
        cmd = ["g++", "-std=c++20", "-O2", f"-I{ROOT / 'include'}", f"-I{STANDIN}", str(FILEIO), "-o", str(out), f"-L{lib_dir}",
               "-lks_b200", f"-Wl,-rpath,{lib_dir}"]
    subprocess.run(cmd, check=True)


def test_reads_files_written_by_the_reference(tmp_path):
    exe = tmp_path / "fileio_b200"
    _build_fileio(exe, reference=False)
    out = subprocess.run([str(exe), "read", str(G / "frame_reference.ksdepth"), str(G / "field_reference.ksesdf"),
                          str(tmp_path / "resaved.ksdepth")], check=True, capture_output=True, text=True).stdout
    assert out == (G / "fileio_expected.txt").read_text()
    # what we write reads back to the same values
    again = subprocess.run([str(exe), "read", str(tmp_path / "resaved.ksdepth"), str(G / "field_reference.ksesdf"),
                            str(tmp_path / "again.ksdepth")], check=True, capture_output=True, text=True).stdout
    assert again == out


def test_reference_reads_files_written_by_us(tmp_path):
    if not os.path.isdir("/root/reference/proj/include"):
        pytest.skip("reference tree not mounted")
    ours, ref = tmp_path / "fileio_b200", tmp_path / "fileio_ref"
    _build_fileio(ours, reference=False)
    _build_fileio(ref, reference=True)
    subprocess.run([str(ours), "read", str(G / "frame_reference.ksdepth"), str(G / "field_reference.ksesdf"),
                    str(tmp_path / "ours.ksdepth")], check=True, capture_output=True)
    out = subprocess.run([str(ref), "read", str(tmp_path / "ours.ksdepth"), str(G / "field_reference.ksesdf"),
                          str(tmp_path / "x.ksdepth")], check=True, capture_output=True, text=True).stdout
    assert out == (G / "fileio_expected.txt").read_text()


# ---- ks.hpp's mesh additions (no reference counterpart: SPEC.md:8) ---------------------------------------
MESH = ROOT / "tests" / "cpp" / "mesh_program.cpp"


def _build_mesh_program(out: Path):
    from paper_2603_05493_b200 import build
    build.build()
    lib_dir = ROOT / "paper_2603_05493_b200"
    subprocess.run(["g++", "-std=c++20", "-O2", f"-I{ROOT / 'include'}", f"-I{STANDIN}", str(MESH), "-o", str(out),
                    f"-L{lib_dir}", "-lks_b200", f"-Wl,-rpath,{lib_dir}"], check=True)


def test_mesh_program_compiles(tmp_path):
    _build_mesh_program(tmp_path / "mesh_b200")


@pytest.mark.gpu
def test_mesh_program_box_mesh_equals_cuboid_stamp(tmp_path):
    exe = tmp_path / "mesh_b200"
    _build_mesh_program(exe)
    out = subprocess.run([str(exe)], check=True, capture_output=True, text=True).stdout.splitlines()
    assert out[0].startswith("triangles 12 blocks ") and out[0].split()[-1] == out[0].split()[-2] != "0"
    assert out[1] == "compared many missing 0 worst ok"
    assert out[2] == "ValidationError: stamp: degenerate mesh triangle"


# ---- mixing with the reference's OWN planner headers (collision.hpp, the way ik.hpp:23 / :117-120 uses the field) ----------
MIXED = ROOT / "tests" / "cpp" / "mixed_program.cpp"
MIXED_GOLD = ROOT / "tests" / "golden" / "mixed_expected.txt"
MIXED_EXE = ROOT / "tests" / "cpp" / "_built" / "mixed_b200"  # built where /root/reference is mounted; travels to the GPU box
REF_INC = Path("/root/reference/proj/include")


def build_mixed(out: Path, reference: bool):
    json_inc = Path(sysconfig.get_paths()["purelib"]) / "include" / "cudnn_frontend" / "thirdparty" / "nlohmann"
    common = [f"-I{ROOT / 'oracle' / 'ref_stubs'}", f"-I{REF_INC}", f"-I{STANDIN}", f"-I{json_inc}", str(MIXED), "-o", str(out)]
    if reference:
        cmd = ["g++", "-std=c++20", "-O2", "-ffp-contract=off"] + common
    else:
        from paper_2603_05493_b200 import build
        build.build()
        out.parent.mkdir(parents=True, exist_ok=True)
        # the overlay directory first: "ks/sdf_world.hpp", "ks/esdf.hpp", "ks/collision.hpp" resolve there
        cmd = ["g++", "-std=c++20", "-O2", f"-I{ROOT / 'include' / 'ks_b200' / 'overlay'}", f"-I{ROOT / 'include'}"] + common + [
            f"-L{ROOT / 'paper_2603_05493_b200'}", "-lks_b200", "-Wl,-rpath,$ORIGIN/../../../paper_2603_05493_b200"]
    subprocess.run(cmd, check=True)


def test_mixed_program_builds_against_the_reference_and_against_the_overlay(tmp_path):
    """One source, no ks_b200 name in it: reference build prints the golden text; the overlay build must compile with the
    reference's own collision.hpp in the same translation unit (self_collision stays the reference's)."""
    if not REF_INC.is_dir():
        pytest.skip("reference tree not mounted")
    ref = tmp_path / "mixed_ref"
    build_mixed(ref, reference=True)
    out = subprocess.run([str(ref)], check=True, capture_output=True, text=True).stdout
    assert out == MIXED_GOLD.read_text()
    build_mixed(MIXED_EXE, reference=False)
    syms = subprocess.run(["nm", "-C", "--undefined-only", str(MIXED_EXE)], check=True, capture_output=True, text=True).stdout
    assert "ks_esdf_scene_collision_static" in syms and "ks_esdf_scene_collision_swept" in syms  # the GPU versions are the ones called


def test_header_order_without_the_overlay(tmp_path):
    """ks_b200/ks.hpp first, then the reference's collision.hpp, no overlay directory on the include path."""
    if not REF_INC.is_dir():
        pytest.skip("reference tree not mounted")
    src = tmp_path / "order.cpp"
    src.write_text('#include "ks_b200/ks.hpp"\n#include "ks/collision.hpp"\n#include "ks/esdf.hpp"\n#include "ks/sdf_world.hpp"\n'
                   "int main() { ks::RobotModel m; std::vector<ks::Vec3> c; ks::DenseEsdf e;\n"
                   "  return ks::self_collision(m, c).worst_first + (&e == nullptr ? ks::scene_collision_static(e, c, m.sphere_radius).worst_first : 0); }\n")
    json_inc = Path(sysconfig.get_paths()["purelib"]) / "include" / "cudnn_frontend" / "thirdparty" / "nlohmann"
    subprocess.run(["g++", "-std=c++20", "-O1", "-fsyntax-only", f"-I{ROOT / 'include'}", f"-I{ROOT / 'oracle' / 'ref_stubs'}", f"-I{REF_INC}",
                    f"-I{STANDIN}", f"-I{json_inc}", str(src)], check=True)


@pytest.mark.gpu
def test_mixed_program_prints_the_reference_output_on_the_gpu():
    if REF_INC.is_dir():
        build_mixed(MIXED_EXE, reference=False)
    if not MIXED_EXE.exists():
        pytest.skip("tests/cpp/_built/mixed_b200 was not prebuilt (needs /root/reference at build time) and no reference tree here")
    out = subprocess.run([str(MIXED_EXE)], check=True, capture_output=True, text=True).stdout
    assert out == MIXED_GOLD.read_text()


# ---- ks::EnvironmentBatch (the batch API the reference lacks) against the free functions of the same header ------
BATCH = ROOT / "tests" / "cpp" / "batch_program.cpp"


def _build_batch_program(out: Path):
    from paper_2603_05493_b200 import build
    build.build()
    lib_dir = ROOT / "paper_2603_05493_b200"
    subprocess.run(["g++", "-std=c++20", "-O2", f"-I{ROOT / 'include'}", f"-I{STANDIN}", str(BATCH), "-o", str(out),
                    f"-L{lib_dir}", "-lks_b200", f"-Wl,-rpath,{lib_dir}"], check=True)


def test_batch_program_compiles(tmp_path):
    _build_batch_program(tmp_path / "batch_b200")


@pytest.mark.gpu
def test_batch_program_every_environment_equals_its_own_world(tmp_path):
    exe = tmp_path / "batch_b200"
    _build_batch_program(exe)
    out = subprocess.run([str(exe)], check=True, capture_output=True, text=True).stdout.splitlines()
    assert len(out) == 4, out
    for k, line in enumerate(out[:3]):
        f = line.split()
        assert f[:4] == ["env", str(100 + k), "same", "1"] and f[4:6] == ["cells", "60000"], line
        assert f[8:] == ["summary", "1", "1", "1", "flags", "1", "1"], line
    assert out[3] == "ValidationError: environment 8: tsdf: pool exhausted, frame r"
