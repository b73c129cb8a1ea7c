"""tools/esdf_bench.cpp: the spec's `ks esdf-bench` command (SPEC.md cmd_esdf_bench) over the drop-in header.
CPU: it builds, and usage / parse errors exit 2 before any device is touched.  GPU: the spec's examples
(stamped sphere with --brute-force: max |delta d| = 0 voxels, recall 1.0; empty scene: graceful no-seed report;
every emitted file parses)."""
import csv
import json
import subprocess
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parent.parent
SRC = ROOT / "tools" / "esdf_bench.cpp"
STANDIN = ROOT / "oracle" / "eigen_standin"  # Eigen is not installed in this image


def build_cli(out: Path) -> Path:
    from paper_2603_05493_b200 import build
    build.build()
    lib_dir = ROOT / "paper_2603_05493_b200"
    subprocess.run(["g++", "-std=c++20", "-O2", f"-I{ROOT / 'include'}", f"-I{STANDIN}", str(SRC), "-o", str(out),
                    f"-L{lib_dir}", "-lks_b200", f"-Wl,-rpath,{lib_dir}"], check=True)
    return out


SPHERE = {"world": {"spheres": [{"center": [0.32, 0.3, 0.28], "radius": 0.15}],
                    "cuboids": [{"center": [0.1, 0.5, 0.1], "half_extents": [0.05, 0.04, 0.06], "rpy": [0.0, 0.0, 0.4]}]},
          "tsdf": {"voxel_size": 0.01, "capacity": 16384},
          "esdf": {"origin": [0.0, 0.0, 0.0], "dims": [64, 60, 56], "voxel_size": 0.01, "seeding": "gather"}}


def test_usage_and_parse_errors_exit_2(tmp_path):
    exe = build_cli(tmp_path / "esdf-bench")
    assert subprocess.run([str(exe)], capture_output=True).returncode == 2
    assert subprocess.run([str(exe), "scenario.json"], capture_output=True).returncode == 2          # no -o
    assert subprocess.run([str(exe), "x.json", "-o", str(tmp_path), "--seeding", "both"], capture_output=True).returncode == 2
    bad = tmp_path / "bad.json"
    bad.write_text('{"esdf": {"origin": [0, 0, 0], "dims": [8, 8')
    r = subprocess.run([str(exe), str(bad), "-o", str(tmp_path / "out")], capture_output=True, text=True)
    assert r.returncode == 2 and "scenario:" in r.stderr
    missing = subprocess.run([str(exe), str(tmp_path / "nope.json"), "-o", str(tmp_path / "out")], capture_output=True, text=True)
    assert missing.returncode == 2


@pytest.mark.gpu
def test_stamped_sphere_with_brute_force(tmp_path):
    exe = build_cli(tmp_path / "esdf-bench")
    scenario = tmp_path / "sphere.json"
    scenario.write_text(json.dumps(SPHERE))
    out = tmp_path / "out"
    r = subprocess.run([str(exe), str(scenario), "-o", str(out), "--brute-force"], capture_output=True, text=True)
    assert r.returncode == 0, r.stderr
    summary = json.loads((out / "summary.json").read_text())
    assert summary["cells"] == 64 * 60 * 56 and summary["tsdf_blocks"] > 0
    assert summary["modes"]["gather"]["seeds"] >= summary["modes"]["scatter"]["seeds"] > 0   # SPEC acceptance #10 ordering
    timings = list(csv.DictReader((out / "timings.csv").open()))
    assert {t["stage"] for t in timings} == {"integrate", "stamp", "seed", "propagate", "recover_signs", "build_esdf"}
    assert all(float(t["median_ms"]) >= 0.0 and int(t["repetitions"]) == 10 for t in timings)
    rows = list(csv.DictReader((out / "recall.csv").open()))
    brute = [x for x in rows if x["truth"] == "brute-force-cells"]
    assert len(brute) == 2 and all(float(x["max_abs_delta_voxels"]) == 0.0 for x in brute)    # exact EDT: 0 voxels off
    gather4 = [x for x in rows if x["seeding"] == "gather" and x["truth"] == "analytic" and float(x["radius_voxels"]) == 4.0][0]
    assert int(gather4["truth_positive"]) > 100 and float(gather4["recall"]) >= 0.97           # SPEC acceptance #9 bar
    assert float(gather4["max_abs_delta_voxels"]) <= 3.0   # seed band (0.9 v each side) + trilinear sampling


@pytest.mark.gpu
def test_empty_scene_reports_no_seeds(tmp_path):
    exe = build_cli(tmp_path / "esdf-bench")
    far = {"world": {"spheres": [{"center": [5.0, 5.0, 5.0], "radius": 0.05}]}, "tsdf": {"voxel_size": 0.02, "capacity": 1024},
           "esdf": {"origin": [0.0, 0.0, 0.0], "dims": [16, 16, 16], "voxel_size": 0.02}}
    scenario = tmp_path / "far.json"
    scenario.write_text(json.dumps(far))
    out = tmp_path / "out"
    r = subprocess.run([str(exe), str(scenario), "-o", str(out), "--seeding", "gather"], capture_output=True, text=True)
    assert r.returncode == 0, r.stderr
    summary = json.loads((out / "summary.json").read_text())
    assert summary["modes"]["gather"] == {"seeds": 0, "has_sites": False, "brute_force_max_abs_delta_voxels": None}
    none = subprocess.run([str(exe), str(scenario).replace("far", "far2"), "-o", str(out)], capture_output=True)
    assert none.returncode == 2
    nothing = tmp_path / "nothing.json"
    nothing.write_text(json.dumps({"esdf": far["esdf"]}))
    r = subprocess.run([str(exe), str(nothing), "-o", str(out)], capture_output=True, text=True)
    assert r.returncode == 1 and "neither depth frames nor primitives" in r.stderr
