"""The C++ drop-in API (include/salvox/*.hpp over the C-ABI): builds with g++,
runs the reference's doctest cases ported in tests/cpp/test_host_api.cpp, and
drives the salvox-b200 CLI."""
import json
import os
import subprocess

import numpy as np
import pytest

from tests import phantoms

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CPP = os.path.join(ROOT, "cpp")


@pytest.fixture(scope="module")
def cpp_build(sx):
    subprocess.run(["make", "-s", "-C", CPP, "all", "test_host_api"], check=True)
    return CPP


def _fnv(b: bytes) -> str:
    h = 0xcbf29ce484222325
    for x in b:
        h = ((h ^ x) * 0x100000001b3) & 0xFFFFFFFFFFFFFFFF
    return f"{h:016x}"


def test_cpp_api_host_cases(cpp_build, oracle):
    r = subprocess.run([os.path.join(cpp_build, "test_host_api"), "cpu"], capture_output=True,
                       text=True)
    assert r.returncode == 0, r.stdout + r.stderr
    # the C++ make_phantom is bit-identical to the oracle's restatement
    line = [ln for ln in r.stdout.splitlines() if ln.startswith("phantom404")][0]
    vol, _ = oracle.make_phantom(phantoms.ball_3d(
        48, (24.0, 24.0, 24.0), 8.0, 404, background={"type": "gaussian", "mean": 8.0,
                                                       "sigma": 2.0}))
    assert line.split()[1] == _fnv(vol.tobytes())


def test_cli_phantom_and_config_errors(cpp_build, tmp_path):
    spec = tmp_path / "spec.json"
    spec.write_text(json.dumps(phantoms.square_2d(64, 31.0, 31.0, 8, 64, 77)))
    cli = os.path.join(cpp_build, "salvox-b200")
    r = subprocess.run([cli, "phantom", str(spec), str(tmp_path / "sq.mhd")], capture_output=True,
                       text=True)
    assert r.returncode == 0, r.stderr
    assert (tmp_path / "sq.raw").stat().st_size == 64 * 64 * 4
    assert json.loads((tmp_path / "sq.gt.json").read_text())["regions"]
    bad = tmp_path / "bad.json"
    bad.write_text('{"bogus": 1}')
    r = subprocess.run([cli, "detect", "--config", str(bad), "--volume", str(tmp_path / "sq.mhd"),
                        "--out", str(tmp_path / "o.json")], capture_output=True, text=True)
    assert r.returncode == 1 and "unknown key" in r.stderr


@pytest.mark.gpu
def test_cpp_api_device_cases(cpp_build):
    r = subprocess.run([os.path.join(cpp_build, "test_host_api"), "gpu"], capture_output=True,
                       text=True)
    assert r.returncode == 0, r.stdout + r.stderr


@pytest.mark.gpu
def test_cli_detect_and_exhaustive(cpp_build, tmp_path, oracle):
    spec = tmp_path / "spec.json"
    spec.write_text(json.dumps(phantoms.square_2d(96, 45.0, 49.0, 9, 64, 303)))
    cli = os.path.join(cpp_build, "salvox-b200")
    subprocess.run([cli, "phantom", str(spec), str(tmp_path / "v.mhd")], check=True)
    out = tmp_path / "r.json"
    args = [cli, "detect", "--volume", str(tmp_path / "v.mhd"), "--out", str(out), "--method",
            "quadrant", "--window", "0:64", "--bins", "64", "--seeds", "lattice:12",
            "--scales", "6,10", "--k", "3", "--dedupe-radius", "8"]
    r = subprocess.run(args, capture_output=True, text=True)
    assert r.returncode == 0, r.stderr
    rep = json.loads(out.read_text())
    assert rep["header"]["volume_dims"] == [96, 96, 1] and rep["detections"]
    # byte-identical reports apart from wall time (test_cli.cpp:120-135)
    out2 = tmp_path / "r2.json"
    subprocess.run(args[:5] + [str(out2)] + args[6:], check=True, capture_output=True)
    a, b = json.loads(out.read_text()), json.loads(out2.read_text())
    a["header"].pop("wall_time_ms")
    b["header"].pop("wall_time_ms")
    assert a == b
    mx = tmp_path / "m.json"
    r = subprocess.run([cli, "exhaustive", "--volume", str(tmp_path / "v.mhd"), "--out", str(mx),
                        "--window", "0:64", "--bins", "64", "--scales", "6,9,12",
                        "--budget", "1000000000"], capture_output=True, text=True)
    assert r.returncode == 0, r.stderr
    got = json.loads(mx.read_text())["maxima"]
    vol, _ = oracle.make_phantom(phantoms.square_2d(96, 45.0, 49.0, 9, 64, 303))
    s, b_, _ = oracle.exhaustive(vol, 0, 64, 64, [6.0, 9.0, 12.0], budget=10**9)
    pos = oracle.local_maxima(s, b_)[0]
    assert np.allclose(got[0]["position"], pos[0])
    # a constant volume has no detections: exit code 2 (tools/main.cpp:147)
    flat = {"dims": [48, 48, 1], "background": {"type": "constant", "value": 3.0}, "regions": []}
    spec.write_text(json.dumps(flat))
    subprocess.run([cli, "phantom", str(spec), str(tmp_path / "f.mhd")], check=True)
    r = subprocess.run([cli, "detect", "--volume", str(tmp_path / "f.mhd"), "--out", str(out),
                        "--window", "0:64", "--seeds", "lattice:16", "--scales", "6"],
                       capture_output=True, text=True)
    assert r.returncode == 2, r.stderr


@pytest.mark.gpu
def test_cli_eval_jaccard(cpp_build, tmp_path):  # test_cli.cpp:169-192
    cli = os.path.join(cpp_build, "salvox-b200")
    ball = {"dims": [48, 48, 48],
            "regions": [{"shape": "ball", "center": [24, 22, 25], "radius": 8,
                         "fill": {"type": "uniform", "levels": 64}}], "rng_seed": 5}
    (tmp_path / "spec.json").write_text(json.dumps(ball))
    subprocess.run([cli, "phantom", str(tmp_path / "spec.json"), str(tmp_path / "ball.mhd")],
                   check=True, capture_output=True)
    r = subprocess.run([cli, "detect", "--method", "shift", "--volume", str(tmp_path / "ball.mhd"),
                        "--window", "0:64", "--seeds", "lattice:12", "--scales", "6,8", "--k", "5",
                        "--out", str(tmp_path / "dets.json")], capture_output=True, text=True)
    assert r.returncode == 0, r.stderr
    r = subprocess.run([cli, "eval", str(tmp_path / "dets.json"), str(tmp_path / "ball.gt.json"),
                        "--out", str(tmp_path / "metrics.json")], capture_output=True, text=True)
    assert r.returncode == 0, r.stderr
    m = json.loads((tmp_path / "metrics.json").read_text())
    assert m["recall"] == 1.0 and m["mean_jaccard_matched"] > 0.0
    small = {"dims": [32, 32, 32], "regions": [{"shape": "ball", "center": [16, 16, 16],
                                                "radius": 6, "fill": {"type": "uniform",
                                                                      "levels": 64}}],
             "rng_seed": 1}
    (tmp_path / "spec2.json").write_text(json.dumps(small))
    subprocess.run([cli, "phantom", str(tmp_path / "spec2.json"), str(tmp_path / "small.mhd")],
                   check=True, capture_output=True)
    r = subprocess.run([cli, "eval", str(tmp_path / "dets.json"), str(tmp_path / "small.gt.json")],
                       capture_output=True, text=True)
    assert r.returncode == 1  # dims mismatch (tools/main.cpp:166-169)


@pytest.mark.gpu
def test_rasterize_window_matches_oracle(sx, oracle):
    rng = np.random.default_rng(9)
    for _ in range(25):
        shape = tuple(int(v) for v in rng.integers(1, 40, size=3))
        center = rng.uniform(-5, 45, size=3)
        A = rng.normal(size=(3, 3)) * rng.uniform(1, 6)
        H = A @ A.T + np.eye(3)
        got = sx.rasterize_window(shape, center, H)
        ref = oracle.rasterize_window(shape, center, H)
        assert np.array_equal(got, ref)
    a = sx.rasterize_window((30, 30, 30), [15, 15, 15], np.diag([25.0] * 3))
    b = sx.rasterize_window((30, 30, 30), [17, 15, 15], np.diag([25.0] * 3))
    inter = len(np.intersect1d(a, b))
    assert sx.jaccard(a, b) == inter / (len(a) + len(b) - inter)
    assert sx.jaccard(a, a) == 1.0
    with pytest.raises(ValueError):
        sx.jaccard([], [])


@pytest.mark.gpu
def test_cli_detect_hu_template(cpp_build, tmp_path, sx):  # tools/main.cpp:130-139
    cli = os.path.join(cpp_build, "salvox-b200")
    spec = {"dims": [64, 64, 24],
            "regions": [{"shape": "ball", "center": [20.0, 32.0, 12.0], "radius": 8.0,
                         "fill": {"type": "constant", "value": 40.0}},
                        {"shape": "box", "center": [46.0, 32.0, 12.0], "half_extents": [10.0, 4.0, 8.0],
                         "fill": {"type": "constant", "value": 40.0}}], "rng_seed": 2}
    (tmp_path / "spec.json").write_text(json.dumps(spec))
    subprocess.run([cli, "phantom", str(tmp_path / "spec.json"), str(tmp_path / "v.mhd")],
                   check=True, capture_output=True)
    y, x = np.mgrid[0:24, 0:24]
    disk = np.where((x - 11.5) ** 2 + (y - 11.5) ** 2 <= 64.0, 40.0, 0.0).astype(np.float32)
    sx.save_volume(disk[None], str(tmp_path / "t.mhd"))
    r = subprocess.run([cli, "detect", "--method", "shift", "--volume", str(tmp_path / "v.mhd"),
                        "--window", "0:64", "--seeds", "lattice:8", "--scales", "6,8", "--k", "4",
                        "--hu-template", str(tmp_path / "t.mhd"), "--out", str(tmp_path / "d.json")],
                       capture_output=True, text=True)
    assert r.returncode == 0, r.stderr
    rep = json.loads((tmp_path / "d.json").read_text())
    dets = rep["detections"]
    assert dets and all("hu_distance" in d for d in dets)
    best = int(rep["header"]["hu_best_index"])
    assert dets[best]["hu_distance"] == min(d["hu_distance"] for d in dets)
