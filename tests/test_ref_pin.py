"""Pins the C oracle AND the product's host code against the REFERENCE ITSELF.

oracle/_ref/libsalvox_ref.so is the reference's own sources
(/root/reference/proj/src/*.cpp, compiled where they lie by `make -C oracle
ref`; Eigen3 is absent, so they build against the repo's Eigen-API subset --
DESIGN.md §4). Every case below runs the same seeded inputs through the
reference and through the restatement (and, where the product has host code,
through the product) and requires BYTE-identical outputs: exhaustive maps,
maxima and visits; shift / quadrant / ABMSOD trajectories, traces, scores and
selections; seeds; phantoms; MetaImage IO; dedupe; rasterisation; Hu moments;
exception messages. CPU only (the GPU side is tests/test_gpu_reference.py).
"""
import math
import os

import numpy as np
import pytest

from tests import phantoms

R = pytest.importorskip("oracle.ref")
pytestmark = pytest.mark.skipif(not R.available(), reason="oracle/_ref not built (no /root/reference)")


def _same(a, b):
    return np.asarray(a).tobytes() == np.asarray(b).tobytes()


# ------------------------------------------------------------------ phantoms
@pytest.mark.parametrize("spec", [
    phantoms.square_2d(64, 31.0, 31.0, 8, 64, 77),
    phantoms.squares_2d(96, [(30.0, 30.0), (66.0, 62.0)], 7, 78),
    phantoms.ball_3d(24, (12.0, 11.0, 13.0), 5.0, 6736, levels=32,
                     background={"type": "gaussian", "mean": 8.0, "sigma": 2.0}),
    phantoms.config_c1(),
    phantoms.config_c3(),
])
def test_phantom_bit_identical(oracle, sx, spec):
    vr, cr = R.make_phantom(spec)
    vo, co = oracle.make_phantom(spec)
    assert _same(vr, vo) and np.array_equal(cr, co)
    vp, gt = sx.make_phantom(spec)  # the product's host make_phantom
    assert _same(vr, vp)


def test_phantom_oblique_ellipsoid(oracle):
    th = math.radians(30.0)
    rz = np.array([[math.cos(th), -math.sin(th), 0], [math.sin(th), math.cos(th), 0], [0, 0, 1]])
    spec = phantoms.ellipsoid_3d(rz @ np.diag([10.0, 7.0, 5.0]), 222, 64)
    assert _same(R.make_phantom(spec)[0], oracle.make_phantom(spec)[0])


# ------------------------------------------------------------- exhaustive KB
EXH = [
    # test_pipeline.cpp:228-236 (square), :247-270 (two squares), :238-245 (constant)
    (phantoms.square_2d(64, 31.0, 31.0, 8, 64, 77), 0.0, 64.0, 64, [4.0, 6.0, 8.0, 10.0]),
    (phantoms.squares_2d(96, [(30.0, 30.0), (66.0, 62.0)], 7, 78), 0.0, 64.0, 64, [6.0, 8.0, 10.0]),
    ({"dims": [48, 48, 1], "background": {"type": "constant", "value": 5.0}, "regions": []},
     0.0, 64.0, 64, [4.0, 6.0]),
    # C2-style 3D (gaussian background, 32 bins)
    (phantoms.ball_3d(24, (12.0, 11.0, 13.0), 5.0, 6736, levels=32,
                      background={"type": "gaussian", "mean": 8.0, "sigma": 2.0}),
     0.0, 32.0, 32, [3.0, 4.0, 5.0, 6.0, 7.0]),
    # non-integer and unsorted scales, ragged dims
    (phantoms.ball_3d(20, (9.0, 10.0, 8.0), 4.0, 5), 0.0, 64.0, 64, [4.5, 3.0, 2.5]),
]


@pytest.mark.parametrize("case", range(len(EXH)))
@pytest.mark.parametrize("kernel", ["identity", "epanechnikov", "gaussian"])
def test_exhaustive_literal_bit_identical(oracle, case, kernel):
    spec, lo, hi, bins, scales = EXH[case]
    if kernel != "identity" and case in (1, 3):
        pytest.skip("kernel variants on the small cases only")
    vol, _ = oracle.make_phantom(spec)
    rs, rb, rm, rv = R.exhaustive(vol, lo, hi, bins, scales, kernel=kernel, budget=10**12)
    os_, ob, ov = oracle.exhaustive(vol, lo, hi, bins, scales, kernel=kernel, budget=10**12,
                                    mode="literal", threads=4)
    assert _same(rs, os_) and _same(rb, ob) and rv == ov
    pos, sc, scale, _ = oracle.local_maxima(os_, ob)
    assert len(rm) == len(pos)
    assert np.array_equal(rm[:, :3], pos) and np.array_equal(rm[:, 3], sc)
    assert np.array_equal(rm[:, 4], scale)


def test_exhaustive_exact_mode_within_float_rounding(oracle):
    spec, lo, hi, bins, scales = EXH[3]
    vol, _ = oracle.make_phantom(spec)
    rs, _, _, _ = R.exhaustive(vol, lo, hi, bins, scales, budget=10**12)
    es, _, _ = oracle.exhaustive(vol, lo, hi, bins, scales, budget=10**12, mode="exact", threads=4)
    assert np.all(np.abs(rs - es) <= 1e-5 * np.maximum(np.abs(rs), np.abs(es)) + 1e-6)


@pytest.mark.parametrize("scales,budget", [([1.5], 10**9), ([], 10**9), ([4.0], 100)])
def test_exhaustive_errors_same_message(oracle, scales, budget):
    vol = np.zeros((1, 32, 32), np.float32)
    with pytest.raises(ValueError) as er:
        R.exhaustive(vol, 0.0, 1.0, 8, scales, budget=budget)
    with pytest.raises(ValueError) as eo:
        oracle.exhaustive(vol, 0.0, 1.0, 8, scales, budget=budget)
    assert str(er.value) == str(eo.value)


# ------------------------------------------------------------------- seeds
@pytest.mark.parametrize("args", [
    ((64, 64, 64), "lattice", 16.0, 0, [8.0], 0),
    ((1, 96, 96), "lattice", 12.0, 0, [6.0, 10.0], 0),
    ((160, 256, 256), "lattice", 16.0, 0, [8.0, 12.0], 0),
    ((128, 128, 128), "lattice", 8.0, 0, [float(s) for s in range(3, 16)], 0),
    ((20, 10, 5), "lattice", 64.0, 0, [3.0], 0),
    ((48, 48, 48), "random", 16.0, 37, [5.0], 9),
    ((1, 64, 64), "random", 16.0, 11, [4.0, 6.0], 3),
])
def test_plan_seeds_bit_identical(oracle, sx, args):
    shape, mode, spacing, count, scales, seed = args
    a, sa = R.plan_seeds(shape, mode, spacing, count, scales, seed)
    b, sb = oracle.plan_seeds(shape, mode, spacing, count, scales, seed)[:2]
    c, sc = sx.plan_seeds(shape, mode, spacing, count, scales, seed)
    assert _same(a, b) and _same(sa, sb) and _same(a, c) and _same(sa, sc)


# --------------------------------------------------------- shift mean shift
@pytest.fixture(scope="module")
def ball32(oracle):
    return oracle.make_phantom(phantoms.ball_3d(32, (16.0, 15.0, 14.0), 6.0, 7))[0]


@pytest.mark.parametrize("kernels", [("identity", "identity"), ("epanechnikov", "epanechnikov"),
                                     ("gaussian", "identity")])
def test_saliency_shift_per_seed_bit_identical(oracle, ball32, kernels):
    step_k, hist_k = kernels
    pos, ss = R.plan_seeds(ball32.shape, spacing=8.0, scales=[4.0, 6.0])
    for p, s in zip(pos, ss):
        dr, vr = R.saliency_shift(ball32, 0, 64, 64, p, [s, s, s], step_kernel=step_k,
                                  hist_kernel=hist_k)
        do, vo = oracle.saliency_shift(ball32, 0, 64, 64, p, [s, s, s], step_kernel=step_k,
                                       hist_kernel=hist_k)
        assert dr.tobytes() == do.tobytes() and vr == vo


def test_shift_step_and_windows_bit_identical(oracle, ball32):
    rng = np.random.default_rng(3)
    for _ in range(12):
        x = rng.uniform(-2, 34, size=3)
        half = rng.uniform(2.0, 9.0, size=3)
        a = R.shift_step(ball32, 0, 64, 64, x, half)
        b = oracle.shift_step(ball32, 0, 64, 64, x, half)
        assert (a[0] is None) == (b[0] is None) and a[1] == b[1]
        if a[0] is not None:
            assert _same(a[0], b[0])
        H = np.diag(half * half)
        pr, vr = R.candidate_histogram(ball32, 0, 64, 64, x, H, kernel="epanechnikov")
        po = oracle.candidate_histogram(ball32, 0, 64, 64, x, H, kernel="epanechnikov")
        assert (pr is None) == (po is None)
        if pr is not None:
            assert _same(pr, po)


@pytest.mark.parametrize("method,kw", [
    ("shift", dict(seed_spacing=8.0, scales=[4.0, 6.0], top_k=8, dedupe_radius=4.0)),
    ("shift", dict(seed_mode="random", seed_count=40, rng_seed=5, scales=[5.0], top_k=6,
                   dedupe_radius=3.0, entropy_quantile=0.5, pdf_quantile=0.25)),
    ("abmsod", dict(seed_spacing=10.0, scales=[5.0], top_k=8, dedupe_radius=4.0,
                    entropy_quantile=0.0)),
])
def test_detect_3d_bit_identical(oracle, ball32, method, kw):
    so, _, vo = oracle.detect(ball32, 0, 64, 64, method=method, **kw)
    sr, vr = R.detect(ball32, 0, 64, 64, method=method, **kw)
    assert len(sr) > 0
    assert sr.tobytes() == so.tobytes() and vr == vo


def test_detect_workers_independent(ball32):  # test_pipeline.cpp:402-436
    kw = dict(seed_spacing=8.0, scales=[4.0, 6.0], top_k=8, dedupe_radius=4.0)
    a, va = R.detect(ball32, 0, 64, 64, method="shift", workers=1, **kw)
    b, vb = R.detect(ball32, 0, 64, 64, method="shift", workers=4, **kw)
    assert a.tobytes() == b.tobytes() and va == vb


# --------------------------------------------------------- quadrant (2D)
@pytest.fixture(scope="module")
def square64(oracle):
    return oracle.make_phantom(phantoms.square_2d(64, 31.0, 31.0, 8, 64, 77))[0]


def test_quadrant_step_and_seek_bit_identical(oracle, square64):
    scales = [4, 6, 8, 10]
    for p in ([20.0, 22.0], [31.0, 31.0], [44.5, 17.25], [1.0, 62.0]):
        mr, sr, _ = R.quadrant_step(square64, 0, 64, 64, p, scales)
        mo, so = oracle.ascent_step(square64, 0, 64, 64, [p[0], p[1]], scales, dims=2)
        assert _same(mr, np.asarray(mo)[:2])
        assert _same(np.array(sr.entropy[:4]), so["entropy"])
        assert _same(np.array(sr.best_scale[:4]), so["best_scale"])
        assert _same(np.array(sr.norm_entropy[:4]), so["norm_entropy"])
        assert bool(sr.degenerate) == so["degenerate"]
        rr, _ = R.quadrant_seek_one(square64, 0, 64, 64, p, scales)
        ro = oracle.ascent_seek_one(square64, 0, 64, 64, [p[0], p[1]], scales, dims=2)
        assert _same(np.array(rr.position[:2]), ro["position"][:2])
        assert (rr.iterations, rr.best_scale, rr.entropy_bits, bool(rr.converged),
                bool(rr.degenerate)) == (ro["iterations"], ro["best_scale"], ro["entropy_bits"],
                                         ro["converged"], ro["degenerate"])


def test_detect_quadrant_bit_identical(oracle, square64):
    kw = dict(seed_spacing=16.0, scales=[4.0, 6.0, 8.0, 10.0], top_k=5, dedupe_radius=5.0)
    so, _, vo = oracle.detect(square64, 0, 64, 64, method="quadrant", **kw)
    sr, vr = R.detect(square64, 0, 64, 64, method="quadrant", **kw)
    assert len(sr) > 0 and sr.tobytes() == so.tobytes() and vr == vo


def test_quadrant_on_3d_same_error(oracle, ball32):
    with pytest.raises(ValueError) as er:
        R.detect(ball32, 0, 64, 64, method="quadrant")
    with pytest.raises(ValueError) as eo:
        oracle.detect(ball32, 0, 64, 64, method="quadrant")
    assert str(er.value) == str(eo.value)


# ------------------------------------------------------------------ ABMSOD
def _oblique(oracle, seed=222, dim=64):
    th = math.radians(30.0)
    rz = np.array([[math.cos(th), -math.sin(th), 0], [math.sin(th), math.cos(th), 0], [0, 0, 1]])
    return oracle.make_phantom(phantoms.ellipsoid_3d(rz @ np.diag([10.0, 7.0, 5.0]), seed, dim))[0]


@pytest.mark.parametrize("offset", [(0.0, 0.0, 0.0), (3.0, -2.0, 1.0), (-6.0, 4.0, -3.0)])
def test_abmsod_trace_bit_identical(oracle, offset):
    vol = _oblique(oracle)
    c = (64 - 1) / 2.0
    seed = [c + offset[0], c + offset[1], c + offset[2]]
    dr, tr, vr = R.abmsod_run(vol, 0, 64, 64, seed, radius=6.0, trace=True)
    do, to, vo = oracle.abmsod_run(vol, 0, 64, 64, seed, radius=6.0, trace=True)
    assert dr.tobytes() == do.tobytes() and tr.tobytes() == to.tobytes() and vr == vo


def test_bandwidth_from_moment_bit_identical(oracle):
    rng = np.random.default_rng(11)
    for _ in range(50):
        A = rng.normal(size=(3, 3))
        outer = A @ A.T * rng.uniform(1, 500)
        w = rng.uniform(0.5, 50)
        a = R.bandwidth_from_moment(outer, w, 3, 4.0, 900.0)
        b = oracle.bandwidth_from_moment(outer, w, 3, 4.0, 900.0)
        assert _same(a, b)
    for bad in ((np.eye(3), 0.0), (np.full((3, 3), np.nan), 1.0)):
        with pytest.raises(ValueError) as er:
            R.bandwidth_from_moment(bad[0], bad[1], 3, 4.0, 900.0)
        with pytest.raises(ValueError) as eo:
            oracle.bandwidth_from_moment(bad[0], bad[1], 3, 4.0, 900.0)
        assert str(er.value) == str(eo.value)


# ---------------------------------------------------------- selection etc.
def test_dedupe_top_k_bit_identical(oracle):
    rng = np.random.default_rng(4)
    from oracle.oracle import DET_DTYPE
    d = np.zeros(200, DET_DTYPE)
    d["center"] = rng.integers(0, 30, size=(200, 3)).astype(np.float64)
    d["pdf_diff"] = rng.integers(0, 20, size=200) / 4.0  # ties exercise the stable order
    d["seed_index"] = np.arange(200)
    for k, r in ((20, 5.0), (7, 2.0), (300, 0.0)):
        assert R.dedupe_top_k(d, k, r).tobytes() == oracle.dedupe_top_k(d, k, r).tobytes()


def test_rasterize_and_hu_bit_identical(oracle):
    rng = np.random.default_rng(9)
    for _ in range(20):
        shape = tuple(int(v) for v in rng.integers(1, 30, size=3))
        center = rng.uniform(-5, 35, size=3)
        A = rng.normal(size=(3, 3)) * rng.uniform(1, 6)
        H = A @ A.T + np.eye(3)
        assert _same(R.rasterize_window(shape, center, H),
                     oracle.rasterize_window(shape, center, H))
    for _ in range(10):
        img = (rng.random((int(rng.integers(3, 40)), int(rng.integers(3, 40)))) * 50).astype(
            np.float32)
        assert _same(R.hu_moments(img), oracle.hu_moments(img))
    vol = _oblique(oracle, dim=48)
    y, x = np.mgrid[0:20, 0:20]
    tmpl = np.where((x - 9.5) ** 2 + (y - 9.5) ** 2 <= 49.0, 40.0, 0.0).astype(np.float32)
    for c in ([23.5, 23.5, 23.5], [10.0, 30.0, 5.0]):
        H = np.diag([36.0, 25.0, 16.0])
        assert R.hu_template_distance(vol, c, H, tmpl) == oracle.hu_template_distance(vol, c, H,
                                                                                        tmpl)


# ------------------------------------------------------------ MetaImage IO
def test_meta_io_both_directions(sx, tmp_path):
    rng = np.random.default_rng(17)
    v = rng.uniform(-100.0, 100.0, size=(5, 7, 9)).astype(np.float32)
    R.save_volume(v, str(tmp_path / "r.mhd"))            # reference writes, product reads
    got, sp = sx.load_volume(str(tmp_path / "r.mhd"))
    assert _same(got, v) and tuple(sp) == (1.0, 1.0, 1.0)
    sx.save_volume(v, str(tmp_path / "p.mhd"), spacing=(0.5, 0.75, 2.0))  # and back
    back, sp2 = R.load_volume(str(tmp_path / "p.mhd"))
    assert _same(back, v) and tuple(sp2) == (0.5, 0.75, 2.0)
    for etype, dt in (("MET_UCHAR", np.uint8), ("MET_SHORT", np.int16),
                      ("MET_USHORT", np.uint16)):
        info = np.iinfo(dt)
        data = rng.integers(info.min, info.max, size=(3, 5, 7), endpoint=True).astype(dt)
        (tmp_path / f"{etype}.raw").write_bytes(data.tobytes())
        (tmp_path / f"{etype}.mhd").write_text(
            f"NDims = 3\nDimSize = 7 5 3\nElementType = {etype}\nElementSpacing = 1 2 3\n"
            f"ElementDataFile = {etype}.raw\n")
        a, spa = R.load_volume(str(tmp_path / f"{etype}.mhd"))
        b, spb = sx.load_volume(str(tmp_path / f"{etype}.mhd"))
        assert _same(a, b) and tuple(spa) == tuple(spb)
    (tmp_path / "bad.raw").write_bytes(bytes(999))
    (tmp_path / "bad.mhd").write_text("NDims = 3\nDimSize = 10 10 10\nElementType = MET_UCHAR\n"
                                      "ElementDataFile = bad.raw\n")
    with pytest.raises(Exception) as er:
        R.load_volume(str(tmp_path / "bad.mhd"))
    with pytest.raises(RuntimeError) as ep:
        sx.load_volume(str(tmp_path / "bad.mhd"))
    assert "size mismatch" in str(er.value) and "size mismatch" in str(ep.value)


def test_fnv_checksum_matches(sx):
    data = os.urandom(1000)
    h = 0xcbf29ce484222325
    for x in data:
        h = ((h ^ x) * 0x100000001b3) & 0xFFFFFFFFFFFFFFFF
    assert R.fnv1a64(data) == h
