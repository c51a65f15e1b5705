"""Pins the oracle (oracle/salvox_oracle.c) against the reference's own tests.

The reference cannot be built here (Eigen3 and vendor/ are absent), so the
restatement is checked against every known-answer test and fixture property the
reference's doctest suites hold for this path (paths relative to
/root/reference/proj/tests). CPU only.
"""
import math

import numpy as np
import pytest

from tests import phantoms


# ------------------------------------------------------------ test_volume.cpp:35-65
def test_bin_of_kats(oracle):
    assert oracle.bin_of(0, 256, 256, 0.0) == 0
    assert oracle.bin_of(0, 100, 10, 55.0) == 5
    assert oracle.bin_of(40, 80, 16, 1000.0) == 15
    assert oracle.bin_of(40, 80, 16, -1000.0) == 0


def test_bin_of_total_monotone_surjective(oracle):
    prev, hit = 0, set()
    for i in range(4001):
        b = oracle.bin_of(-3.0, 17.0, 23, -10.0 + i * 0.01)
        assert 0 <= b < 23 and b >= prev
        prev = b
        hit.add(b)
    assert hit == set(range(23))


# ------------------------------------------------------------ test_entropy.cpp:13-26
@pytest.mark.parametrize("mode", [0, 1])
def test_entropy_kats(oracle, mode):
    oracle.set_log_mode(mode)
    try:
        d = np.zeros(16)
        d[3] = 1.0
        assert oracle.entropy_bits(d) == 0.0
        assert oracle.entropy_bits(np.full(256, 1.0 / 256)) == pytest.approx(8.0, rel=1e-12)
        assert oracle.entropy_bits(np.array([0.5, 0.25, 0.25, 0.0])) == pytest.approx(1.5,
                                                                                     rel=1e-12)
    finally:
        oracle.set_log_mode(0)


def test_shared_log_vs_glibc(oracle):
    """sx_log (include/salvox/sx_log.h) is within a few ulp of glibc log."""
    rng = np.random.default_rng(0)
    xs = np.concatenate([rng.random(20000), rng.random(2000) * 1e-6, [1.0, 0.5, 2.0 ** -30,
                                                                      0.999999999, 1e-300]])
    worst = 0.0
    for x in xs:
        if x <= 0:
            continue
        a, b = oracle.log_portable(float(x)), math.log(float(x))
        if b != 0.0:
            worst = max(worst, abs(a - b) / abs(b))
        else:
            assert a == 0.0
    assert worst < 4e-16


# ------------------------------------------------------------ test_entropy.cpp:120-139
def test_importance_weight_floor(oracle):
    # weight_for_bin is exercised through shift_step: on a constant volume every
    # voxel has weight sqrt((1/M)/1) and the step lands on the plain centroid
    vol = np.full((32, 32, 32), 3.0, np.float32)  # test_seek.cpp:321-331
    out, _ = oracle.shift_step(vol, 0, 64, 64, [16.0, 16.0, 16.0], [6.0, 6.0, 6.0])
    assert np.linalg.norm(out - [16, 16, 16]) < 1e-9


# ------------------------------------------------------------ Eigen restatement
def test_eigen_inverse_diagonal_and_general(oracle):
    for a in [4.0, 36.0, 64.0, 144.0, 225.0]:
        inv = oracle.eigen_inverse3(np.diag([a, a, a]))
        assert np.allclose(inv, np.diag([1 / a] * 3), rtol=2e-16, atol=0)
    m = np.array([[4.0, 1.0, 0.5], [1.0, 3.0, 0.2], [0.5, 0.2, 2.0]])
    assert np.allclose(oracle.eigen_inverse3(m) @ m, np.eye(3), atol=1e-14)


# ------------------------------------------------------------ test_pipeline.cpp:15-53
def test_plan_seeds_lattice_counts(oracle):
    pos, sc = oracle.plan_seeds((64, 64, 64), "lattice", 16.0, scales=[8.0])
    assert len(pos) == 64
    assert np.all((pos >= 0) & (pos <= 63))
    assert len(oracle.plan_seeds((64, 64, 64), "lattice", 16.0, scales=[6.0, 10.0])[0]) == 128
    pos, _ = oracle.plan_seeds((32, 32, 32), "lattice", 100.0, scales=[4.0])
    assert len(pos) == 1 and pos[0, 0] == 16.0


def test_plan_seeds_random_deterministic(oracle):
    a, _ = oracle.plan_seeds((48, 48, 48), "random", count=37, scales=[5.0], rng_seed=9)
    b, _ = oracle.plan_seeds((48, 48, 48), "random", count=37, scales=[5.0], rng_seed=9)
    assert len(a) == 37 and np.array_equal(a, b) and np.all((a >= 0) & (a <= 47))


def _dets(xs, pdfs):
    d = np.zeros(len(xs), np.dtype([("center", "<f8", (3,)), ("H", "<f8", (9,)),
                                   ("entropy_bits", "<f8"), ("pdf_diff", "<f8"),
                                   ("bhattacharyya", "<f8"), ("iterations", "<i4"),
                                   ("flags", "<u4"), ("seed_index", "<i4"), ("pad_", "<i4")]))
    d["center"][:, 0] = xs
    d["pdf_diff"] = pdfs
    d["seed_index"] = np.arange(len(xs))
    return d


def test_dedupe_top_k(oracle):  # test_pipeline.cpp:55-83
    out = oracle.dedupe_top_k(_dets([10, 11], [1.0, 2.0]), 20, 5.0)
    assert len(out) == 1 and out[0]["pdf_diff"] == 2.0
    rng = np.random.default_rng(4)
    d = _dets(rng.uniform(0, 500, 400), rng.random(400))
    out = oracle.dedupe_top_k(d, 20, 5.0)
    assert len(out) <= 20
    assert np.all(np.diff(out["pdf_diff"]) <= 0)
    for i in range(len(out)):
        for j in range(i + 1, len(out)):
            assert np.linalg.norm(out[i]["center"] - out[j]["center"]) > 5.0
    assert len(oracle.dedupe_top_k(d[:0], 20, 5.0)) == 0


# ------------------------------------------------------------ test_pipeline.cpp:228-276
def test_exhaustive_square_at_scale(oracle):
    vol, _ = oracle.make_phantom(phantoms.square_2d(64, 31.0, 31.0, 8, 64, 77))
    s, b, _ = oracle.exhaustive(vol, 0, 64, 64, [4.0, 6.0, 8.0, 10.0])
    pos, sc, scale, _ = oracle.local_maxima(s, b)
    assert np.linalg.norm(pos[0] - [31, 31, 0]) <= 2.0
    assert abs(scale[0] - 8.0) <= 2.0


def test_exhaustive_constant_zero(oracle):
    vol = np.full((1, 48, 48), 2.0, np.float32)
    s, b, _ = oracle.exhaustive(vol, 0, 64, 64, [4.0, 6.0])
    assert (s == 0).all()
    assert len(oracle.local_maxima(s, b)[0]) == 0


def test_exhaustive_two_squares(oracle):
    vol, _ = oracle.make_phantom(phantoms.squares_2d(96, [(24.0, 24.0), (68.0, 66.0)], 8, 78))
    s, b, _ = oracle.exhaustive(vol, 0, 64, 64, [6.0, 8.0, 10.0], budget=10**9)
    pos, sc, scale, _ = oracle.local_maxima(s, b)
    d = _dets(pos[:, 0], sc)
    d["center"] = pos
    top2 = oracle.dedupe_top_k(d, 2, 10.0)
    assert len(top2) == 2
    assert any(np.linalg.norm(t["center"] - [24, 24, 0]) <= 3 for t in top2)
    assert any(np.linalg.norm(t["center"] - [68, 66, 0]) <= 3 for t in top2)


def test_exhaustive_budget_and_scale_guards(oracle):
    with pytest.raises(oracle.OracleError, match="budget exceeded"):
        oracle.exhaustive(np.zeros((34, 256, 256), np.float32), 0, 64, 64, [4.0, 6.0])
    with pytest.raises(oracle.OracleError, match="scales must be >= 2"):
        oracle.exhaustive(np.zeros((1, 8, 8), np.float32), 0, 64, 64, [1.5])


def test_exhaustive_literal_equals_exact(oracle):
    """The exact-integer form (S_b(r) / T(r)) reproduces the literal fp64 sums to 1e-12."""
    vol, _ = oracle.make_phantom(phantoms.ball_3d(20, (10.0, 9.0, 10.0), 5.0, 3, levels=16))
    a, ab, av = oracle.exhaustive(vol, 0, 16, 16, [2.0, 3.0, 4.0], budget=10**9, threads=8)
    c, cb, cv = oracle.exhaustive(vol, 0, 16, 16, [2.0, 3.0, 4.0], budget=10**9, mode="exact",
                                  threads=8)
    assert av == cv
    assert np.allclose(a, c, rtol=1e-6, atol=0)  # float32 maps of fp64 values
    assert (ab == cb).mean() > 0.999


# ------------------------------------------------------------ test_seek.cpp:59-212
def _brute_quadrant_entropy(v, px, py, qx, qy, k, bins):  # test_seek.cpp:35-55
    x0, x1 = sorted([px, px + qx * k])
    y0, y1 = sorted([py, py + qy * k])
    counts = np.zeros(bins)
    total = 0
    for y in range(v.shape[1]):
        for x in range(v.shape[2]):
            if x < math.ceil(x0) or x > math.floor(x1) or y < math.ceil(y0) or y > math.floor(y1):
                continue
            counts[min(max(int(math.floor(v[0, y, x] / 64.0 * 64)), 0), 63)] += 1
            total += 1
    if total < 4:
        return 0.0
    p = counts[counts > 0] / total
    return float(-(p * np.log2(p)).sum())


def test_quadrant_step_matches_bruteforce(oracle):
    vol, _ = oracle.make_phantom(phantoms.square_2d(96, 47.0, 47.0, 12, 64, 41))
    moved, st = oracle.ascent_step(vol, 0, 64, 64, [40.0, 44.0], [4, 8, 12])
    dirs = [(1, 1), (-1, 1), (-1, -1), (1, -1)]
    ee, kk = [], []
    for qx, qy in dirs:
        be, bk = 0.0, 4
        for k in (4, 8, 12):
            e = _brute_quadrant_entropy(vol, 40.0, 44.0, qx, qy, k, 64)
            if e > be:
                be, bk = e, k
        ee.append(be)
        kk.append(bk)
    tot = sum(ee)
    ed = np.zeros(2)
    for q, (qx, qy) in enumerate(dirs):
        assert st["entropy"][q] == pytest.approx(ee[q], rel=1e-12)
        assert st["best_scale"][q] == kk[q]
        ed += np.array([qx, qy]) * ee[q] / tot * kk[q]
    assert np.linalg.norm(st["displacement"][:2] - ed) < 1e-12
    assert np.linalg.norm(moved[:2] - (np.array([40.0, 44.0]) + ed)) < 1e-12
    assert st["displacement"][0] > 0.0


def test_quadrant_norm_entropy_sums_to_one(oracle):
    vol, _ = oracle.make_phantom(phantoms.square_2d(64, 31.0, 31.0, 10, 64, 17))
    rng = np.random.default_rng(3)
    for _ in range(20):
        p = rng.uniform(8, 55, 2)
        _, st = oracle.ascent_step(vol, 0, 64, 64, p, [4, 6, 10])
        if st["degenerate"]:
            continue
        assert st["norm_entropy"].sum() == pytest.approx(1.0, rel=1e-9)
        assert np.linalg.norm(st["displacement"]) <= math.sqrt(2) * 10 + 1e-12


def test_quadrant_balanced_and_degenerate(oracle):
    v, c = phantoms.symmetric_square_2d()
    _, st = oracle.ascent_step(v, 0, 64, 64, [c, c], [4, 8, 12])
    assert not st["degenerate"] and np.linalg.norm(st["displacement"]) < 0.5
    flat = np.full((1, 64, 64), 7.0, np.float32)
    moved, st = oracle.ascent_step(flat, 0, 64, 64, [32.0, 32.0], [4, 8])
    assert st["degenerate"] and tuple(moved[:2]) == (32.0, 32.0)


def test_quadrant_seek_grid_finds_square(oracle):
    vol, _ = oracle.make_phantom(phantoms.square_2d(128, 63.0, 63.0, 12, 64, 23))
    hit = False
    for y in range(8, 128, 16):
        for x in range(8, 128, 16):
            r = oracle.ascent_seek_one(vol, 0, 64, 64, [float(x), float(y)], [4, 8, 12, 16])
            if not r["degenerate"] and np.linalg.norm(r["position"][:2] - [63, 63]) <= 3.0:
                hit = True
    assert hit


def test_quadrant_mirror_symmetry(oracle):
    vol, _ = oracle.make_phantom(phantoms.square_2d(96, 40.0, 47.0, 10, 64, 57))
    m = np.ascontiguousarray(vol[:, :, ::-1])
    a = oracle.ascent_seek_one(vol, 0, 64, 64, [32.0, 44.0], [4, 6, 10], max_iters=8)
    b = oracle.ascent_seek_one(m, 0, 64, 64, [95.0 - 32.0, 44.0], [4, 6, 10], max_iters=8)
    assert not a["degenerate"] and not b["degenerate"]
    assert a["position"][0] == pytest.approx(95.0 - b["position"][0], rel=1e-9)
    assert a["position"][1] == pytest.approx(b["position"][1], rel=1e-9)


def test_quadrant_requires_2d(oracle):
    with pytest.raises(oracle.OracleError):
        oracle.ascent_step(np.zeros((4, 8, 8), np.float32), 0, 64, 64, [4.0, 4.0, 1.0], [2])


# ------------------------------------------------------------ NEW: octant (3D quadrant)
def test_octant_balanced_at_symmetric_centre(oracle):
    v, c = phantoms.symmetric_cube_octant()
    _, st = oracle.ascent_step(v, 0, 64, 64, [c, c, c], [3, 6, 9], dims=3)
    assert not st["degenerate"]
    assert np.linalg.norm(st["displacement"]) < 0.5
    assert st["norm_entropy"].sum() == pytest.approx(1.0, rel=1e-12)


def test_octant_constant_degenerate_and_ascends(oracle):
    flat = np.full((24, 24, 24), 5.0, np.float32)
    moved, st = oracle.ascent_step(flat, 0, 64, 64, [12.0, 12.0, 12.0], [3, 6], dims=3)
    assert st["degenerate"] and tuple(moved) == (12.0, 12.0, 12.0)
    vol, _ = oracle.make_phantom(phantoms.cube_3d(48, 7, 71))
    r = oracle.ascent_seek_one(vol, 0, 64, 64, [30.0, 28.0, 20.0], [3, 6, 9], dims=3)
    assert not r["degenerate"]
    assert np.linalg.norm(r["position"] - [23.5, 23.5, 23.5]) <= 4.0


# ------------------------------------------------------------ test_seek.cpp:270-421
def _brute_shift_step(v, x, radius, bins):  # test_seek.cpp:235-266 (Eigen-free oracle)
    z, y, xx = np.meshgrid(np.arange(v.shape[0]), np.arange(v.shape[1]), np.arange(v.shape[2]),
                           indexing="ij")
    d = ((xx - x[0]) ** 2 + (y - x[1]) ** 2 + (z - x[2]) ** 2) / (radius * radius)
    m = d <= 1.0
    b = np.clip(np.floor(v[m].astype(np.float64) / 64.0 * bins).astype(int), 0, bins - 1)
    p = np.bincount(b, weights=d[m], minlength=bins)
    p /= p.sum()
    w = np.sqrt((1.0 / bins) / np.maximum(p[b], 1e-6))
    pts = np.stack([xx[m], y[m], z[m]], 1)
    return (w[:, None] * pts).sum(0) / w.sum()


def test_shift_step_matches_bruteforce(oracle):
    vol, _ = oracle.make_phantom(phantoms.ball_3d(48, (28.0, 24.0, 24.0), 9.0, 61))
    x = [16.0, 20.0, 22.0]
    got, _ = oracle.shift_step(vol, 0, 64, 64, x, [7.0, 7.0, 7.0])
    assert np.linalg.norm(got - _brute_shift_step(vol, x, 7.0, 64)) < 1e-9
    ball = np.array([28.0, 24.0, 24.0])
    assert np.linalg.norm(got - ball) < np.linalg.norm(np.array(x) - ball)


def test_shift_fixed_point_and_constant(oracle):
    v, c = phantoms.symmetric_cube_3d()
    got, _ = oracle.shift_step(v, 0, 64, 64, [c, c, c], [8.0, 8.0, 8.0])
    assert np.linalg.norm(got - c) < 0.5


def test_saliency_shift_converges_and_reseeds(oracle):
    vol, cent = oracle.make_phantom(phantoms.cube_3d(64, 8, 71))
    c = cent[0]
    d, _ = oracle.saliency_shift(vol, 0, 64, 64, c + [6.0, 0.0, 0.0], [8.0, 8.0, 8.0])
    assert not d["flags"] & 2 and d["iterations"] <= 20
    assert np.linalg.norm(d["center"] - c) <= 2.0
    again, _ = oracle.saliency_shift(vol, 0, 64, 64, d["center"], [8.0, 8.0, 8.0])
    assert again["flags"] & 1 and again["iterations"] == 1
    assert np.linalg.norm(again["center"] - d["center"]) < 0.1


def test_saliency_shift_bandwidth_fixed_in_bounds(oracle):
    vol, _ = oracle.make_phantom(phantoms.cube_3d(48, 7, 83))
    H0 = np.diag([36.0, 25.0, 16.0]).ravel()
    rng = np.random.default_rng(13)
    for _ in range(10):
        d, _ = oracle.saliency_shift(vol, 0, 64, 64, rng.uniform(0, 47, 3), [6.0, 5.0, 4.0])
        assert np.array_equal(d["H"], H0)
        assert np.all((d["center"] >= 0) & (d["center"] <= 47))


def test_shift_self_target_lands_on_centroid(oracle):  # test_seek.cpp:400-421
    vol, cent = oracle.make_phantom(phantoms.cube_3d(48, 10, 91))
    x = cent[0] + [4.0, 2.0, 0.0]
    H = np.diag([36.0, 36.0, 36.0])
    target = oracle.candidate_histogram(vol, 0, 64, 64, x, H)
    got, _ = oracle.shift_step(vol, 0, 64, 64, x, [6.0, 6.0, 6.0], target=target)
    z, y, xx = np.meshgrid(np.arange(48), np.arange(48), np.arange(48), indexing="ij")
    lo = np.ceil(x - 6.0)
    hi = np.floor(x + 6.0)
    m = ((xx - x[0]) ** 2 / 36 + (y - x[1]) ** 2 / 36 + (z - x[2]) ** 2 / 36 <= 1.0)
    m &= (xx >= lo[0]) & (xx <= hi[0]) & (y >= lo[1]) & (y <= hi[1]) & (z >= lo[2]) & (z <= hi[2])
    cen = np.array([xx[m].mean(), y[m].mean(), z[m].mean()])
    assert np.linalg.norm(got - cen) < 1e-9


def test_candidate_histogram_and_pdf_properties(oracle):  # test_entropy.cpp:159-254
    flat = np.full((16, 16, 16), 5.0, np.float32)
    for k in ("identity", "epanechnikov", "gaussian"):
        p = oracle.candidate_histogram(flat, 0, 64, 64, [8, 8, 8], np.diag([25.0] * 3), k)
        assert oracle.entropy_bits(p) == 0.0 and p[5] == pytest.approx(1.0)
    assert oracle.candidate_histogram(np.zeros((8, 8, 8), np.float32), 0, 8, 8, [4, 4, 4],
                                      np.diag([0.25] * 3)) is None
    assert oracle.pdf_difference(np.full((32, 32, 32), 9.0, np.float32), 0, 64, 64,
                                 [16, 16, 16], np.diag([36.0] * 3), "epanechnikov") == 0.0
    with pytest.raises(oracle.OracleError):
        oracle.pdf_difference(np.zeros((16, 16, 16), np.float32), 0, 8, 8, [8, 8, 8],
                              np.diag([2.25] * 3), "epanechnikov")


# ------------------------------------------------------------ test_pipeline.cpp:296-400
def test_detect_shift_finds_ball(oracle):
    vol, cent = oracle.make_phantom(phantoms.ball_3d(64, (36.0, 30.0, 28.0), 9.0, 101))
    sel, _, _ = oracle.detect(vol, 0, 64, 64, method="shift", seed_spacing=16.0,
                              scales=[6.0, 9.0], top_k=5, dedupe_radius=6.0, workers=8)
    assert len(sel) and np.linalg.norm(sel[0]["center"] - cent[0]) <= 2.0


def test_detect_2d_methods_land_on_exhaustive_top1(oracle):
    vol, _ = oracle.make_phantom(phantoms.square_2d(96, 45.0, 49.0, 9, 64, 303))
    s, b, _ = oracle.exhaustive(vol, 0, 64, 64, [6.0, 9.0, 12.0], budget=10**9)
    best = oracle.local_maxima(s, b)[0][0]
    for m in ("quadrant", "shift"):
        sel, _, _ = oracle.detect(vol, 0, 64, 64, method=m, seed_spacing=12.0,
                                  scales=[6.0, 10.0], top_k=3, dedupe_radius=8.0)
        assert len(sel) and any(np.linalg.norm(d["center"] - best) <= 3.0 for d in sel)


def test_detect_constant_empty_and_worker_independence(oracle):
    flat = np.ones((48, 48, 48), np.float32)
    sel, _, _ = oracle.detect(flat, 0, 64, 64, method="shift", seed_spacing=16.0, scales=[6.0])
    assert len(sel) == 0
    with pytest.raises(oracle.OracleError, match="requires a 2D volume"):
        oracle.detect(np.zeros((16, 16, 16), np.float32), 0, 64, 64, method="quadrant")
    spec = phantoms.ball_3d(48, (24.0, 24.0, 24.0), 8.0, 404,
                            background={"type": "gaussian", "mean": 8.0, "sigma": 2.0})
    vol, _ = oracle.make_phantom(spec)
    a, _, _ = oracle.detect(vol, 0, 64, 64, method="shift", seed_spacing=12.0,
                            scales=[5.0, 8.0], top_k=10, workers=1)
    b, _, _ = oracle.detect(vol, 0, 64, 64, method="shift", seed_spacing=12.0,
                            scales=[5.0, 8.0], top_k=10, workers=4)
    assert a.tobytes() == b.tobytes()
