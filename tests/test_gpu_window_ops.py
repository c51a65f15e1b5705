"""The seek path's building blocks as device calls (salvox_window_ops /
salvox_ascent_step) against the reference's own functions (oracle/_ref, the
reference's sources compiled here) on the same inputs:

  candidate_histogram / try_candidate_histogram  window.cpp:5-27
  pdf_difference                                 window.cpp:30-51
  shift_step                                     shift.cpp:15-34
  box_entropy_bits                               quadrant.cpp:18-35
  quadrant_step                                  quadrant.cpp:37-81

Histograms, pdf differences and shift steps are BIT-identical for the
identity and Epanechnikov kernels (same fp64 operations in the same order; the
window geometry is built on the host with glibc pow/sqrt like the reference);
the Gaussian kernel (libdevice-free shared sx_exp vs glibc exp) and the
entropies (sx_log vs glibc log) agree within 1e-12.
"""
import math

import numpy as np
import pytest

from tests import phantoms

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def R():
    from oracle import ref

    if not ref.available():
        pytest.skip("oracle/_ref/libsalvox_ref.so not built")
    return ref


@pytest.fixture(scope="module")
def vol3(oracle):
    return oracle.make_phantom(phantoms.ball_3d(32, (16.0, 15.0, 14.0), 6.0, 7))[0]


def _windows(rng, n, lo=-3.0, hi=35.0):
    out = []
    for i in range(n):
        c = rng.uniform(lo, hi, size=3)
        if i % 2:
            A = rng.normal(size=(3, 3)) * rng.uniform(1.0, 3.0)
            H = A @ A.T + np.eye(3) * rng.uniform(2.0, 10.0)
        else:
            H = np.diag(rng.uniform(2.0, 9.0, size=3) ** 2)
        out.append((c, H))
    return out


@pytest.mark.parametrize("kernel", ["identity", "epanechnikov", "gaussian"])
def test_candidate_histogram_matches_reference(sx, R, vol3, kernel):
    from paper_1310_6736_b200._lib import WINDOW_OP_DTYPE, WOP_HIST

    rng = np.random.default_rng(1)
    wins = _windows(rng, 40)
    ops = np.zeros(len(wins), WINDOW_OP_DTYPE)
    for i, (c, H) in enumerate(wins):
        ops[i]["op"] = WOP_HIST
        ops[i]["kernel"] = {"identity": 0, "epanechnikov": 1, "gaussian": 2}[kernel]
        ops[i]["center"] = c
        ops[i]["H"] = H.reshape(9)
    res, pmf = sx.window_ops(vol3, ops, 0.0, 64.0, 64, want_pmf=True)  # one launch
    for i, (c, H) in enumerate(wins):
        p, visits = R.candidate_histogram(vol3, 0.0, 64.0, 64, c, H, kernel=kernel)
        assert bool(res[i]["ok"]) == (p is not None)
        assert int(res[i]["visits"]) == visits
        if p is None:
            continue
        if kernel == "gaussian":
            np.testing.assert_allclose(pmf[i], p, rtol=1e-12, atol=1e-15)
        else:
            assert pmf[i].tobytes() == p.tobytes()


def test_candidate_histogram_api_and_error(sx, R, vol3):
    H = np.diag([25.0, 16.0, 9.0])
    p = sx.candidate_histogram(vol3, [16.0, 15.0, 14.0], H, 0.0, 64.0, 64)  # epanechnikov
    ref, _ = R.candidate_histogram(vol3, 0.0, 64.0, 64, [16.0, 15.0, 14.0], H,
                                   kernel="epanechnikov")
    assert p.tobytes() == ref.tobytes()
    with pytest.raises(ValueError, match="no usable in-bounds voxel"):
        sx.candidate_histogram(vol3, [-40.0, -40.0, -40.0], H, 0.0, 64.0, 64)


@pytest.mark.parametrize("kernel", ["identity", "epanechnikov"])
def test_pdf_difference_matches_reference(sx, R, vol3, kernel):
    rng = np.random.default_rng(2)
    for _ in range(12):
        c = rng.uniform(0.0, 31.0, size=3)
        s = float(rng.uniform(2.0, 10.0))
        H = np.diag([s * s] * 3)
        try:
            want, _ = R.pdf_difference(vol3, 0.0, 64.0, 64, c, H, kernel=kernel)
        except ValueError:
            with pytest.raises(ValueError):
                sx.pdf_difference(vol3, c, s, 0.0, 64.0, 64, kernel=kernel)
            continue
        got = sx.pdf_difference(vol3, c, s, 0.0, 64.0, 64, kernel=kernel)
        assert got == want
    with pytest.raises(ValueError, match="degenerate scale"):
        sx.pdf_difference(vol3, [16.0, 16.0, 16.0], 1.5, 0.0, 64.0, 64)


@pytest.mark.parametrize("kernels", [("identity", "identity"), ("epanechnikov", "epanechnikov"),
                                     ("gaussian", "identity")])
def test_shift_step_matches_reference(sx, R, vol3, kernels):
    step_k, hist_k = kernels
    rng = np.random.default_rng(3)
    for _ in range(16):
        x = rng.uniform(-2.0, 33.0, size=3)
        half = rng.uniform(2.0, 9.0, size=3)
        want, _ = R.shift_step(vol3, 0.0, 64.0, 64, x, half, step_kernel=step_k, hist_kernel=hist_k)
        got = sx.shift_step(vol3, x, half, 0.0, 64.0, 64, step_kernel=step_k, hist_kernel=hist_k)
        assert (got is None) == (want is None)
        if got is not None:
            if step_k == "gaussian":
                np.testing.assert_allclose(got, want, rtol=0, atol=1e-12)
            else:
                assert got.tobytes() == want.tobytes()


def test_box_entropy_and_quadrant_step_match_reference(sx, R, oracle):
    img, _ = oracle.make_phantom(phantoms.square_2d(64, 31.0, 31.0, 8, 64, 77))
    rng = np.random.default_rng(4)
    for _ in range(20):
        x0, x1, y0, y1 = rng.uniform(-5, 70, size=4)
        want, _ = R.box_entropy_bits(img, 0.0, 64.0, 64, x0, x1, y0, y1)
        got = sx.box_entropy_bits(img, x0, x1, y0, y1, window_low=0.0, window_high=64.0, bins=64)
        assert math.isclose(got, want, rel_tol=1e-12, abs_tol=1e-15)
    pts = rng.uniform(0, 63, size=(24, 2))
    moved, st, visits = sx.ascent_step(img, pts, [4, 6, 8, 10], 0.0, 64.0, 64, dims=2)
    total = 0
    for i, p in enumerate(pts):
        m, s, v = R.quadrant_step(img, 0.0, 64.0, 64, p, [4, 6, 8, 10])
        total += v
        np.testing.assert_allclose(moved[i][:2], m, rtol=0, atol=1e-9)
        assert list(st[i]["best_scale"][:4]) == list(s.best_scale[:4])
        np.testing.assert_allclose(st[i]["entropy"][:4], list(s.entropy[:4]), rtol=1e-12)
        assert bool(st[i]["degenerate"]) == bool(s.degenerate)
    assert visits == total


def test_octant_step_and_3d_box_bit_exact_vs_oracle_shared_log(sx, oracle, vol3):
    """The octant step (NEW, no reference) and 3D boxes against the oracle's restatement
    in the device's own math (shared sx_log): bit-identical."""
    rng = np.random.default_rng(5)
    pts = rng.uniform(0, 31, size=(16, 3))
    scales = [3, 5, 7]
    moved, st, visits = sx.ascent_step(vol3, pts, scales, 0.0, 64.0, 64, dims=3)
    oracle.set_log_mode(1)
    try:
        for i, p in enumerate(pts):
            m, s = oracle.ascent_step(vol3, 0.0, 64.0, 64, p, scales, dims=3)
            assert moved[i].tobytes() == np.asarray(m).tobytes()
            assert st[i]["entropy"].tobytes() == s["entropy"].tobytes()
            assert list(st[i]["best_scale"]) == list(s["best_scale"])
            assert st[i]["norm_entropy"].tobytes() == s["norm_entropy"].tobytes()
        for _ in range(12):
            b = rng.uniform(-4, 36, size=6)
            got = sx.box_entropy_bits(vol3, *b, window_low=0.0, window_high=64.0, bins=64,
                                      min_voxels=8)
            want = oracle.box_entropy_bits(vol3, 0.0, 64.0, 64, *b, min_voxels=8)
            assert got == want
    finally:
        oracle.set_log_mode(0)
