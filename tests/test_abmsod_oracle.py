"""ABMSOD oracle pinned to the reference's own tests (tests/test_seek.cpp:427-622,
tests/test_pipeline.cpp:321-354): bandwidth_from_moment known answers, the
SelfAdjointEigenSolver restatement, the shared exp/pow, and abmsod_run's
fixed point, orientation recovery, trace invariants, constant-volume rho,
self-target centroid and rotation equivariance."""
import math

import numpy as np
import pytest

from tests import phantoms


def test_bandwidth_two_voxels_on_x_axis(oracle):  # test_seek.cpp:427-440
    d = 3.0
    outer = np.zeros((3, 3))
    for s in (d, -d):
        v = np.array([s, 0.0, 0.0])
        outer += np.outer(v, v)
    H = oracle.bandwidth_from_moment(outer, 2.0, 3, 4.0, 1024.0)
    ev = np.sort(np.linalg.eigvalsh(H))
    assert ev == pytest.approx([4.0, 4.0, 5.0 * d * d])


def test_bandwidth_rank1_clamped_spd(oracle):  # test_seek.cpp:442-450
    r = np.array([2.0, -1.0, 3.0])
    outer = 0.7 * np.outer(r, r)
    H = oracle.bandwidth_from_moment(outer, 0.7, 3, 4.0, 4096.0)
    assert np.linalg.eigvalsh(H).min() >= 4.0 - 1e-12
    assert np.linalg.norm(H - H.T) < 1e-12
    with pytest.raises(oracle.OracleError):
        oracle.bandwidth_from_moment(outer, 0.0, 3, 4.0, 4096.0)
    bad = outer.copy()
    bad[0, 1] = np.inf
    with pytest.raises(oracle.OracleError):
        oracle.bandwidth_from_moment(bad, 0.7, 3, 4.0, 4096.0)


def test_bandwidth_uniform_box_aligns_with_axes(oracle):  # test_seek.cpp:452-466
    outer = np.zeros((3, 3))
    wsum = 0.0
    for z in range(-2, 3):
        for y in range(-4, 5):
            for x in range(-6, 7):
                v = np.array([x, y, z], np.float64)
                outer += np.outer(v, v)
                wsum += 1.0
    H = oracle.bandwidth_from_moment(outer, wsum, 3, 1.0, 4096.0)
    _, vecs = oracle.sym_eigen3(H)
    assert abs(vecs[:, 2] @ np.array([1.0, 0.0, 0.0])) > math.cos(math.radians(5.0))


@pytest.mark.parametrize("seed", [1, 2, 3, 4])
def test_sym_eigen3_matches_lapack(oracle, seed):
    rng = np.random.default_rng(seed)
    a = rng.normal(size=(3, 3))
    a = a @ a.T + np.diag(rng.uniform(0.1, 5.0, 3))
    if seed == 4:
        a[2, 0] = a[0, 2] = 0.0  # already tridiagonal: the v1norm2 <= tol branch
    vals, vecs = oracle.sym_eigen3(a)
    assert np.allclose(vals, np.linalg.eigvalsh(a), rtol=1e-13, atol=1e-13)
    assert np.all(np.diff(vals) >= 0)
    assert np.allclose(a @ vecs, vecs * vals, atol=1e-12)
    assert np.allclose(vecs.T @ vecs, np.eye(3), atol=1e-13)


def test_shared_exp_pow_close_to_glibc(oracle):
    for x in np.concatenate([-np.linspace(0, 0.5, 101), np.linspace(-30, 30, 61)]):
        assert oracle.exp_portable(x) == pytest.approx(math.exp(x), rel=4e-16, abs=0)
    for x in [1e-3, 0.5, 2.0, 81.0 * 36.0 * 16.0, 1e6, 1e12]:
        for y in [0.25, 1.0 / 6.0]:
            assert oracle.pow_portable(x, y) == pytest.approx(x ** y, rel=2e-15)


def _ellipsoid(oracle, axes, seed, dim=64):
    vol, _ = oracle.make_phantom(phantoms.ellipsoid_3d(axes, seed, dim))
    c = (dim - 1) / 2.0
    return vol, np.array([c, c, c]), phantoms.ellipsoid_H(axes)


def test_abmsod_fixed_point_matched_ellipsoid(oracle):  # test_seek.cpp:495-514
    vol, c, H = _ellipsoid(oracle, np.diag([9.0, 6.0, 4.0]), 111)
    det, _, _ = oracle.abmsod_run(vol, 0, 64, 64, c, H=H)
    assert not det["flags"] & 2
    assert np.linalg.norm(det["center"] - c) <= 1.0
    ev = np.sqrt(np.linalg.eigvalsh(det["H"].reshape(3, 3)))
    assert ev == pytest.approx([4.0, 6.0, 9.0], rel=0.10)


def test_abmsod_recovers_oblique_orientation(oracle):  # test_seek.cpp:516-541
    axes = phantoms.rot_z(45.0) @ np.diag([9.0, 4.0, 4.0])
    vol, c, H = _ellipsoid(oracle, axes, 222)
    det, trace, _ = oracle.abmsod_run(vol, 0, 64, 64, c, radius=6.0, trace=True)
    assert not det["flags"] & 2
    got = np.linalg.eigh(det["H"].reshape(3, 3))[1][:, 2]
    want = np.linalg.eigh(H)[1][:, 2]
    assert abs(got @ want) > math.cos(math.radians(15.0))
    lmax = (64 / 2.0) ** 2
    prev = 0.0
    assert len(trace) >= 1
    for rec in trace:
        assert rec["eig_min"] >= 4.0 - 1e-9
        assert rec["eig_max"] <= lmax + 1e-9
        assert rec["max_bhattacharyya"] >= prev
        prev = rec["max_bhattacharyya"]


def test_abmsod_fitted_beats_cuboid(oracle):  # test_seek.cpp:543-559
    axes = phantoms.rot_z(45.0) @ np.diag([9.0, 4.0, 4.0])
    vol, c, _ = _ellipsoid(oracle, axes, 333)
    seed = c + np.array([2.0, 1.0, 0.0])
    cub, _ = oracle.saliency_shift(vol, 0, 64, 64, seed, [8.0, 8.0, 8.0])
    fit, _, _ = oracle.abmsod_run(vol, 0, 64, 64, seed, radius=8.0)
    assert not cub["flags"] & 2 and not fit["flags"] & 2
    assert fit["entropy_bits"] > cub["entropy_bits"]


def test_abmsod_constant_volume_rho(oracle):  # test_seek.cpp:561-571
    vol = np.full((32, 32, 32), 20.0, np.float32)
    det, trace, _ = oracle.abmsod_run(vol, 0, 64, 64, [16.0, 16.0, 16.0], radius=6.0, trace=True)
    assert len(trace) >= 1
    assert trace[0]["bhattacharyya"] == pytest.approx(math.sqrt(1.0 / 64), rel=1e-12)
    assert det["entropy_bits"] == 0.0


def test_abmsod_self_target_first_update_is_kernel_centroid(oracle):  # test_seek.cpp:573-593
    vol, c, _ = _ellipsoid(oracle, np.diag([8.0, 6.0, 5.0]), 444)
    seed = c + np.array([3.0, 0.0, 0.0])
    Hs = np.diag([36.0, 36.0, 36.0])
    target = oracle.candidate_histogram(vol, 0, 64, 64, seed, Hs, kernel="gaussian")
    det, trace, _ = oracle.abmsod_run(vol, 0, 64, 64, seed, radius=6.0, max_iterations=1,
                                      target=target, trace=True)
    assert len(trace) == 1
    num, den = np.zeros(3), 0.0
    nz, ny, nx = vol.shape
    for z in range(nz):
        for y in range(ny):
            for x in range(nx):
                d2 = ((x - seed[0]) ** 2 + (y - seed[1]) ** 2 + (z - seed[2]) ** 2) / 36.0
                if d2 <= 1.0:
                    g = 0.5 * math.exp(-0.5 * d2)
                    num += g * np.array([x, y, z], np.float64)
                    den += g
    assert np.linalg.norm(trace[0]["position"] - num / den) < 1e-9


def test_abmsod_equivariant_under_rotation(oracle):  # test_seek.cpp:595-622
    axes = phantoms.rot_z(30.0) @ np.diag([8.0, 4.0, 4.0])
    vol, c, _ = _ellipsoid(oracle, axes, 555, dim=48)
    rv = np.zeros_like(vol)  # (x, y) -> (47 - y, x)
    for y in range(48):
        for x in range(48):
            rv[:, x, 47 - y] = vol[:, y, x]
    off = np.array([3.0, 1.0, 0.0])
    plain, _, _ = oracle.abmsod_run(vol, 0, 64, 64, c + off, radius=6.0)
    R = np.array([[0.0, -1.0, 0.0], [1.0, 0.0, 0.0], [0.0, 0.0, 1.0]])
    t = np.array([47.0, 0.0, 0.0])
    rot, _, _ = oracle.abmsod_run(rv, 0, 64, 64, R @ (c + off) + t, radius=6.0)
    assert not plain["flags"] & 2 and not rot["flags"] & 2
    assert np.linalg.norm(rot["center"] - (R @ plain["center"] + t)) < 1e-6
    Hp = plain["H"].reshape(3, 3)
    assert np.linalg.norm(rot["H"].reshape(3, 3) - R @ Hp @ R.T) < 1e-6


def test_abmsod_detect_and_invalid_params(oracle):  # test_pipeline.cpp:321-354 (shape)
    axes = phantoms.rot_z(45.0) @ np.diag([9.0, 4.0, 4.0])
    vol, c, _ = _ellipsoid(oracle, axes, 333, dim=48)
    sel, seeds, visits = oracle.detect(vol, 0, 64, 64, method="abmsod", seed_spacing=16.0,
                                       scales=[6.0], top_k=5, dedupe_radius=5.0)
    assert len(seeds) == 27 and visits > 0
    assert len(sel) >= 1
    assert np.linalg.norm(sel[0]["center"] - c) < 6.0
    with pytest.raises(oracle.OracleError):
        oracle.abmsod_run(vol, 0, 64, 64, c, radius=6.0, threshold=0.0)


def test_capi_bandwidth_from_moment_matches_oracle(sx, oracle):
    """salvox_bandwidth_from_moment (host C-ABI, same sx_eig3.h) == the oracle, bit for bit."""
    rng = np.random.default_rng(7)
    for _ in range(20):
        pts = rng.normal(scale=rng.uniform(1, 6, 3), size=(50, 3))
        w = rng.uniform(0.1, 2.0, 50)
        outer = sum(wi * np.outer(p, p) for wi, p in zip(w, pts))
        a = sx.bandwidth_from_moment(outer, w.sum(), 3, 4.0, 1024.0)
        b = oracle.bandwidth_from_moment(outer, w.sum(), 3, 4.0, 1024.0)
        assert a.tobytes() == b.tobytes()
    with pytest.raises(ValueError, match="zero weight mass"):
        sx.bandwidth_from_moment(np.eye(3), 0.0, 3, 4.0, 1024.0)
