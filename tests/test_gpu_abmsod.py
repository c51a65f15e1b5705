"""GPU parity of the ABMSOD adaptive-bandwidth seek vs the
oracle restatement of src/abmsod.cpp.

Contract: with the oracle in shared-math mode (sx_log + sx_exp + sx_pow, mode 7:
the functions the kernel evaluates) every output is bit-exact -- best centre,
bandwidth H, iterations, flags, scores, per-iteration trace, EvalCounter
visits, and detect()'s per-seed and selected detections. Against the glibc
oracle (mode 0) trajectories agree to 1e-9 (exp/pow differ by ulps). The
reference's own ABMSOD properties (tests/test_seek.cpp:495-622) hold on the
device results.
"""
import math

import numpy as np
import pytest

from tests import phantoms

pytestmark = pytest.mark.gpu

SHARED = 7  # oracle math: sx_log | sx_exp | sx_pow
FIELDS = ["center", "H", "iterations", "flags", "entropy_bits", "pdf_diff", "bhattacharyya"]


def _ellipsoid(oracle, axes, seed, dim=64):
    vol, _ = oracle.make_phantom(phantoms.ellipsoid_3d(axes, seed, dim))
    c = (dim - 1) / 2.0
    return vol, np.array([c, c, c]), phantoms.ellipsoid_H(axes)


def _oracle_run(oracle, vol, seeds, mode=SHARED, **kw):
    oracle.set_log_mode(mode)
    try:
        return [oracle.abmsod_run(vol, 0, 64, 64, s, **kw) for s in seeds]
    finally:
        oracle.set_log_mode(0)


def _same(gpu, ref):
    for f in FIELDS:
        assert np.array_equal(gpu[f], ref[f]), f


def test_abmsod_oblique_ellipsoid_bit_exact_with_trace(sx, oracle):
    axes = phantoms.rot_z(45.0) @ np.diag([9.0, 4.0, 4.0])
    vol, c, _ = _ellipsoid(oracle, axes, 222)
    seeds = [c, c + [2.0, 1.0, 0.0], c + [-5.0, 3.5, 2.25], [0.0, 0.0, 0.0], [63.0, 10.0, 31.5]]
    gpu, traces, visits = sx.abmsod_records(vol, seeds, radius=6.0, window_low=0, window_high=64,
                                            trace=True)
    refs = _oracle_run(oracle, vol, seeds, radius=6.0, trace=True)
    rv = 0
    for g, t, (r, rt, v) in zip(gpu, traces, refs):
        _same(g, r)
        assert t.tobytes() == rt.tobytes()
        rv += v
    assert visits == rv


def test_abmsod_matched_fixed_point_and_reference_properties(sx, oracle):  # test_seek.cpp:495-514
    vol, c, H = _ellipsoid(oracle, np.diag([9.0, 6.0, 4.0]), 111)
    gpu, _, visits = sx.abmsod_records(vol, [c], H=H, window_low=0, window_high=64)
    (r, _, v), = _oracle_run(oracle, vol, [c], H=H)
    _same(gpu[0], r)
    assert visits == v
    assert not gpu[0]["flags"] & 2
    assert np.linalg.norm(gpu[0]["center"] - c) <= 1.0
    ev = np.sqrt(np.linalg.eigvalsh(gpu[0]["H"].reshape(3, 3)))
    assert ev == pytest.approx([4.0, 6.0, 9.0], rel=0.10)


def test_abmsod_constant_volume_and_self_target(sx, oracle):  # test_seek.cpp:561-593
    vol = np.full((32, 32, 32), 20.0, np.float32)
    gpu, tr, _ = sx.abmsod_records(vol, [[16.0, 16.0, 16.0]], radius=6.0, window_low=0,
                                   window_high=64, trace=True)
    assert tr[0][0]["bhattacharyya"] == pytest.approx(math.sqrt(1.0 / 64), rel=1e-12)
    assert gpu[0]["entropy_bits"] == 0.0
    vol2, c, _ = _ellipsoid(oracle, np.diag([8.0, 6.0, 5.0]), 444)
    seed = c + [3.0, 0.0, 0.0]
    oracle.set_log_mode(SHARED)
    try:
        target = oracle.candidate_histogram(vol2, 0, 64, 64, seed, np.diag([36.0] * 3), "gaussian")
    finally:
        oracle.set_log_mode(0)
    g2, t2, _ = sx.abmsod_records(vol2, [seed], radius=6.0, window_low=0, window_high=64,
                                  max_iterations=1, target=target, trace=True)
    dev_target = sx.api.histogram_from_array(target)  # what the Python layer hands the device
    (r2, rt2, _), = _oracle_run(oracle, vol2, [seed], radius=6.0, max_iterations=1,
                                target=dev_target, trace=True)
    _same(g2[0], r2)
    assert t2[0].tobytes() == rt2.tobytes()


def test_abmsod_2d_and_glibc_tolerance(sx, oracle):
    vol, _ = oracle.make_phantom(phantoms.square_2d(80, 41.0, 37.0, 9, 64, 92))
    seeds = [[36.0, 33.0, 0.0], [50.5, 40.25, 0.0]]
    gpu, _, visits = sx.abmsod_records(vol, seeds, radius=7.0, window_low=0, window_high=64)
    refs = _oracle_run(oracle, vol, seeds, radius=7.0)
    for g, (r, _, _) in zip(gpu, refs):
        _same(g, r)
    assert visits == sum(v for _, _, v in refs)
    axes = phantoms.rot_z(30.0) @ np.diag([8.0, 4.0, 4.0])
    vol3, c, _ = _ellipsoid(oracle, axes, 555, dim=48)
    g3, _, _ = sx.abmsod_records(vol3, [c + [3.0, 1.0, 0.0]], radius=6.0, window_low=0,
                                 window_high=64)
    (r3, _, _), = _oracle_run(oracle, vol3, [c + [3.0, 1.0, 0.0]], mode=0, radius=6.0)
    assert np.allclose(g3[0]["center"], r3["center"], rtol=0, atol=1e-9)
    assert np.allclose(g3[0]["H"], r3["H"], rtol=1e-9, atol=1e-9)
    assert g3[0]["iterations"] == r3["iterations"]


def test_abmsod_equivariant_under_rotation(sx, oracle):  # test_seek.cpp:595-622
    axes = phantoms.rot_z(30.0) @ np.diag([8.0, 4.0, 4.0])
    vol, c, _ = _ellipsoid(oracle, axes, 555, dim=48)
    rv = np.zeros_like(vol)
    for y in range(48):
        for x in range(48):
            rv[:, x, 47 - y] = vol[:, y, x]
    off = np.array([3.0, 1.0, 0.0])
    R = np.array([[0.0, -1.0, 0.0], [1.0, 0.0, 0.0], [0.0, 0.0, 1.0]])
    t = np.array([47.0, 0.0, 0.0])
    p, _, _ = sx.abmsod_records(vol, [c + off], radius=6.0, window_low=0, window_high=64)
    q, _, _ = sx.abmsod_records(rv, [R @ (c + off) + t], radius=6.0, window_low=0, window_high=64)
    assert np.linalg.norm(q[0]["center"] - (R @ p[0]["center"] + t)) < 1e-6
    Hp = p[0]["H"].reshape(3, 3)
    assert np.linalg.norm(q[0]["H"].reshape(3, 3) - R @ Hp @ R.T) < 1e-6


def test_abmsod_detect_matches_oracle(sx, oracle):  # pipeline.cpp:371-379 + selection
    axes = phantoms.rot_z(45.0) @ np.diag([9.0, 4.0, 4.0])
    vol, c, _ = _ellipsoid(oracle, axes, 333, dim=48)
    kw = dict(seed_spacing=12.0, scales=[5.0, 7.0], k=5, dedupe_radius=5.0)
    sel, seeds, visits = sx.detect_records(vol, "abmsod", window_low=0, window_high=64, bins=64,
                                           per_seed=True, **kw)
    okw = dict(kw)
    okw["top_k"] = okw.pop("k")
    oracle.set_log_mode(SHARED)
    try:
        rsel, rseeds, rv = oracle.detect(vol, 0, 64, 64, method="abmsod", **okw)
    finally:
        oracle.set_log_mode(0)
    assert seeds.tobytes() == rseeds.tobytes()
    assert sel.tobytes() == rsel.tobytes()
    assert visits == rv
    assert np.linalg.norm(sel[0]["center"] - c) < 6.0
    d = sx.abmsod(vol, c + [2.0, 1.0, 0.0], 8.0, window_low=0, window_high=64)
    assert "degenerate" not in d["flags"] and d["entropy_bits"] > 0.0


def test_gaussian_shift_bit_exact_in_shared_math(sx, oracle):
    vol, _ = oracle.make_phantom(phantoms.cube_3d(32, 6, 3))
    seeds = np.array([[10.0, 12.0, 14.0], [20.0, 18.0, 16.0]])
    gpu, _ = sx.seek_records(vol, seeds, half_extents=[5.0, 5.0, 5.0], method="shift",
                             window_low=0, window_high=64, bins=64,
                             shift_hist_kernel="gaussian", shift_step_kernel="gaussian")
    oracle.set_log_mode(3)
    try:
        for i, s in enumerate(seeds):
            ref, _ = oracle.saliency_shift(vol, 0, 64, 64, s, [5.0, 5.0, 5.0],
                                           hist_kernel="gaussian", step_kernel="gaussian")
            for f in ["center", "iterations", "flags", "entropy_bits", "bhattacharyya"]:
                assert np.array_equal(gpu[i][f], ref[f]), f
    finally:
        oracle.set_log_mode(0)
