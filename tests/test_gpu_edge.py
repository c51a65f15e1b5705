"""GPU parity on edge cases: ragged and tiny volumes, thin slabs, the maximum
halo, out-of-window intensities, duplicate / non-integer scales, boundary seeds,
the other histogram kernels, random seed plans and custom targets."""
import numpy as np
import pytest

from tests import phantoms

pytestmark = pytest.mark.gpu

RTOL, ATOL = 1e-5, 1e-6


def _noise(shape, seed, lo=-5.0, hi=40.0):
    rng = np.random.default_rng(seed)
    return rng.uniform(lo, hi, size=shape).astype(np.float32)


def _exh_equal(sx, oracle, vol, low, high, bins, scales):
    score, best, maxima, visits = sx.kadir_brady_exhaustive_records(vol, scales, low, high, bins,
                                                                    budget=10**12)
    rs, rb, rv = oracle.exhaustive(vol, low, high, bins, scales, budget=10**12, mode="exact",
                                   threads=8)
    excess = np.abs(score.astype(np.float64) - rs) - (
        RTOL * np.maximum(np.abs(score), np.abs(rs)) + ATOL)
    assert excess.max() <= 0.0
    assert (best == rb).mean() > 0.995
    assert visits == rv
    lin = oracle.local_maxima(score, best)[3]
    assert np.array_equal(maxima["linear_index"], lin)


@pytest.mark.parametrize("shape,scales,bins", [
    ((23, 29, 37), [3.0, 4.0, 5.0, 6.0, 7.0], 32),   # ragged vs the 8^3 tile
    ((2, 40, 33), [3.0, 5.0], 16),                    # thin slab
    ((3, 4, 5), [2.0, 3.0], 32),                      # smaller than the halo
    ((34, 36, 40), [float(s) for s in range(3, 16)], 16),  # R = 16, C1-style scale set
    ((1, 77, 61), [4.0, 6.0, 8.0, 10.0], 16),         # 2D, 17-bin path
    ((20, 20, 20), [4.0, 4.0, 6.0], 64),              # duplicate scales, 65-bin path
    ((16, 18, 20), [2.5, 3.5], 32),                   # non-integer but ring-adjacent radii
])
def test_exhaustive_edge_shapes(sx, oracle, shape, scales, bins):
    vol = _noise(shape, sum(shape))  # includes values below and above the window
    _exh_equal(sx, oracle, vol, 0.0, 32.0, bins, scales)


def test_exhaustive_single_voxel_and_unsupported(sx, oracle):
    s, b, m, v = sx.kadir_brady_exhaustive_records(np.ones((1, 1, 1), np.float32), [2.0], 0, 8, 8)
    assert s.shape == (1, 1, 1) and s[0, 0, 0] == 0.0 and len(m) == 0
    with pytest.raises(NotImplementedError):  # s-1, s, s+1 not adjacent radii
        sx.kadir_brady_exhaustive(np.ones((8, 8, 8), np.float32), [2.5, 3.0], 0, 8, 8)
    with pytest.raises(NotImplementedError):  # halo > 16 voxels
        sx.kadir_brady_exhaustive(np.ones((8, 8, 8), np.float32), [16.0], 0, 8, 8)
    with pytest.raises(NotImplementedError):  # Gaussian: no exact integer shell form
        sx.kadir_brady_exhaustive(np.ones((8, 8, 8), np.float32), [3.0], 0, 8, 8,
                                  kernel="gaussian")


def _seek_equal(gpu, ref, exact=True):
    for f in ["center", "H", "iterations", "flags"]:
        assert np.array_equal(gpu[f], ref[f]), f
    for f in ["entropy_bits", "pdf_diff", "bhattacharyya"]:
        if exact:
            assert np.array_equal(gpu[f], ref[f]), f
        else:
            assert np.allclose(gpu[f], ref[f], rtol=1e-9, atol=1e-12), f


@pytest.mark.parametrize("hist_kernel,step_kernel", [("identity", "identity"),
                                                     ("epanechnikov", "identity"),
                                                     ("identity", "epanechnikov")])
def test_shift_boundary_seeds_and_kernels(sx, oracle, hist_kernel, step_kernel):
    vol, _ = oracle.make_phantom(phantoms.ball_3d(40, (30.0, 9.0, 20.0), 7.0, 5))
    seeds = np.array([[0.0, 0.0, 0.0], [39.0, 39.0, 39.0], [-5.0, 20.0, 50.0], [30.0, 3.0, 20.0],
                      [35.5, 9.25, 19.75], [20.0, 20.0, 20.0]])
    gpu, gv = sx.seek_records(vol, seeds, half_extents=[6.0, 6.0, 6.0], method="shift",
                              window_low=0, window_high=64, bins=64, shift_hist_kernel=hist_kernel,
                              shift_step_kernel=step_kernel)
    oracle.set_log_mode(1)
    try:
        rv = 0
        for i, s in enumerate(seeds):
            ref, v = oracle.saliency_shift(vol, 0, 64, 64, s, [6.0, 6.0, 6.0],
                                           hist_kernel=hist_kernel, step_kernel=step_kernel)
            rv += v
            _seek_equal(gpu[i], ref)
        assert gv == rv
    finally:
        oracle.set_log_mode(0)


def test_shift_gaussian_kernel_within_tolerance(sx, oracle):
    """exp() differs between libdevice and glibc by <= 1 ulp: Gaussian-kernel
    trajectories agree to 1e-9, not bit for bit."""
    vol, _ = oracle.make_phantom(phantoms.cube_3d(32, 6, 3))
    seeds = np.array([[10.0, 12.0, 14.0], [20.0, 18.0, 16.0]])
    gpu, _ = sx.seek_records(vol, seeds, half_extents=[5.0, 5.0, 5.0], method="shift",
                             window_low=0, window_high=64, bins=64,
                             shift_hist_kernel="gaussian", shift_step_kernel="gaussian")
    oracle.set_log_mode(1)
    try:
        for i, s in enumerate(seeds):
            ref, _ = oracle.saliency_shift(vol, 0, 64, 64, s, [5.0, 5.0, 5.0],
                                           hist_kernel="gaussian", step_kernel="gaussian")
            assert np.allclose(gpu[i]["center"], ref["center"], rtol=0, atol=1e-9)
            assert gpu[i]["iterations"] == ref["iterations"]
    finally:
        oracle.set_log_mode(0)


def test_detect_random_seeds_custom_target_and_2d(sx, oracle):
    vol, _ = oracle.make_phantom(phantoms.ball_3d(48, (24.0, 20.0, 26.0), 8.0, 404,
                                                 background={"type": "gaussian", "mean": 8.0,
                                                             "sigma": 2.0}))
    kw = dict(method="shift", seed_mode="random", seed_count=37, rng_seed=9, scales=[5.0, 8.0],
              k=10, dedupe_radius=4.0)
    sel, seeds, visits = sx.detect_records(vol, window_low=0, window_high=64, bins=64,
                                           per_seed=True, **kw)
    okw = dict(kw)
    okw["top_k"] = okw.pop("k")
    oracle.set_log_mode(1)
    try:
        rsel, rseeds, rv = oracle.detect(vol, 0, 64, 64, **okw)
    finally:
        oracle.set_log_mode(0)
    for f in ["center", "iterations", "flags", "seed_index", "entropy_bits", "pdf_diff"]:
        assert np.array_equal(seeds[f], rseeds[f]), f
        assert np.array_equal(sel[f], rsel[f]), f
    assert visits == rv
    # custom (non-uniform) target pmf: histogram_from_array normalizes it
    target = np.linspace(1.0, 2.0, 64)
    d, _ = sx.seek_records(vol, [[20.0, 22.0, 24.0]], half_extents=[6.0, 6.0, 6.0],
                           method="shift", window_low=0, window_high=64, bins=64, target=target)
    oracle.set_log_mode(1)
    try:
        mass = 0.0
        for t in target:  # Histogram::normalize: sequential mass (histogram.hpp:21-33)
            mass += float(t)
        ref, _ = oracle.saliency_shift(vol, 0, 64, 64, [20.0, 22.0, 24.0], [6.0, 6.0, 6.0],
                                       target=target / mass)
    finally:
        oracle.set_log_mode(0)
    _seek_equal(d[0], ref)


def test_octant_on_2d_and_single_scale_quadrant(sx, oracle):
    vol, _ = oracle.make_phantom(phantoms.square_2d(64, 31.0, 31.0, 8, 64, 77))
    res, _ = sx.quadrant_seek(vol, [[20.0, 20.0, 0.0]], [5], 0, 64, 64, octant=True)
    oracle.set_log_mode(1)
    try:
        ref = oracle.ascent_seek_one(vol, 0, 64, 64, [20.0, 20.0, 0.0], [5], dims=3)
        assert np.array_equal(res[0]["position"], ref["position"])
        res2, _ = sx.quadrant_seek(vol, [[20.0, 20.0]], [6], 0, 64, 64)
        ref2 = oracle.ascent_seek_one(vol, 0, 64, 64, [20.0, 20.0], [6])
        assert np.array_equal(res2[0]["position"], ref2["position"])
    finally:
        oracle.set_log_mode(0)


@pytest.mark.parametrize("dims,scales", [
    (3, list(range(1, 41))),   # 40 scales x 64 bins: the shell-by-shell kernel (tables > 160 KB)
    (3, [2, 3, 5, 8, 13]),     # level-table kernel, sparse scale set
    (2, list(range(1, 61))),   # quadrant, shell kernel
    (2, [0, 1, 4, 9]),         # quadrant, level tables, k = 0 (empty boxes)
])
def test_ascent_both_kernels_match_oracle(sx, oracle, dims, scales):
    if dims == 3:
        vol, _ = oracle.make_phantom(phantoms.ball_3d(36, (20.0, 15.0, 17.0), 7.0, 91))
        seeds = [[10.0, 12.0, 14.0], [25.5, 20.25, 9.0], [0.0, 35.0, 35.0]]
    else:
        vol, _ = oracle.make_phantom(phantoms.square_2d(80, 41.0, 37.0, 9, 64, 92))
        seeds = [[30.0, 30.0, 0.0], [60.5, 12.25, 0.0], [0.0, 79.0, 0.0]]
    res, _ = sx.quadrant_seek(vol, seeds, scales, 0, 64, 64, octant=dims == 3)
    oracle.set_log_mode(1)
    try:
        for r, s in zip(res, seeds):
            ref = oracle.ascent_seek_one(vol, 0, 64, 64, s if dims == 3 else s[:2], scales,
                                         dims=dims)
            assert np.array_equal(r["position"][:dims], np.asarray(ref["position"])[:dims])
            assert r["iterations"] == ref["iterations"]
            assert r["best_scale"] == ref["best_scale"]
            assert r["entropy_bits"] == ref["entropy_bits"]
    finally:
        oracle.set_log_mode(0)
