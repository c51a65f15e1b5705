"""Parity at BASELINE.json's full sizes (C1, C2, C3), where the oracle cannot
redo the whole job in test time: exact histograms at random voxels, oracle
scores on sampled rows, size-independent properties of the full outputs
(strict 26-neighbour maxima, the stable order, visits closed form), and
bit-exact trajectories for random samples of the seeds."""
import numpy as np
import pytest

from tests import phantoms

pytestmark = pytest.mark.gpu
C2_SCALES = [float(s) for s in range(3, 16)]


@pytest.fixture(scope="module")
def c2(sx):
    vol, _ = sx.make_phantom(phantoms.config_c2())
    score, best, maxima, visits = sx.kadir_brady_exhaustive_records(vol, C2_SCALES, 0, 32, 32,
                                                                    budget=10**13)
    return vol, score, best, maxima, visits


def test_c2_exact_histograms_at_random_voxels(sx, oracle, c2):
    vol = c2[0]
    rng = np.random.default_rng(2)
    lin = np.concatenate([[0, vol.size - 1], rng.integers(0, vol.size, 30)])
    radii, hist = sx.exhaustive_debug_hist(lin, 32, len(C2_SCALES))
    for i, l in enumerate(lin):
        z, y, x = np.unravel_index(l, vol.shape)
        for ri in (0, len(radii) // 2, len(radii) - 1):
            S = oracle.voxel_shell_hist(vol, 0, 32, 32, int(x), int(y), int(z), radii[ri])
            assert np.array_equal(hist[i, ri, :32].astype(np.uint64), S)


def test_c2_scores_on_sampled_rows(oracle, c2):
    vol, score, best = c2[0], c2[1], c2[2]
    for z, y in ((128, 90), (200, 190), (3, 250)):
        rs, rb, _ = oracle.exhaustive(vol, 0, 32, 32, C2_SCALES, budget=10**13, mode="exact",
                                      threads=8, z_range=(z, z + 1), y_range=(y, y + 1))
        g, r = score[z, y].astype(np.float64), rs[z, y].astype(np.float64)
        excess = np.abs(g - r) - (1e-5 * np.maximum(np.abs(g), np.abs(r)) + 1e-6)
        assert excess.max() <= 0.0
        assert (best[z, y] == rb[z, y]).mean() > 0.99


def test_c2_maxima_properties_and_visits(c2):
    vol, score, best, maxima, visits = c2
    nz, ny, nx = score.shape
    # strict 26-neighbour maxima with score > 0 (pipeline.cpp:143-160), checked by numpy
    pad = np.pad(score, 1, constant_values=-np.inf)
    strict = score > 0
    for dz in (-1, 0, 1):
        for dy in (-1, 0, 1):
            for dx in (-1, 0, 1):
                if dz == dy == dx == 0:
                    continue
                strict &= score > pad[1 + dz:1 + dz + nz, 1 + dy:1 + dy + ny, 1 + dx:1 + dx + nx]
    lin = np.flatnonzero(strict.ravel())
    assert len(maxima) == len(lin)
    assert np.array_equal(np.sort(maxima["linear_index"]), lin)
    order = np.lexsort((lin, -score.ravel()[lin]))  # stable_sort: score desc, index asc
    assert np.array_equal(maxima["linear_index"], lin[order])
    # EvalCounter: N * sum_r |B(r)| (pipeline.cpp:118, 141)
    per = 0
    for r in range(2, 17):
        g = np.arange(-r, r + 1)
        z, y, x = np.meshgrid(g, g, g, indexing="ij")
        per += int(((x * x + y * y + z * z) <= r * r).sum())
    assert visits == vol.size * per


def test_c3_random_seed_trajectories_bit_exact(sx, oracle):
    vol, _ = sx.make_phantom(phantoms.config_c3())
    sel, seeds, visits = sx.detect_records(vol, "shift", 16.0, [8.0, 12.0], 20, 5.0, 0, 64, 64,
                                           per_seed=True)
    assert len(seeds) == 5120 and len(sel) == 20
    pos, sc = sx.plan_seeds(vol.shape, spacing=16.0, scales=[8.0, 12.0])
    rng = np.random.default_rng(3)
    oracle.set_log_mode(1)
    try:
        for i in rng.choice(len(seeds), 24, replace=False):
            s = sc[i]
            ref, _ = oracle.saliency_shift(vol, 0, 64, 64, pos[i], [s, s, s])
            for f in ["center", "iterations", "flags", "entropy_bits", "pdf_diff", "bhattacharyya"]:
                assert np.array_equal(seeds[i][f], ref[f]), (i, f)
    finally:
        oracle.set_log_mode(0)


def test_c1_random_octant_trajectories_bit_exact(sx, oracle):
    vol, _ = sx.make_phantom(phantoms.config_c1())
    scales = [float(s) for s in range(3, 16)]
    res, _ = sx.quadrant_seek(vol, [[float(x), float(y), float(z)] for z in (4, 60, 124)
                                    for y in (4, 68) for x in (12, 76, 124)],
                              [int(s) for s in scales], 0, 16, 16, octant=True)
    oracle.set_log_mode(1)
    try:
        for r, (z, y, x) in zip(res, [(z, y, x) for z in (4, 60, 124) for y in (4, 68)
                                      for x in (12, 76, 124)]):
            ref = oracle.ascent_seek_one(vol, 0, 16, 16, [x, y, z], [int(s) for s in scales],
                                         dims=3)
            assert np.array_equal(r["position"], ref["position"])
            assert r["iterations"] == ref["iterations"] and r["entropy_bits"] == ref["entropy_bits"]
    finally:
        oracle.set_log_mode(0)
