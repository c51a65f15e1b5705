"""GPU parity of the seed-grid detector (shift / quadrant / octant) vs the oracle.

Contract: converged positions, iteration counts, flags, seed indices, window H
are bit-exact; with the oracle in shared-log mode (sx_log on both sides) the
scores (entropy, Bhattacharyya, pdf_diff) are bit-exact too, and the selected
detections (thresholds + dedupe) are identical. Against the glibc-log oracle the
scores agree to 1e-12 relative.
"""
import numpy as np
import pytest

from tests import phantoms

pytestmark = pytest.mark.gpu

FIELDS_EXACT = ["center", "H", "iterations", "flags", "seed_index"]
FIELDS_SCORE = ["entropy_bits", "pdf_diff", "bhattacharyya"]


def _same(gpu, ref, scores_exact=True):
    assert len(gpu) == len(ref)
    for f in FIELDS_EXACT:
        assert np.array_equal(gpu[f], ref[f]), f
    for f in FIELDS_SCORE:
        if scores_exact:
            assert np.array_equal(gpu[f], ref[f]), f
        else:
            assert np.allclose(gpu[f], ref[f], rtol=1e-12, atol=1e-14), f


def _both(sx, oracle, vol, low, high, bins, **kw):
    sel, seeds, visits = sx.detect_records(vol, window_low=low, window_high=high, bins=bins,
                                           per_seed=True, **kw)
    okw = dict(kw)
    okw["top_k"] = okw.pop("k", 20)
    oracle.set_log_mode(1)
    try:
        rsel, rseeds, rvis = oracle.detect(vol, low, high, bins, **okw)
    finally:
        oracle.set_log_mode(0)
    return sel, seeds, visits, rsel, rseeds, rvis


def test_shift_finds_ball_center(sx, oracle):  # test_pipeline.cpp:296-319
    vol, cent = oracle.make_phantom(phantoms.ball_3d(64, (36.0, 30.0, 28.0), 9.0, 101))
    sel, seeds, visits, rsel, rseeds, rvis = _both(
        sx, oracle, vol, 0, 64, 64, method="shift", seed_spacing=16.0, scales=[6.0, 9.0], k=5,
        dedupe_radius=6.0)
    _same(seeds, rseeds)
    _same(sel, rsel)
    assert visits == rvis
    assert len(sel) > 0 and np.linalg.norm(sel[0]["center"] - cent[0]) <= 2.0


def test_shift_2d_and_anisotropic(sx, oracle):
    vol, _ = oracle.make_phantom(phantoms.cube_3d(48, 7, 83))
    rng = np.random.default_rng(13)
    seeds = rng.uniform(0, 47, size=(10, 3))
    gpu, _ = sx.seek_records(vol, seeds, half_extents=[6.0, 5.0, 4.0], method="shift",
                             window_low=0, window_high=64, bins=64)
    oracle.set_log_mode(1)
    try:
        for i, s in enumerate(seeds):  # test_seek.cpp:360-375
            ref, _ = oracle.saliency_shift(vol, 0, 64, 64, s, [6.0, 5.0, 4.0])
            for f in FIELDS_EXACT[:4] + FIELDS_SCORE:
                assert np.array_equal(gpu[i][f], ref[f]), (i, f)
    finally:
        oracle.set_log_mode(0)
    vol2, _ = oracle.make_phantom(phantoms.square_2d(96, 45.0, 49.0, 9, 64, 303))
    sel, seeds2, visits, rsel, rseeds, rvis = _both(
        sx, oracle, vol2, 0, 64, 64, method="shift", seed_spacing=12.0, scales=[6.0, 10.0], k=3,
        dedupe_radius=8.0)
    _same(seeds2, rseeds)
    _same(sel, rsel)


def test_shift_constant_volume_empty(sx, oracle):  # test_pipeline.cpp:381-392
    vol = np.ones((48, 48, 48), np.float32)
    assert sx.detect(vol, method="shift", seed_spacing=16.0, scales=[6.0], window_low=0,
                     window_high=64, bins=64) == []


def test_quadrant_matches_oracle(sx, oracle):  # test_pipeline.cpp:356-379 + test_seek.cpp:148-166
    vol, _ = oracle.make_phantom(phantoms.square_2d(128, 63.0, 63.0, 12, 64, 23))
    sel, seeds, visits, rsel, rseeds, rvis = _both(
        sx, oracle, vol, 0, 64, 64, method="quadrant", seed_spacing=16.0,
        scales=[4.0, 8.0, 12.0, 16.0], k=3, dedupe_radius=8.0)
    _same(seeds, rseeds)
    _same(sel, rsel)
    assert visits == rvis
    assert any(np.linalg.norm(d["center"][:2] - [63, 63]) <= 3 for d in seeds
               if not d["flags"] & 2)


def test_quadrant_requires_2d(sx):  # test_pipeline.cpp:394-400
    with pytest.raises(ValueError, match="requires a 2D volume"):
        sx.detect(np.zeros((16, 16, 16), np.float32), method="quadrant", window_low=0,
                  window_high=64, bins=64)


def test_octant_matches_oracle(sx, oracle):
    spec = phantoms.ball_3d(48, (26.0, 22.0, 24.0), 8.0, 55, levels=16,
                            background={"type": "gaussian", "mean": 4.0, "sigma": 1.5})
    vol, cent = oracle.make_phantom(spec)
    sel, seeds, visits, rsel, rseeds, rvis = _both(
        sx, oracle, vol, 0, 16, 16, method="octant", seed_spacing=12.0, scales=[3.0, 5.0, 7.0, 9.0],
        k=5, dedupe_radius=6.0)
    _same(seeds, rseeds)
    _same(sel, rsel)
    assert visits == rvis


def test_select_matches_oracle(sx, oracle):
    rng = np.random.default_rng(4)
    d = np.zeros(400, sx.DET_DTYPE)
    d["center"][:, 0] = rng.uniform(0, 500, 400)
    d["pdf_diff"] = rng.random(400)
    d["entropy_bits"] = rng.random(400) * 5
    d["flags"] = np.where(rng.random(400) < 0.1, 2, 1)
    d["entropy_bits"][::37] = 0.0
    d["seed_index"] = np.arange(400)
    got = sx.select(d, 0.9, 0.2, 20, 5.0)
    ref = oracle.select(d.view(oracle.DET_DTYPE), 0.9, 0.2, 20, 5.0)
    assert np.array_equal(got["seed_index"], ref["seed_index"])
    got2 = sx.dedupe_top_k(d, 20, 5.0)  # test_pipeline.cpp:55-83
    ref2 = oracle.dedupe_top_k(d.view(oracle.DET_DTYPE), 20, 5.0)
    assert np.array_equal(got2["seed_index"], ref2["seed_index"])
    assert len(sx.dedupe_top_k(d[:0], 20, 5.0)) == 0
    pair = np.zeros(2, sx.DET_DTYPE)
    pair["center"][:, 0] = [10, 11]
    pair["pdf_diff"] = [1.0, 2.0]
    out = sx.dedupe_top_k(pair, 20, 5.0)
    assert len(out) == 1 and out[0]["pdf_diff"] == 2.0


def test_raw_quadrant_and_octant_seek_match_oracle(sx, oracle):
    """salvox_ascent_seek == quadrant_seek_one (quadrant.cpp:83-114), bit for bit."""
    vol, _ = oracle.make_phantom(phantoms.square_2d(96, 40.0, 47.0, 10, 64, 57))
    seeds = [[32.0, 44.0], [60.5, 50.25], [5.0, 90.0], [47.0, 47.0]]
    res, visits = sx.quadrant_seek(vol, seeds, [4, 6, 10], 0, 64, 64, max_iters=8)
    oracle.set_log_mode(1)
    try:
        rv = 0
        for r, s in zip(res, seeds):
            ref = oracle.ascent_seek_one(vol, 0, 64, 64, s, [4, 6, 10], max_iters=8)
            assert np.array_equal(r["position"], ref["position"])
            assert r["best_scale"] == ref["best_scale"] and r["iterations"] == ref["iterations"]
            assert r["entropy_bits"] == ref["entropy_bits"]
            assert bool(r["converged"]) == ref["converged"]
            assert bool(r["degenerate"]) == ref["degenerate"]
        vol3, _ = oracle.make_phantom(phantoms.cube_3d(48, 7, 71))
        seeds3 = [[30.0, 28.0, 20.0], [10.0, 12.0, 40.0], [23.5, 23.5, 23.5]]
        res3, _ = sx.quadrant_seek(vol3, seeds3, [3, 6, 9], 0, 64, 64, octant=True)
        for r, s in zip(res3, seeds3):
            ref = oracle.ascent_seek_one(vol3, 0, 64, 64, s, [3, 6, 9], dims=3)
            assert np.array_equal(r["position"], ref["position"])
            assert r["best_scale"] == ref["best_scale"] and r["entropy_bits"] == ref["entropy_bits"]
    finally:
        oracle.set_log_mode(0)
    with pytest.raises(ValueError, match="must be 2D"):
        sx.quadrant_seek(np.zeros((4, 8, 8), np.float32), [[2.0, 2.0]], [2], 0, 64, 64)


@pytest.mark.parametrize("method,kw", [
    ("shift", dict(seed_spacing=8.0, scales=[3.0, 5.0], k=6, dedupe_radius=4.0)),
    ("octant", dict(seed_spacing=8.0, scales=[3.0, 4.0, 5.0], k=6, dedupe_radius=4.0)),
])
def test_detect_shard_interleave_equals_detect(sx, oracle, method, kw):
    """each rank's seed share, regathered in plan order and selected
    once, equals the 1-GPU detect byte for byte (ranks run one after another
    here: no rank waits on another)."""
    from paper_1310_6736_b200 import sharding

    vol, _ = oracle.make_phantom(phantoms.ball_3d(24, (12.0, 10.0, 13.0), 5.0, 33))
    sel, seeds, visits = sx.detect_records(vol, method, window_low=0, window_high=64, bins=64,
                                           per_seed=True, **kw)
    for world in (1, 2, 3):
        parts, vis = [], 0
        for r in range(world):
            loc, n_total, v = sx.detect_shard(vol, r, world, method, window_low=0,
                                              window_high=64, bins=64, **kw)
            assert n_total == len(seeds)
            parts.append(loc)
            vis += v
        all_dets = sharding.interleave_detections(parts, n_total)
        assert all_dets.tobytes() == seeds.tobytes()
        got = sx.select(all_dets, 0.9, 0.0, kw["k"], kw["dedupe_radius"])
        assert got.tobytes() == sel.tobytes()
        assert vis == visits


@pytest.mark.parametrize("method", ["shift", "octant"])
def test_batch_device_equals_per_volume_detect(sx, oracle, method):
    """salvox_detect_batch_device: one seek launch over every volume's seeds
    equals detect() volume by volume."""
    import torch

    vols = [oracle.make_phantom(phantoms.ball_3d(20, (8.0 + i, 10.0, 9.0 + 2 * i), 4.0 + i,
                                                 50 + i))[0] for i in range(3)]
    kw = dict(seed_spacing=6.0, scales=[3.0, 4.0], k=5, dedupe_radius=3.0, window_low=0,
              window_high=64, bins=64)
    dv = torch.from_numpy(np.stack(vols)).cuda()
    got, visits = sx.detect_batch_device(dv.data_ptr(), 3, vols[0].shape, method, **kw)
    tot = 0
    for v, g in zip(vols, got):
        ref, _, vis = sx.detect_records(v, method, **kw)
        assert g.tobytes() == ref.tobytes()
        tot += vis
    assert visits == tot


def test_detect_batch_sharded_single_rank_device_path(sx, oracle):
    """sharding.detect_batch_sharded without a process group: the rank's block is
    the whole batch, uploaded and run through one salvox_detect_batch_device."""
    from paper_1310_6736_b200 import sharding

    vols = np.stack([oracle.make_phantom(phantoms.ball_3d(20, (9.0, 10.0 + i, 9.0), 4.0,
                                                          70 + i))[0] for i in range(4)])
    kw = dict(seed_spacing=6.0, scales=[3.0, 4.0], k=5, dedupe_radius=3.0, window_low=0,
              window_high=64, bins=64)
    got, visits = sharding.detect_batch_sharded(vols, method="shift", **kw)
    tot = 0
    for v, g in zip(vols, got):
        ref, _, vis = sx.detect_records(v, "shift", **kw)
        assert g.tobytes() == ref.tobytes()
        tot += vis
    assert visits == tot
