"""Randomised GPU-vs-oracle parity: random shapes (incl. 2D and thin slabs),
intensity distributions, windows, bin counts, scales, seed plans and methods.
Every case must be bit-exact against the oracle in the device's math mode
(per-seed trajectories, scores, selection, visits) -- the same contract as the
fixed-case suites, over inputs nobody hand-picked (seeded, reproducible)."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _case(rng):
    two_d = rng.random() < 0.25
    nz = 1 if two_d else int(rng.integers(6, 28))
    ny, nx = int(rng.integers(10, 40)), int(rng.integers(10, 40))
    kind = rng.integers(0, 3)
    if kind == 0:
        vol = rng.normal(20.0, 6.0, size=(nz, ny, nx))
    elif kind == 1:
        vol = rng.integers(0, 64, size=(nz, ny, nx)).astype(np.float64)
    else:  # blobs on a ramp
        z, y, x = np.meshgrid(np.arange(nz), np.arange(ny), np.arange(nx), indexing="ij")
        vol = 0.5 * x + 10.0 * np.exp(-((x - nx / 2) ** 2 + (y - ny / 3) ** 2 + (z - nz / 2) ** 2) / 20.0)
    vol = vol.astype(np.float32)
    bins = int(rng.choice([8, 16, 31, 32, 48, 64]))
    return vol, two_d, bins


@pytest.mark.parametrize("seed", range(48))
def test_fuzz_detect_all_methods(sx, oracle, seed):
    rng = np.random.default_rng(1000 + seed)
    vol, two_d, bins = _case(rng)
    methods = ["shift", "abmsod"] + (["quadrant"] if two_d else ["octant"])
    method = methods[seed % len(methods)]
    lo, hi = float(np.floor(vol.min())), float(np.ceil(vol.max()) + 1.0)
    scales = sorted({float(s) for s in rng.integers(2, 7, size=int(rng.integers(1, 4)))})
    kw = dict(seed_spacing=float(rng.integers(4, 9)), scales=scales, k=int(rng.integers(3, 9)),
              dedupe_radius=float(rng.uniform(2.0, 6.0)))
    extra = {}
    if method == "shift":
        extra = dict(shift_hist_kernel=str(rng.choice(["identity", "epanechnikov", "gaussian"])),
                     shift_step_kernel=str(rng.choice(["identity", "gaussian"])),
                     shift_max_iters=int(rng.integers(1, 30)))
    if rng.random() < 0.3:
        extra.update(seed_mode="random", seed_count=int(rng.integers(5, 40)),
                     rng_seed=int(rng.integers(0, 1000)))
    sel, seeds, visits = sx.detect_records(vol, method, window_low=lo, window_high=hi, bins=bins,
                                           per_seed=True, **kw, **extra)
    okw = dict(kw)
    okw["top_k"] = okw.pop("k")
    # the device's math: sx_log + sx_exp everywhere; window scale() via glibc pow
    # on the host for the fixed shift/ascent geometries, via sx_pow on the device
    # for ABMSOD's evolving bandwidth
    oracle.set_log_mode(7 if method == "abmsod" else 3)
    try:
        rsel, rseeds, rv = oracle.detect(vol, lo, hi, bins, method=method, **okw, **extra)
    finally:
        oracle.set_log_mode(0)
    assert seeds.tobytes() == rseeds.tobytes(), method
    assert sel.tobytes() == rsel.tobytes(), method
    assert visits == rv


@pytest.mark.parametrize("seed", range(16))
def test_fuzz_exhaustive(sx, oracle, seed):
    rng = np.random.default_rng(2000 + seed)
    vol, two_d, bins = _case(rng)
    bins = min(bins, 64)
    smax = int(rng.integers(3, 9))
    scales = [float(s) for s in range(int(rng.integers(2, smax)), smax + 1)]
    lo, hi = float(np.floor(vol.min())), float(np.ceil(vol.max()) + 1.0)
    score, best, maxima, visits = sx.kadir_brady_exhaustive_records(vol, scales, lo, hi, bins,
                                                                    budget=10**12)
    rs, rb, rv = oracle.exhaustive(vol, lo, hi, bins, scales, budget=10**12, mode="exact",
                                   threads=8)
    excess = np.abs(score.astype(np.float64) - rs) - (1e-5 * np.maximum(np.abs(score), np.abs(rs))
                                                      + 1e-6)
    assert excess.max() <= 0.0
    assert (best == rb).mean() > 0.99
    assert visits == rv
    assert np.array_equal(maxima["linear_index"], oracle.local_maxima(score, best)[3])
