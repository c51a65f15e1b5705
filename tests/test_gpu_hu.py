"""Hu moments on the device vs the oracle restatement of
src/hu.cpp and pipeline.cpp:218-271, plus the reference's own Hu tests
(tests/test_pipeline.cpp:149-206, :440-474)."""
import math

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _disk(n, c, r, val=1.0):
    y, x = np.mgrid[0:n, 0:n]
    return np.where((x - c) ** 2 + (y - c) ** 2 <= r * r, val, 0.0).astype(np.float32)


def test_hu_disk_matches_bruteforce_and_oracle(sx, oracle):  # test_pipeline.cpp:172-206
    img = _disk(64, 31.5, 14.0)
    got = sx.hu_moments(img)
    ys, xs = np.mgrid[0:64, 0:64]
    m00 = img.sum(dtype=np.float64)
    cx, cy = (img * xs).sum() / m00, (img * ys).sum() / m00
    mu = lambda p, q: (img * (xs - cx) ** p * (ys - cy) ** q).sum(dtype=np.float64)  # noqa: E731
    eta = lambda p, q: mu(p, q) / m00 ** (1.0 + (p + q) / 2.0)  # noqa: E731
    e20, e02, e11 = eta(2, 0), eta(0, 2), eta(1, 1)
    assert abs(got[0] - (e20 + e02)) < 1e-9
    assert abs(got[1] - ((e20 - e02) ** 2 + 4 * e11 * e11)) < 1e-9
    assert np.all(np.abs(got[2:]) < 1e-9)
    with pytest.raises(ValueError, match="zero total mass"):
        sx.hu_moments(np.zeros((8, 8), np.float32))
    rng = np.random.default_rng(31)
    img2 = np.zeros((96, 96), np.float32)
    img2[24:72, 24:72] = rng.uniform(0, 64, size=(48, 48))
    oracle.set_log_mode(4)  # pow(m00, 2.5) via the shared sx_pow, like the device
    try:
        ref = oracle.hu_moments(img2)
    finally:
        oracle.set_log_mode(0)
    assert np.array_equal(sx.hu_moments(img2), ref)
    glibc = oracle.hu_moments(img2)
    assert np.allclose(sx.hu_moments(img2), glibc, rtol=1e-12, atol=0)


def test_hu_invariances(sx):  # test_pipeline.cpp:149-170
    rng = np.random.default_rng(31)
    img = np.zeros((96, 96), np.float32)
    img[24:72, 24:72] = rng.uniform(0, 64, size=(48, 48))
    base = sx.hu_moments(img)
    shifted = sx.hu_moments(np.roll(np.roll(img, 3, axis=0), 5, axis=1))
    assert np.all(np.abs(shifted - base) < 1e-9)
    rotated = sx.hu_moments(np.rot90(img).copy())
    assert np.all(np.abs(rotated - base) <= 1e-6 * np.maximum(1e-12, np.abs(base)))
    up = np.kron(img, np.ones((2, 2), np.float32))
    scaled = sx.hu_moments(up)
    assert np.all(np.abs(scaled - base) <= 1e-3 * np.maximum(np.maximum(np.abs(base), np.abs(scaled)), 1e-12))


def test_hu_filter_picks_the_disk_like_region(sx, oracle):  # test_pipeline.cpp:440-474
    spec = {"dims": [96, 96, 32],
            "regions": [{"shape": "ball", "center": [28.0, 48.0, 16.0], "radius": 10.0,
                         "fill": {"type": "constant", "value": 40.0}},
                        {"shape": "box", "center": [68.0, 48.0, 16.0], "half_extents": [12.0, 5.0, 10.0],
                         "fill": {"type": "constant", "value": 40.0}}],
            "rng_seed": 1}
    vol, _ = sx.make_phantom(spec)
    on_ball = {"center": (28.0, 48.0, 16.0), "H": np.diag([144.0, 144.0, 144.0])}
    on_box = {"center": (68.0, 48.0, 16.0), "H": np.diag([196.0, 49.0, 144.0])}
    tmpl = _disk(32, 15.5, 10.0, 40.0)
    assert sx.hu_filter([on_ball, on_box], vol, tmpl) == 0
    assert sx.hu_filter([on_box, on_ball], vol, tmpl) == 1
    assert sx.hu_filter([on_box], vol, tmpl) == 0
    with pytest.raises(ValueError):
        sx.hu_filter([], vol, tmpl)
    d = sx.hu_template_distance([on_ball, on_box], vol, tmpl)
    for det, got in zip([on_ball, on_box], d):
        ref = oracle.hu_template_distance(vol, det["center"], det["H"], tmpl)
        assert math.isclose(got, ref, rel_tol=1e-9)
