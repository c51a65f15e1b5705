"""Host-side data formats either side of the hot path (no GPU needed): the
product's make_phantom / plan_seeds (C++ in libsalvox_b200) reproduce the
oracle's restatement of phantom.cpp / seeds.cpp bit for bit."""
import numpy as np
import pytest

from tests import phantoms

SPECS = [
    phantoms.square_2d(64, 31.0, 31.0, 8, 64, 77),
    phantoms.ball_3d(48, (24.0, 24.0, 24.0), 8.0, 404,
                     background={"type": "gaussian", "mean": 8.0, "sigma": 2.0}),
    phantoms.cube_3d(40, 6, 5),
]


@pytest.mark.parametrize("spec", SPECS)
def test_make_phantom_bit_identical(sx, oracle, spec):
    a, gt = sx.make_phantom(spec)
    b, cent = oracle.make_phantom(spec)
    assert a.tobytes() == b.tobytes()
    assert np.array_equal(np.array([g["center"] for g in gt]), cent)


def test_make_phantom_c3_ellipsoid_matches(sx, oracle):
    spec = phantoms.config_c3()
    spec["dims"] = [128, 128, 96]  # same generator, smaller grid
    spec["regions"][0]["center"] = [70.0, 60.0, 48.0]
    spec["regions"][1]["center"] = [20.0, 20.0, 20.0]
    a, _ = sx.make_phantom(spec)
    b, _ = oracle.make_phantom(spec)
    assert a.tobytes() == b.tobytes()


def test_make_phantom_errors(sx):
    with pytest.raises(RuntimeError, match="outside the volume"):
        sx.make_phantom({"dims": [16, 16, 16], "regions": [
            {"shape": "ball", "center": [2.0, 8.0, 8.0], "radius": 5.0}]})
    with pytest.raises(RuntimeError, match="overlap"):
        sx.make_phantom({"dims": [32, 32, 32], "regions": [
            {"shape": "ball", "center": [16.0, 16.0, 16.0], "radius": 5.0},
            {"shape": "ball", "center": [18.0, 16.0, 16.0], "radius": 5.0}]})


@pytest.mark.parametrize("args", [
    ((64, 64, 64), "lattice", 16.0, 0, [8.0], 0),
    ((1, 96, 96), "lattice", 12.0, 0, [6.0, 10.0], 0),
    ((160, 256, 256), "lattice", 16.0, 0, [8.0, 12.0], 0),
    ((48, 48, 48), "random", 16.0, 37, [5.0], 9),
    ((1, 64, 64), "random", 16.0, 11, [4.0, 6.0], 3),
])
def test_plan_seeds_identical(sx, oracle, args):
    shape, mode, spacing, count, scales, seed = args
    a, sa = sx.plan_seeds(shape, mode, spacing, count, scales, seed)
    b, sb = oracle.plan_seeds(shape, mode, spacing, count, scales, seed)
    assert np.array_equal(a, b) and np.array_equal(sa, sb)


def test_plan_seeds_validation(sx):
    with pytest.raises(ValueError, match="spacing must be > 0"):
        sx.plan_seeds((8, 8, 8), "lattice", 0.0)
    with pytest.raises(ValueError, match="count must be >= 1"):
        sx.plan_seeds((8, 8, 8), "random", 16.0, 0)
    with pytest.raises(ValueError, match="scales must be > 0"):
        sx.plan_seeds((8, 8, 8), "lattice", 4.0, 0, [0.0])
