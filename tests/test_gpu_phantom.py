"""make_phantom generated on the device vs the host
generator (itself bit-identical to the reference's phantom.cpp:237-294 and
rng.hpp; pinned by tests/test_oracle_kats.py and the golden fixtures).

Contract: integer (uniform) fills, constant fills, constant backgrounds and the
region centroids are bit-identical; a gaussian background (libdevice
log/sin/cos vs glibc) differs in at most the last float place on a vanishing
fraction of voxels. Error cases raise the host generator's exceptions in the
reference's order.
"""
import numpy as np
import pytest

from tests import phantoms

pytestmark = pytest.mark.gpu


def _both(sx, spec):
    h, hgt = sx.make_phantom(spec)
    d, dgt = sx.make_phantom_device(spec)
    return h, hgt, d.cpu().numpy(), dgt


def _centroids_equal(a, b):
    assert len(a) == len(b)
    for x, y in zip(a, b):
        assert x["center"] == y["center"]
        assert np.array_equal(x["H"], y["H"])


@pytest.mark.parametrize("spec", [
    phantoms.cube_3d(48, 9, 5), phantoms.box_3d(40, 7, 64, 3), phantoms.square_2d(80, 41.0, 37.0, 9, 64, 92),
    phantoms.ellipsoid_3d(phantoms.rot_z(45.0) @ np.diag([9.0, 4.0, 4.0]), 222),
    phantoms.squares_2d(96, [(30, 30), (66, 62)], 8, 7), phantoms.ball_3d(48, [24, 22, 25], 8, 5),
], ids=["cube", "box", "square2d", "ellipsoid", "squares2d", "ball"])
def test_device_phantom_bit_identical(sx, spec):
    h, hgt, d, dgt = _both(sx, spec)
    assert d.tobytes() == h.tobytes()
    _centroids_equal(hgt, dgt)


def test_device_phantom_gaussian_background(sx):
    for spec in (phantoms.config_c1(), phantoms.config_c3(), phantoms.paper_pet()):
        h, hgt, d, dgt = _both(sx, spec)
        _centroids_equal(hgt, dgt)
        diff = d != h
        # region voxels (integer / constant fills) are exact; background within 1 float ulp
        assert diff.mean() < 1e-5, diff.mean()
        if diff.any():
            assert np.all(np.abs(d[diff] - h[diff]) <= np.spacing(np.abs(h[diff])))


def test_device_phantom_c2_full_size(sx):  # the bench volume: 256^3, four regions
    spec = phantoms.config_c2()
    h, hgt, d, dgt = _both(sx, spec)
    _centroids_equal(hgt, dgt)
    diff = d != h
    assert diff.mean() < 1e-5
    # every region voxel (uniform 32 levels) is exact
    for r in spec["regions"]:
        c = [int(round(x)) for x in r["center"]]
        assert d[c[2], c[1], c[0]] == h[c[2], c[1], c[0]]


def test_device_phantom_out_buffer_and_errors(sx):
    import torch

    spec = phantoms.cube_3d(32, 6, 3)
    out = torch.full((32, 32, 32), -1.0, device="cuda")
    got, _ = sx.make_phantom_device(spec, out=out)
    assert got.data_ptr() == out.data_ptr()
    assert np.array_equal(out.cpu().numpy(), sx.make_phantom(spec)[0])
    with pytest.raises(ValueError):
        sx.make_phantom_device(spec, out=torch.empty((2, 2, 2), device="cuda"))
    u = {"type": "uniform", "levels": 8}
    bad = [
        {"dims": [32, 32, 32], "regions": [  # overlap (phantom.cpp:278)
            {"shape": "ball", "center": [10, 10, 10], "radius": 5, "fill": u},
            {"shape": "ball", "center": [14, 10, 10], "radius": 5, "fill": u}]},
        {"dims": [32, 32, 32], "regions": [  # outside (phantom.cpp:255-256)
            {"shape": "ball", "center": [3, 10, 10], "radius": 5, "fill": u}]},
        {"dims": [32, 32, 32], "regions": [  # overlap in region 1 reported before region 2 is outside
            {"shape": "ball", "center": [10, 10, 10], "radius": 5, "fill": u},
            {"shape": "ball", "center": [12, 10, 10], "radius": 4, "fill": u},
            {"shape": "ball", "center": [30, 10, 10], "radius": 5, "fill": u}]},
        {"dims": [32, 32, 32], "regions": [  # no voxel (phantom.cpp:288)
            {"shape": "box", "center": [10.5, 10.5, 10.5], "half_extents": [0.2, 0.2, 0.2], "fill": u}]},
    ]
    for spec in bad:
        with pytest.raises(RuntimeError) as eh:
            sx.make_phantom(spec)
        with pytest.raises(RuntimeError) as ed:
            sx.make_phantom_device(spec)
        assert str(ed.value) == str(eh.value)
