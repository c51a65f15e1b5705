"""Phantom specs of the reference's own tests (PhantomSpec dicts, phantom.cpp:226-277).

Each helper cites the reference test it reproduces (paths relative to
/root/reference/proj/tests).
"""
import math

import numpy as np


def square_2d(dim, cx, cy, half, levels, seed):  # test_seek.cpp:19-31
    return {"dims": [dim, dim, 1],
            "regions": [{"shape": "box", "center": [cx, cy, 0.0], "half_extents": [half, half, 0.0],
                         "fill": {"type": "uniform", "levels": levels}}],
            "rng_seed": seed}


def squares_2d(dim, centers, half, seed):  # test_pipeline.cpp:210-224
    return {"dims": [dim, dim, 1],
            "regions": [{"shape": "box", "center": [cx, cy, 0.0], "half_extents": [half, half, 0.0],
                         "fill": {"type": "uniform", "levels": 64}} for cx, cy in centers],
            "rng_seed": seed}


def cube_3d(dim, half, seed):  # test_seek.cpp:220-232
    c = (dim - 1) / 2.0
    return {"dims": [dim, dim, dim],
            "regions": [{"shape": "box", "center": [c, c, c], "half_extents": [half, half, half],
                         "fill": {"type": "uniform", "levels": 64}}],
            "rng_seed": seed}


def box_3d(dim, half, levels, seed):  # test_entropy.cpp:143-155
    c = (dim - 1) / 2.0
    return {"dims": [dim, dim, dim],
            "regions": [{"shape": "box", "center": [c, c, c], "half_extents": [half, half, half],
                         "fill": {"type": "uniform", "levels": levels}}],
            "rng_seed": seed}


def ball_3d(dim, center, radius, seed, levels=64, background=None):  # test_pipeline.cpp:296-306
    spec = {"dims": [dim, dim, dim],
            "regions": [{"shape": "ball", "center": list(center), "radius": radius,
                         "fill": {"type": "uniform", "levels": levels}}],
            "rng_seed": seed}
    if background is not None:
        spec["background"] = background
    return spec


def symmetric_square_2d():  # test_seek.cpp:117-125 (noise-free, radially symmetric)
    v = np.zeros((1, 96, 96), np.float32)
    c = 47.0
    for y in range(96):
        for x in range(96):
            if abs(x - c) <= 12 and abs(y - c) <= 12:
                dx, dy = int(abs(x - c)), int(abs(y - c))
                v[0, y, x] = float((dx * dx + dy * dy) % 64)
    return v, c


def symmetric_cube_3d(dim=64, half=14):  # test_seek.cpp:300-311
    c = (dim - 1) / 2.0
    z, y, x = np.meshgrid(np.arange(dim), np.arange(dim), np.arange(dim), indexing="ij")
    dx, dy, dz = x - c, y - c, z - c
    inside = (np.abs(dx) <= half) & (np.abs(dy) <= half) & (np.abs(dz) <= half)
    v = np.where(inside, (dx * dx + dy * dy + dz * dz).astype(np.int64) % 64, 0).astype(np.float32)
    return v, c


def symmetric_cube_octant(dim=48, half=10):
    """Noise-free cube whose intensity depends only on |x-c|,|y-c|,|z-c| (integer c):
    the octant analogue of the quadrant balance fixture."""
    c = (dim - 1) // 2
    z, y, x = np.meshgrid(np.arange(dim), np.arange(dim), np.arange(dim), indexing="ij")
    ax, ay, az = np.abs(x - c), np.abs(y - c), np.abs(z - c)
    inside = (ax <= half) & (ay <= half) & (az <= half)
    v = np.where(inside, (ax * ax + ay * ay + az * az) % 64, 0).astype(np.float32)
    return v, float(c)


# ---- BASELINE.json configs ----
def config_c1(seed=1310, jitter=None):
    c = [70.0, 58.0, 64.0]
    if jitter is not None:
        c = [c[i] + jitter[i] for i in range(3)]
    return {"dims": [128, 128, 128],
            "background": {"type": "gaussian", "mean": 4.0, "sigma": 1.5},
            "regions": [{"shape": "ball", "center": c, "radius": 12.0,
                         "fill": {"type": "uniform", "levels": 16}}],
            "rng_seed": seed}


def config_c2():
    u = {"type": "uniform", "levels": 32}
    return {"dims": [256, 256, 256],
            "background": {"type": "gaussian", "mean": 8.0, "sigma": 2.0},
            "regions": [
                {"shape": "ball", "center": [64.0, 64.0, 64.0], "radius": 8.0, "fill": u},
                {"shape": "ball", "center": [180.0, 90.0, 128.0], "radius": 12.0, "fill": u},
                {"shape": "ball", "center": [120.0, 190.0, 200.0], "radius": 15.0, "fill": u},
                {"shape": "box", "center": [200.0, 200.0, 60.0], "half_extents": [10.0, 10.0, 10.0],
                 "fill": u}],
            "rng_seed": 6736}


def config_c3():
    a = math.radians(30.0)
    rz = np.array([[math.cos(a), -math.sin(a), 0.0], [math.sin(a), math.cos(a), 0.0],
                   [0.0, 0.0, 1.0]])
    axes = rz @ np.diag([20.0, 12.0, 10.0])
    return {"dims": [256, 256, 160],
            "background": {"type": "gaussian", "mean": 24.0, "sigma": 4.0},
            "regions": [
                {"shape": "ellipsoid", "center": [150.0, 110.0, 80.0], "axes": axes.tolist(),
                 "fill": {"type": "uniform", "levels": 64}},
                {"shape": "ball", "center": [60.0, 60.0, 40.0], "radius": 8.0,
                 "fill": {"type": "constant", "value": 60.0}}],
            "rng_seed": 176}


def rot_z(degrees):  # test_seek.cpp:483-488
    a = math.radians(degrees)
    return np.array([[math.cos(a), -math.sin(a), 0.0], [math.sin(a), math.cos(a), 0.0],
                     [0.0, 0.0, 1.0]])


def ellipsoid_3d(axes, seed, dim=64):  # test_seek.cpp:468-481 (ellipsoid_phantom)
    c = (dim - 1) / 2.0
    return {"dims": [dim, dim, dim],
            "regions": [{"shape": "ellipsoid", "center": [c, c, c],
                         "axes": np.asarray(axes, np.float64).tolist(),
                         "fill": {"type": "uniform", "levels": 64}}],
            "rng_seed": seed}


def ellipsoid_H(axes):  # RegionSpec ellipsoid H = A A^T (phantom.cpp:198-222)
    a = np.asarray(axes, np.float64)
    return a @ a.T


def paper_pet():
    """The paper's PET case shape (128x128x34, 400 seeds): C1-style
    background with a high-entropy ball (the LV analogue)."""
    return {"dims": [128, 128, 34],
            "background": {"type": "gaussian", "mean": 4.0, "sigma": 1.5},
            "regions": [{"shape": "ball", "center": [70.0, 58.0, 17.0], "radius": 10.0,
                         "fill": {"type": "uniform", "levels": 16}}],
            "rng_seed": 264}


def paper_mr():
    """The paper's MR case shape (256x256x176, 700 seeds): the C3
    tumour phantom on 176 planes."""
    spec = config_c3()
    spec["dims"] = [256, 256, 176]
    spec["rng_seed"] = 290
    return spec


def config_c4():
    """C4: 512^3, the C2 generator with centres x2 plus four more regions,
    rng_seed 512."""
    u = {"type": "uniform", "levels": 32}
    regs = [{"shape": r["shape"], "center": [2.0 * c for c in r["center"]], "fill": u,
             **({"radius": 2.0 * r["radius"]} if "radius" in r else
                {"half_extents": [2.0 * h for h in r["half_extents"]]})}
            for r in config_c2()["regions"]]
    regs += [{"shape": "ball", "center": [100.0, 400.0, 300.0], "radius": 14.0, "fill": u},
             {"shape": "ball", "center": [420.0, 120.0, 420.0], "radius": 10.0, "fill": u},
             {"shape": "box", "center": [300.0, 300.0, 100.0], "half_extents": [12.0, 8.0, 10.0],
              "fill": u},
             {"shape": "ball", "center": [60.0, 60.0, 460.0], "radius": 15.0, "fill": u}]
    return {"dims": [512, 512, 512],
            "background": {"type": "gaussian", "mean": 8.0, "sigma": 2.0},
            "regions": regs, "rng_seed": 512}
