"""TEST INFRASTRUCTURE ONLY -- ctypes view of the C restatement (liboracle.so).

Imported by tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
--impl reference legs, always as the checker or the CPU baseline, never as the
product path. Each wrapper names the reference function it restates
(paths relative to /root/reference/proj).
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB = None

DET_DTYPE = np.dtype(
    [
        ("center", "<f8", (3,)),
        ("H", "<f8", (9,)),
        ("entropy_bits", "<f8"),
        ("pdf_diff", "<f8"),
        ("bhattacharyya", "<f8"),
        ("iterations", "<i4"),
        ("flags", "<u4"),
        ("seed_index", "<i4"),
        ("pad_", "<i4"),
    ]
)
assert DET_DTYPE.itemsize == 136

FLAG_CONVERGED, FLAG_DEGENERATE, FLAG_CLAMPED = 1, 2, 4
KERNELS = {"identity": 0, "epanechnikov": 1, "gaussian": 2}
METHODS = {"quadrant": 0, "shift": 1, "abmsod": 2, "octant": 3}


class OracleError(ValueError):
    """invalid_argument raised by the restated reference function."""


def build():
    subprocess.run(["make", "-s", "-C", _HERE], check=True)


def lib():
    global _LIB
    if _LIB is None:
        path = os.path.join(_HERE, "liboracle.so")
        if not os.path.exists(path):
            build()
        _LIB = C.CDLL(path)
        _declare(_LIB)
    return _LIB


_f32p = np.ctypeslib.ndpointer(np.float32, flags="C_CONTIGUOUS")
_f64p = np.ctypeslib.ndpointer(np.float64, flags="C_CONTIGUOUS")
_i32p = np.ctypeslib.ndpointer(np.int32, flags="C_CONTIGUOUS")
_u64p = np.ctypeslib.ndpointer(np.uint64, flags="C_CONTIGUOUS")
_i64p = np.ctypeslib.ndpointer(np.int64, flags="C_CONTIGUOUS")
_detp = np.ctypeslib.ndpointer(DET_DTYPE, flags="C_CONTIGUOUS")
_vp = C.c_void_p


class _DetectParams(C.Structure):
    _fields_ = [
        ("method", C.c_int),
        ("seed_mode", C.c_int),
        ("seed_spacing", C.c_double),
        ("seed_count", C.c_int),
        ("rng_seed", C.c_uint64),
        ("scales", C.POINTER(C.c_double)),
        ("n_scales", C.c_int),
        ("top_k", C.c_int),
        ("dedupe_radius", C.c_double),
        ("entropy_quantile", C.c_double),
        ("pdf_quantile", C.c_double),
        ("workers", C.c_int),
        ("quadrant_eta", C.c_double),
        ("quadrant_max_iters", C.c_int),
        ("quadrant_scales", C.POINTER(C.c_int)),
        ("n_quadrant_scales", C.c_int),
        ("shift_min_step", C.c_double),
        ("shift_max_iters", C.c_int),
        ("shift_step_kernel", C.c_int),
        ("shift_hist_kernel", C.c_int),
        ("shift_min_inbounds_fraction", C.c_double),
        ("abmsod_threshold", C.c_double),
        ("abmsod_max_iters", C.c_int),
        ("abmsod_kernel", C.c_int),
        ("abmsod_lambda_min", C.c_double),
        ("abmsod_lambda_max", C.c_double),
        ("abmsod_min_inbounds_fraction", C.c_double),
    ]


class _AbmsodParams(C.Structure):
    _fields_ = [
        ("threshold", C.c_double),
        ("max_iterations", C.c_int),
        ("kernel", C.c_int),
        ("lambda_min", C.c_double),
        ("lambda_max", C.c_double),
        ("min_inbounds_fraction", C.c_double),
        ("target", C.c_void_p),
    ]


ABMSOD_ITER_DTYPE = np.dtype([("position", "<f8", (3,)), ("H", "<f8", (9,)),
                              ("bhattacharyya", "<f8"), ("max_bhattacharyya", "<f8"),
                              ("eig_min", "<f8"), ("eig_max", "<f8")])


class _AscentState(C.Structure):
    _fields_ = [
        ("entropy", C.c_double * 8),
        ("best_scale", C.c_int32 * 8),
        ("norm_entropy", C.c_double * 8),
        ("displacement", C.c_double * 3),
        ("degenerate", C.c_int32),
        ("pad_", C.c_int32),
    ]


class _AscentResult(C.Structure):
    _fields_ = [
        ("position", C.c_double * 3),
        ("best_scale", C.c_int32),
        ("iterations", C.c_int32),
        ("entropy_bits", C.c_double),
        ("converged", C.c_int32),
        ("degenerate", C.c_int32),
    ]


def _declare(L):
    L.sxo_rng_next_u64.restype = C.c_uint64
    L.sxo_make_phantom.restype = C.c_int
    L.sxo_make_phantom.argtypes = [C.c_int] * 4 + [C.c_double] * 3 + [
        C.c_int, _i32p, _f64p, _f64p, _f64p, _f64p, _i32p, _i32p, _f64p, C.c_uint64, _f32p,
        _f64p, C.c_char_p, C.c_int]
    L.sxo_bin_of.restype = C.c_int
    L.sxo_bin_of.argtypes = [C.c_double, C.c_double, C.c_int, C.c_double]
    L.sxo_exhaustive.restype = C.c_int
    L.sxo_exhaustive.argtypes = [_f32p, C.c_int, C.c_int, C.c_int, C.c_double, C.c_double, C.c_int,
                                 _f64p, C.c_int, C.c_int, C.c_uint64, C.c_int, C.c_int, C.c_int,
                                 C.c_int, C.c_int, C.c_int, _f32p, _f32p, _u64p, C.c_char_p,
                                 C.c_int]
    L.sxo_voxel_shell_hist.restype = C.c_int
    L.sxo_voxel_shell_hist.argtypes = [_f32p, C.c_int, C.c_int, C.c_int, C.c_double, C.c_double,
                                       C.c_int, C.c_int, C.c_int, C.c_int, C.c_double, _u64p]
    L.sxo_local_maxima.restype = C.c_int64
    L.sxo_local_maxima.argtypes = [_f32p, _f32p, C.c_int, C.c_int, C.c_int, _vp, _vp, _vp, _vp,
                                   C.c_int64]
    L.sxo_plan_seeds.restype = C.c_int64
    L.sxo_plan_seeds.argtypes = [C.c_int, C.c_int, C.c_int, C.c_int, C.c_double, C.c_int, _f64p,
                                 C.c_int, C.c_uint64, _vp, _vp, C.c_int64]
    L.sxo_set_log_mode.argtypes = [C.c_int]
    L.sxo_shift_step.restype = C.c_int
    L.sxo_shift_step.argtypes = [_f32p, C.c_int, C.c_int, C.c_int, C.c_double, C.c_double, C.c_int,
                                 _f64p, _f64p, C.c_int, C.c_int, _vp, _f64p, _u64p]
    L.sxo_saliency_shift.restype = C.c_int
    L.sxo_saliency_shift.argtypes = [_f32p, C.c_int, C.c_int, C.c_int, C.c_double, C.c_double,
                                     C.c_int, _f64p, _f64p, C.c_int, C.c_int, C.c_int, C.c_double,
                                     _vp, C.c_double, _detp, _u64p]
    L.sxo_candidate_histogram.restype = C.c_int
    L.sxo_candidate_histogram.argtypes = [_f32p, C.c_int, C.c_int, C.c_int, C.c_double, C.c_double,
                                          C.c_int, _f64p, _f64p, C.c_int, _f64p, _u64p]
    L.sxo_pdf_difference.restype = C.c_int
    L.sxo_pdf_difference.argtypes = [_f32p, C.c_int, C.c_int, C.c_int, C.c_double, C.c_double,
                                     C.c_int, _f64p, _f64p, C.c_int, _f64p, _u64p]
    L.sxo_entropy_bits.restype = C.c_double
    L.sxo_entropy_bits.argtypes = [_f64p, C.c_int]
    L.sxo_box_entropy_bits.restype = C.c_double
    L.sxo_box_entropy_bits.argtypes = [_f32p, C.c_int, C.c_int, C.c_int, C.c_double, C.c_double,
                                       C.c_int] + [C.c_double] * 6 + [C.c_int, _u64p]
    L.sxo_ascent_step.restype = C.c_int
    L.sxo_ascent_step.argtypes = [_f32p, C.c_int, C.c_int, C.c_int, C.c_double, C.c_double, C.c_int,
                                  C.c_int, _f64p, _i32p, C.c_int, _f64p, C.POINTER(_AscentState),
                                  _u64p]
    L.sxo_ascent_seek_one.restype = C.c_int
    L.sxo_ascent_seek_one.argtypes = [_f32p, C.c_int, C.c_int, C.c_int, C.c_double, C.c_double,
                                      C.c_int, C.c_int, _f64p, _i32p, C.c_int, C.c_double, C.c_int,
                                      C.POINTER(_AscentResult), _u64p]
    L.sxo_detect.restype = C.c_int64
    L.sxo_detect.argtypes = [_f32p, C.c_int, C.c_int, C.c_int, C.c_double, C.c_double, C.c_int,
                             C.POINTER(_DetectParams), _vp, C.c_int64, C.POINTER(C.c_int64), _detp,
                             C.c_int64, _u64p, C.c_char_p, C.c_int]
    L.sxo_select.restype = C.c_int64
    L.sxo_select.argtypes = [_detp, C.c_int64, C.c_double, C.c_double, C.c_int, C.c_double, _detp]
    L.sxo_dedupe_top_k.restype = C.c_int64
    L.sxo_dedupe_top_k.argtypes = [_detp, C.c_int64, C.c_int, C.c_double, _detp]
    L.sxo_eigen_inverse3.argtypes = [_f64p, _f64p]
    L.sxo_eigen_det3.restype = C.c_double
    L.sxo_eigen_det3.argtypes = [_f64p]
    L.sxo_log_portable.restype = C.c_double
    L.sxo_log_portable.argtypes = [C.c_double]
    L.sxo_hu_moments.restype = C.c_int
    L.sxo_hu_moments.argtypes = [_f32p, C.c_int, C.c_int, C.c_int, _f64p]
    L.sxo_hu_template_distance.restype = C.c_double
    L.sxo_hu_template_distance.argtypes = [_f32p, C.c_int, C.c_int, C.c_int, _f64p, _f64p, _f32p,
                                           C.c_int, C.c_int, C.c_int]
    L.sxo_rasterize_window.restype = C.c_int64
    L.sxo_rasterize_window.argtypes = [C.c_int, C.c_int, C.c_int, _f64p, _f64p, _vp, C.c_int64]
    L.sxo_exp_portable.restype = C.c_double
    L.sxo_exp_portable.argtypes = [C.c_double]
    L.sxo_pow_portable.restype = C.c_double
    L.sxo_pow_portable.argtypes = [C.c_double, C.c_double]
    L.sxo_bandwidth_from_moment.restype = C.c_int
    L.sxo_bandwidth_from_moment.argtypes = [_f64p, C.c_double, C.c_int, C.c_double, C.c_double,
                                            _f64p]
    L.sxo_sym_eigen3.restype = C.c_int
    L.sxo_sym_eigen3.argtypes = [_f64p, _f64p, _f64p]
    L.sxo_abmsod_run.restype = C.c_int
    L.sxo_abmsod_run.argtypes = [_f32p, C.c_int, C.c_int, C.c_int, C.c_double, C.c_double, C.c_int,
                                 _f64p, _f64p, C.POINTER(_AbmsodParams), _detp, _vp, C.c_int,
                                 C.POINTER(C.c_int), _u64p]


def _vol(v):
    v = np.ascontiguousarray(v, dtype=np.float32)
    if v.ndim == 2:
        v = v[None]
    nz, ny, nx = v.shape
    return v, nx, ny, nz


# ---------------------------------------------------------------- phantom.cpp
SHAPES = {"box": 0, "ball": 1, "ellipsoid": 2}


def make_phantom(spec):
    """phantom.cpp:364-421. spec mirrors PhantomSpec JSON (phantom.cpp:226-277)."""
    nx, ny, nz = (int(d) for d in spec["dims"])
    bg = spec.get("background", {"type": "constant", "value": 0.0})
    regions = spec.get("regions", [])
    n = len(regions)
    shape = np.zeros(max(n, 1), np.int32)
    center = np.zeros(3 * max(n, 1))
    half = np.zeros(3 * max(n, 1))
    radius = np.zeros(max(n, 1))
    axes = np.tile(np.eye(3).ravel(), max(n, 1)).astype(np.float64)
    ftype = np.zeros(max(n, 1), np.int32)
    flev = np.full(max(n, 1), 64, np.int32)
    fval = np.zeros(max(n, 1))
    for i, r in enumerate(regions):
        shape[i] = SHAPES[r["shape"]]
        center[3 * i:3 * i + 3] = r["center"]
        if r["shape"] == "box":
            half[3 * i:3 * i + 3] = r["half_extents"]
        elif r["shape"] == "ball":
            radius[i] = r["radius"]
        else:
            axes[9 * i:9 * i + 9] = np.asarray(r["axes"], np.float64).ravel()
        f = r.get("fill", {"type": "uniform", "levels": 64})
        ftype[i] = 0 if f["type"] == "uniform" else 1
        flev[i] = int(f.get("levels", 64))
        fval[i] = float(f.get("value", 0.0))
    out = np.zeros((nz, ny, nx), np.float32)
    cent = np.zeros(3 * max(n, 1))
    err = C.create_string_buffer(256)
    rc = lib().sxo_make_phantom(
        nx, ny, nz, 0 if bg["type"] == "constant" else 1, float(bg.get("value", 0.0)),
        float(bg.get("mean", 0.0)), float(bg.get("sigma", 1.0)), n, shape, center, half, radius,
        axes, ftype, flev, fval, int(spec.get("rng_seed", 0)), out, cent, err, 256)
    if rc != 0:
        raise RuntimeError(err.value.decode())
    return out, cent[: 3 * n].reshape(n, 3)


def bin_of(low, high, bins, intensity):
    return lib().sxo_bin_of(low, high, bins, intensity)


# ------------------------------------------------------------- pipeline.cpp exhaustive
def exhaustive(vol, low, high, bins, scales, kernel="identity", budget=2_000_000, mode="literal",
               threads=1, z_range=None, y_range=None):
    """pipeline.cpp:63-141. Returns (score, best_scale, visits) as (nz,ny,nx) float32."""
    v, nx, ny, nz = _vol(vol)
    sc = np.ascontiguousarray(scales, np.float64)
    score = np.zeros(v.shape, np.float32)
    best = np.zeros(v.shape, np.float32)
    visits = np.zeros(1, np.uint64)
    err = C.create_string_buffer(256)
    z0, z1 = z_range if z_range is not None else (0, nz)
    y0, y1 = y_range if y_range is not None else (0, ny)
    rc = lib().sxo_exhaustive(v, nx, ny, nz, low, high, bins, sc, len(sc), KERNELS[kernel],
                              int(budget), 0 if mode == "literal" else 1, int(threads), int(z0),
                              int(z1), int(y0), int(y1), score, best, visits, err, 256)
    if rc != 0:
        raise OracleError(err.value.decode())
    return score, best, int(visits[0])


def voxel_shell_hist(vol, low, high, bins, x, y, z, radius):
    v, nx, ny, nz = _vol(vol)
    S = np.zeros(bins, np.uint64)
    lib().sxo_voxel_shell_hist(v, nx, ny, nz, low, high, bins, x, y, z, radius, S)
    return S


def local_maxima(score, best_scale):
    """pipeline.cpp:143-165 -> list of (position(3), score, scale, linear index)."""
    s, nx, ny, nz = _vol(score)
    b, _, _, _ = _vol(best_scale)
    n = lib().sxo_local_maxima(s, b, nx, ny, nz, None, None, None, None, 0)
    pos = np.zeros((max(n, 1), 3))
    sc = np.zeros(max(n, 1))
    scale = np.zeros(max(n, 1))
    lin = np.zeros(max(n, 1), np.int64)
    lib().sxo_local_maxima(s, b, nx, ny, nz, pos.ctypes.data, sc.ctypes.data, scale.ctypes.data,
                           lin.ctypes.data, n)
    return pos[:n], sc[:n], scale[:n], lin[:n]


def plan_seeds(shape_zyx, mode="lattice", spacing=16.0, count=0, scales=(8.0,), rng_seed=0):
    """seeds.cpp:7-45 -> (positions (n,3), scales (n,))."""
    nz, ny, nx = shape_zyx
    sc = np.ascontiguousarray(scales, np.float64)
    m = 0 if mode == "lattice" else 1
    n = lib().sxo_plan_seeds(nx, ny, nz, m, spacing, count, sc, len(sc), rng_seed, None, None, 0)
    if n < 0:
        raise OracleError("seed plan: invalid")
    pos = np.zeros((n, 3))
    ss = np.zeros(n)
    lib().sxo_plan_seeds(nx, ny, nz, m, spacing, count, sc, len(sc), rng_seed, pos.ctypes.data,
                         ss.ctypes.data, n)
    return pos, ss


def set_log_mode(mode):
    """0: glibc log (reference); 1: sx_log, the shared host/device log."""
    lib().sxo_set_log_mode(int(mode))


def shift_step(vol, low, high, bins, x, half, step_kernel="identity", hist_kernel="identity",
               target=None):
    v, nx, ny, nz = _vol(vol)
    out = np.zeros(3)
    visits = np.zeros(1, np.uint64)
    t = None if target is None else np.ascontiguousarray(target, np.float64)
    ok = lib().sxo_shift_step(v, nx, ny, nz, low, high, bins, np.asarray(x, np.float64),
                              np.asarray(half, np.float64), KERNELS[step_kernel],
                              KERNELS[hist_kernel], None if t is None else t.ctypes.data, out,
                              visits)
    return (out if ok else None), int(visits[0])


def saliency_shift(vol, low, high, bins, seed, half, step_kernel="identity",
                   hist_kernel="identity", max_iters=50, min_step=0.1, target=None,
                   min_inbounds_fraction=0.1):
    v, nx, ny, nz = _vol(vol)
    det = np.zeros(1, DET_DTYPE)
    visits = np.zeros(1, np.uint64)
    t = None if target is None else np.ascontiguousarray(target, np.float64)
    rc = lib().sxo_saliency_shift(v, nx, ny, nz, low, high, bins, np.asarray(seed, np.float64),
                                  np.asarray(half, np.float64), KERNELS[step_kernel],
                                  KERNELS[hist_kernel], max_iters, min_step,
                                  None if t is None else t.ctypes.data, min_inbounds_fraction, det,
                                  visits)
    if rc != 0:
        raise OracleError("shift: invalid params")
    return det[0], int(visits[0])


def candidate_histogram(vol, low, high, bins, center, H, kernel="identity"):
    v, nx, ny, nz = _vol(vol)
    p = np.zeros(bins)
    visits = np.zeros(1, np.uint64)
    ok = lib().sxo_candidate_histogram(v, nx, ny, nz, low, high, bins,
                                       np.asarray(center, np.float64),
                                       np.ascontiguousarray(H, np.float64).ravel(),
                                       KERNELS[kernel], p, visits)
    return p if ok else None


def pdf_difference(vol, low, high, bins, center, H, kernel="identity"):
    v, nx, ny, nz = _vol(vol)
    out = np.zeros(1)
    visits = np.zeros(1, np.uint64)
    ok = lib().sxo_pdf_difference(v, nx, ny, nz, low, high, bins, np.asarray(center, np.float64),
                                  np.ascontiguousarray(H, np.float64).ravel(), KERNELS[kernel], out,
                                  visits)
    if not ok:
        raise OracleError("pdf_difference: degenerate")
    return float(out[0])


def entropy_bits(p):
    p = np.ascontiguousarray(p, np.float64)
    return lib().sxo_entropy_bits(p, len(p))


def box_entropy_bits(vol, low, high, bins, x0, x1, y0, y1, z0=0.0, z1=0.0, min_voxels=4):
    v, nx, ny, nz = _vol(vol)
    visits = np.zeros(1, np.uint64)
    return lib().sxo_box_entropy_bits(v, nx, ny, nz, low, high, bins, x0, x1, y0, y1, z0, z1,
                                      min_voxels, visits)


def ascent_step(vol, low, high, bins, p, scales, dims=2):
    v, nx, ny, nz = _vol(vol)
    st = _AscentState()
    moved = np.zeros(3)
    visits = np.zeros(1, np.uint64)
    pp = np.zeros(3)
    pp[: len(p)] = p
    rc = lib().sxo_ascent_step(v, nx, ny, nz, low, high, bins, dims, pp,
                               np.ascontiguousarray(scales, np.int32), len(scales), moved,
                               C.byref(st), visits)
    if rc != 0:
        raise OracleError("quadrant_step: volume must be 2D (nz == 1)")
    nq = 4 if dims == 2 else 8
    return moved, {
        "entropy": np.array(st.entropy[:nq]),
        "best_scale": np.array(st.best_scale[:nq]),
        "norm_entropy": np.array(st.norm_entropy[:nq]),
        "displacement": np.array(st.displacement[:]),
        "degenerate": bool(st.degenerate),
    }


def ascent_seek_one(vol, low, high, bins, seed, scales, dims=2, eta=0.5, max_iters=50):
    v, nx, ny, nz = _vol(vol)
    r = _AscentResult()
    visits = np.zeros(1, np.uint64)
    pp = np.zeros(3)
    pp[: len(seed)] = seed
    rc = lib().sxo_ascent_seek_one(v, nx, ny, nz, low, high, bins, dims, pp,
                                   np.ascontiguousarray(scales, np.int32), len(scales), eta,
                                   max_iters, C.byref(r), visits)
    if rc != 0:
        raise OracleError("quadrant: invalid")
    return {
        "position": np.array(r.position[:]),
        "best_scale": r.best_scale,
        "iterations": r.iterations,
        "entropy_bits": r.entropy_bits,
        "converged": bool(r.converged),
        "degenerate": bool(r.degenerate),
    }


def detect(vol, low, high, bins, method="shift", seed_mode="lattice", seed_spacing=16.0,
           seed_count=400, scales=(8.0,), rng_seed=0, top_k=20, dedupe_radius=5.0,
           entropy_quantile=0.9, pdf_quantile=0.0, workers=1, quadrant_eta=0.5,
           quadrant_max_iters=50, quadrant_scales=None, shift_min_step=0.1, shift_max_iters=50,
           shift_step_kernel="identity", shift_hist_kernel="identity",
           min_inbounds_fraction=0.1, abmsod_threshold=1e-4, abmsod_max_iters=15,
           abmsod_kernel="gaussian", lambda_min=4.0, lambda_max=0.0):
    """pipeline.cpp:311-402 -> (selected detections, per-seed detections, visits)."""
    v, nx, ny, nz = _vol(vol)
    sc = (C.c_double * len(scales))(*scales)
    P = _DetectParams()
    P.method = METHODS[method]
    P.seed_mode = 0 if seed_mode == "lattice" else 1
    P.seed_spacing = seed_spacing
    P.seed_count = seed_count
    P.rng_seed = rng_seed
    P.scales = sc
    P.n_scales = len(scales)
    P.top_k = top_k
    P.dedupe_radius = dedupe_radius
    P.entropy_quantile = entropy_quantile
    P.pdf_quantile = pdf_quantile
    P.workers = workers
    P.quadrant_eta = quadrant_eta
    P.quadrant_max_iters = quadrant_max_iters
    qs = None
    if quadrant_scales is not None:
        qs = (C.c_int * len(quadrant_scales))(*quadrant_scales)
        P.quadrant_scales = qs
        P.n_quadrant_scales = len(quadrant_scales)
    P.shift_min_step = shift_min_step
    P.shift_max_iters = shift_max_iters
    P.shift_step_kernel = KERNELS[shift_step_kernel]
    P.shift_hist_kernel = KERNELS[shift_hist_kernel]
    P.shift_min_inbounds_fraction = min_inbounds_fraction
    P.abmsod_threshold = abmsod_threshold
    P.abmsod_max_iters = abmsod_max_iters
    P.abmsod_kernel = KERNELS[abmsod_kernel]
    P.abmsod_lambda_min = lambda_min
    P.abmsod_lambda_max = lambda_max
    P.abmsod_min_inbounds_fraction = min_inbounds_fraction
    ns = plan_seeds((nz, ny, nx), seed_mode, seed_spacing, seed_count, scales, rng_seed)[0].shape[0]
    per_seed = np.zeros(max(ns, 1), DET_DTYPE)
    out = np.zeros(max(ns, 1), DET_DTYPE)
    n_seed = C.c_int64(0)
    visits = np.zeros(1, np.uint64)
    err = C.create_string_buffer(256)
    k = lib().sxo_detect(v, nx, ny, nz, low, high, bins, C.byref(P), per_seed.ctypes.data, ns,
                         C.byref(n_seed), out, ns, visits, err, 256)
    if k < 0:
        raise OracleError(err.value.decode())
    return out[:k].copy(), per_seed[: n_seed.value].copy(), int(visits[0])


def abmsod_run(vol, low, high, bins, seed, H=None, radius=None, threshold=1e-4, max_iterations=15,
               kernel="gaussian", lambda_min=4.0, lambda_max=0.0, min_inbounds_fraction=0.1,
               target=None, trace=False):
    """abmsod.cpp:43-169 -> (detection record, trace records or None, visits). The seed
    window is H (3x3) or EllipsoidWindow::isotropic(seed, radius) (window.hpp:46-48)."""
    v, nx, ny, nz = _vol(vol)
    if H is None:
        r2 = float(radius) ** 2
        H = np.diag([r2, r2, 1.0 if nz == 1 else r2])
    P = _AbmsodParams(threshold, max_iterations, KERNELS[kernel], lambda_min, lambda_max,
                      min_inbounds_fraction, None)
    t = None
    if target is not None:
        t = np.ascontiguousarray(target, np.float64)
        P.target = t.ctypes.data
    det = np.zeros(1, DET_DTYPE)
    cap = max_iterations if trace else 0
    tr = np.zeros(max(cap, 1), ABMSOD_ITER_DTYPE)
    nt = C.c_int(0)
    visits = np.zeros(1, np.uint64)
    s = np.zeros(3)
    s[: len(seed)] = seed
    rc = lib().sxo_abmsod_run(v, nx, ny, nz, low, high, bins, s,
                              np.ascontiguousarray(np.asarray(H, np.float64).reshape(9)),
                              C.byref(P), det, tr.ctypes.data if trace else None, cap,
                              C.byref(nt), visits)
    if rc == -1:
        raise OracleError("abmsod: invalid params")
    if rc == -2:
        raise OracleError("abmsod: eigen decomposition failed")
    return det[0], (tr[: nt.value].copy() if trace else None), int(visits[0])


def bandwidth_from_moment(outer, wsum, dim, lambda_min, lambda_max):
    H = np.zeros(9)
    rc = lib().sxo_bandwidth_from_moment(np.ascontiguousarray(outer, np.float64).reshape(9),
                                         float(wsum), int(dim), float(lambda_min),
                                         float(lambda_max), H)
    if rc in (1, 2):
        raise OracleError("bandwidth update: " + ("zero weight mass" if rc == 1 else
                                                   "non-finite moment"))
    if rc == 3:
        raise OracleError("abmsod: eigen decomposition failed")
    return H.reshape(3, 3)


def sym_eigen3(a):
    """SelfAdjointEigenSolver<Matrix3d> restatement -> (ascending values, vectors as columns)."""
    vals, vecs = np.zeros(3), np.zeros(9)
    if lib().sxo_sym_eigen3(np.ascontiguousarray(a, np.float64).reshape(9), vals, vecs) != 0:
        raise OracleError("abmsod: eigen decomposition failed")
    return vals, vecs.reshape(3, 3)


def hu_moments(img):
    a = np.ascontiguousarray(img, np.float32)
    if a.ndim == 3:
        a = a[0]
    out = np.zeros(7)
    if lib().sxo_hu_moments(a, a.shape[1], a.shape[0], a.shape[1], out) != 0:
        raise OracleError("hu_moments: zero total mass")
    return out


def hu_template_distance(vol, center, H, tmpl, slices=5):
    v, nx, ny, nz = _vol(vol)
    t = np.ascontiguousarray(tmpl, np.float32)
    if t.ndim == 3:
        t = t[0]
    return lib().sxo_hu_template_distance(v, nx, ny, nz, np.ascontiguousarray(center, np.float64),
                                          np.ascontiguousarray(np.asarray(H, np.float64).reshape(9)),
                                          t, t.shape[1], t.shape[0], int(slices))


def rasterize_window(shape_zyx, center, H):
    nz, ny, nx = shape_zyx
    c = np.ascontiguousarray(center, np.float64)
    h = np.ascontiguousarray(np.asarray(H, np.float64).reshape(9))
    n = lib().sxo_rasterize_window(nx, ny, nz, c, h, None, 0)
    out = np.zeros(max(n, 1), np.uint64)
    lib().sxo_rasterize_window(nx, ny, nz, c, h, out.ctypes.data, n)
    return out[:n]


def exp_portable(x):
    return lib().sxo_exp_portable(float(x))


def pow_portable(x, y):
    return lib().sxo_pow_portable(float(x), float(y))


def select(dets, q_entropy=0.9, q_pdf=0.0, k=20, radius=5.0):
    d = np.ascontiguousarray(dets, DET_DTYPE)
    out = np.zeros(max(len(d), 1), DET_DTYPE)
    n = lib().sxo_select(d, len(d), q_entropy, q_pdf, k, radius, out)
    return out[:n].copy()


def dedupe_top_k(dets, k, radius):
    d = np.ascontiguousarray(dets, DET_DTYPE)
    out = np.zeros(max(len(d), 1), DET_DTYPE)
    n = lib().sxo_dedupe_top_k(d, len(d), k, radius, out)
    return out[:n].copy()


def eigen_inverse3(m):
    out = np.zeros(9)
    lib().sxo_eigen_inverse3(np.ascontiguousarray(m, np.float64).ravel(), out)
    return out.reshape(3, 3)


def log_portable(x):
    return lib().sxo_log_portable(float(x))
