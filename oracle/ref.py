"""TEST INFRASTRUCTURE ONLY -- ctypes view of the REFERENCE's own C++.

oracle/_ref/libsalvox_ref.so is the reference's sources
(/root/reference/proj/src/*.cpp, compiled where they lie by `make -C oracle
ref`) plus the C-ABI glue oracle/ref_shim.cpp. Only tests/, smoke() and
bench.py's reference arm use it, always as the checker or the timed
reference, never as the product. The .so is prebuilt here and travels to the
GPU box; /root/reference itself is never read at run time.

Wrappers mirror oracle/oracle.py (same argument names, same record dtypes) so a
test can run one case through the restatement, the reference and the device.
"""
from __future__ import annotations

import ctypes as C
import json
import os

import numpy as np

from oracle.oracle import (ABMSOD_ITER_DTYPE, DET_DTYPE, KERNELS, METHODS, OracleError,
                           _AbmsodParams, _AscentResult, _AscentState, _DetectParams, _vol)

_HERE = os.path.dirname(os.path.abspath(__file__))
PATH = os.path.join(_HERE, "_ref", "libsalvox_ref.so")
_LIB = None


class ReferenceError_(ValueError):
    """std::invalid_argument (code 1) or another std::exception (code 2) from the reference."""


def available():
    return os.path.exists(PATH)


def lib():
    global _LIB
    if _LIB is None:
        if not available():
            raise FileNotFoundError(f"{PATH} not built (make -C oracle ref, needs /root/reference)")
        _LIB = C.CDLL(PATH)
        _LIB.sxr_entropy_bits.restype = C.c_double
        _LIB.sxr_box_entropy_bits.restype = C.c_double
        _LIB.sxr_dedupe_top_k.restype = C.c_int64
        _LIB.sxr_rasterize_window.restype = C.c_int64
        _LIB.sxr_hu_template_distance.restype = C.c_double
        _LIB.sxr_fnv1a64.restype = C.c_uint64
        for name in ("sxr_exhaustive", "sxr_plan_seeds", "sxr_saliency_shift", "sxr_detect",
                     "sxr_abmsod_run", "sxr_make_phantom", "sxr_load_volume"):
            getattr(_LIB, name).restype = C.c_int
    return _LIB


def _p(a):
    return a.ctypes.data_as(C.c_void_p)


def _check(rc, err):
    if rc == 1:
        raise OracleError(err.value.decode())
    if rc != 0:
        raise ReferenceError_(err.value.decode())


def _err():
    return C.create_string_buffer(512)


def make_phantom(spec):
    """phantom.cpp:99-150 + :237-294 from the PhantomSpec JSON -> (volume zyx, centres)."""
    text = json.dumps(spec).encode()
    dims = np.zeros(3, np.int32)
    cent = np.zeros(3 * 64)
    err = _err()
    _check(lib().sxr_make_phantom(text, None, 0, _p(dims), _p(cent), 64, err, 512), err)
    nx, ny, nz = (int(d) for d in dims)
    out = np.zeros((nz, ny, nx), np.float32)
    _check(lib().sxr_make_phantom(text, _p(out), out.size, _p(dims), _p(cent), 64, err, 512), err)
    n = len(spec.get("regions", []))
    return out, cent[: 3 * n].reshape(n, 3)


def bin_of(low, high, bins, intensity):
    return lib().sxr_bin_of(C.c_double(low), C.c_double(high), int(bins), C.c_double(intensity))


def entropy_bits(p):
    a = np.ascontiguousarray(p, np.float64)
    return lib().sxr_entropy_bits(_p(a), len(a))


def exhaustive(vol, low, high, bins, scales, kernel="identity", budget=2_000_000):
    """pipeline.cpp:63-166 -> (score, best_scale, maxima (n,5): x y z score scale, visits)."""
    v, nx, ny, nz = _vol(vol)
    sc = np.ascontiguousarray(scales, np.float64)
    score = np.zeros(v.shape, np.float32)
    best = np.zeros(v.shape, np.float32)
    cap = v.size
    maxima = np.zeros((max(cap, 1), 5))
    n = C.c_int64(0)
    visits = C.c_uint64(0)
    err = _err()
    _check(lib().sxr_exhaustive(_p(v), nx, ny, nz, C.c_double(low), C.c_double(high), bins,
                                _p(sc), len(sc), KERNELS[kernel], C.c_uint64(int(budget)),
                                _p(score), _p(best), _p(maxima), C.c_int64(cap), C.byref(n),
                                C.byref(visits), err, 512), err)
    return score, best, maxima[: n.value].copy(), int(visits.value)


def plan_seeds(shape_zyx, mode="lattice", spacing=16.0, count=0, scales=(8.0,), rng_seed=0):
    nz, ny, nx = shape_zyx
    sc = np.ascontiguousarray(scales, np.float64)
    n = C.c_int64(0)
    err = _err()
    args = (nx, ny, nz, 0 if mode == "lattice" else 1, C.c_double(spacing), int(count), _p(sc),
            len(sc), C.c_uint64(rng_seed))
    _check(lib().sxr_plan_seeds(*args, None, None, C.c_int64(0), C.byref(n), err, 512), err)
    pos = np.zeros((max(n.value, 1), 3))
    ss = np.zeros(max(n.value, 1))
    _check(lib().sxr_plan_seeds(*args, _p(pos), _p(ss), C.c_int64(n.value), C.byref(n), err, 512),
           err)
    return pos[: n.value], ss[: n.value]


def saliency_shift(vol, low, high, bins, seed, half, step_kernel="identity",
                   hist_kernel="identity", max_iters=50, min_step=0.1, target=None,
                   min_inbounds_fraction=0.1):
    """shift.cpp:36-107 -> (detection record, visits)."""
    v, nx, ny, nz = _vol(vol)
    s = np.ascontiguousarray(seed, np.float64)
    h = np.ascontiguousarray(half, np.float64)
    t = None if target is None else np.ascontiguousarray(target, np.float64)
    out = np.zeros(1, DET_DTYPE)
    visits = C.c_uint64(0)
    err = _err()
    _check(lib().sxr_saliency_shift(_p(v), nx, ny, nz, C.c_double(low), C.c_double(high), bins,
                                    _p(s), _p(h), KERNELS[step_kernel], KERNELS[hist_kernel],
                                    int(max_iters), C.c_double(min_step),
                                    None if t is None else _p(t),
                                    C.c_double(min_inbounds_fraction), _p(out), C.byref(visits),
                                    err, 512), err)
    return out[0], int(visits.value)


def shift_step(vol, low, high, bins, x, half, step_kernel="identity", hist_kernel="identity",
               target=None):
    """shift.cpp:15-34 -> (new position or None, visits)."""
    v, nx, ny, nz = _vol(vol)
    xx = np.ascontiguousarray(x, np.float64)
    h = np.ascontiguousarray(half, np.float64)
    t = None if target is None else np.ascontiguousarray(target, np.float64)
    out = np.zeros(3)
    visits = C.c_uint64(0)
    rc = lib().sxr_shift_step(_p(v), nx, ny, nz, C.c_double(low), C.c_double(high), bins, _p(xx),
                              _p(h), KERNELS[step_kernel], KERNELS[hist_kernel],
                              None if t is None else _p(t), _p(out), C.byref(visits))
    if rc < 0:
        raise ReferenceError_("shift_step failed")
    return (out if rc == 1 else None), int(visits.value)


def candidate_histogram(vol, low, high, bins, center, H, kernel="identity"):
    v, nx, ny, nz = _vol(vol)
    c = np.ascontiguousarray(center, np.float64)
    h = np.ascontiguousarray(np.asarray(H, np.float64).reshape(9))
    p = np.zeros(bins)
    visits = C.c_uint64(0)
    rc = lib().sxr_candidate_histogram(_p(v), nx, ny, nz, C.c_double(low), C.c_double(high), bins,
                                       _p(c), _p(h), KERNELS[kernel], _p(p), C.byref(visits))
    if rc < 0:
        raise ReferenceError_("candidate_histogram failed")
    return (p if rc == 1 else None), int(visits.value)


def pdf_difference(vol, low, high, bins, center, H, kernel="identity"):
    v, nx, ny, nz = _vol(vol)
    c = np.ascontiguousarray(center, np.float64)
    h = np.ascontiguousarray(np.asarray(H, np.float64).reshape(9))
    out = C.c_double(0.0)
    visits = C.c_uint64(0)
    err = _err()
    _check(lib().sxr_pdf_difference(_p(v), nx, ny, nz, C.c_double(low), C.c_double(high), bins,
                                    _p(c), _p(h), KERNELS[kernel], C.byref(out), C.byref(visits),
                                    err, 512), err)
    return out.value, int(visits.value)


def box_entropy_bits(vol, low, high, bins, x0, x1, y0, y1, min_pixels=4):
    v, nx, ny, nz = _vol(vol)
    visits = C.c_uint64(0)
    e = lib().sxr_box_entropy_bits(_p(v), nx, ny, nz, C.c_double(low), C.c_double(high), bins,
                                   C.c_double(x0), C.c_double(x1), C.c_double(y0), C.c_double(y1),
                                   int(min_pixels), C.byref(visits))
    return e, int(visits.value)


def quadrant_step(vol, low, high, bins, p, scales):
    """quadrant.cpp:37-81 -> (moved (2,), state, visits)."""
    v, nx, ny, nz = _vol(vol)
    pp = np.ascontiguousarray(p[:2], np.float64)
    sc = np.ascontiguousarray(scales, np.int32)
    moved = np.zeros(2)
    st = _AscentState()
    visits = C.c_uint64(0)
    err = _err()
    _check(lib().sxr_quadrant_step(_p(v), nx, ny, nz, C.c_double(low), C.c_double(high), bins,
                                   _p(pp), _p(sc), len(sc), _p(moved), C.byref(st),
                                   C.byref(visits), err, 512), err)
    return moved, st, int(visits.value)


def quadrant_seek_one(vol, low, high, bins, seed, scales, eta=0.5, max_iters=50):
    """quadrant.cpp:83-114 -> (result struct, visits)."""
    v, nx, ny, nz = _vol(vol)
    s = np.ascontiguousarray(seed[:2], np.float64)
    sc = np.ascontiguousarray(scales, np.int32)
    out = _AscentResult()
    visits = C.c_uint64(0)
    err = _err()
    _check(lib().sxr_quadrant_seek_one(_p(v), nx, ny, nz, C.c_double(low), C.c_double(high), bins,
                                       _p(s), _p(sc), len(sc), C.c_double(eta), int(max_iters),
                                       C.byref(out), C.byref(visits), err, 512), err)
    return out, int(visits.value)


def detect(vol, low, high, bins, method="shift", seed_mode="lattice", seed_spacing=16.0,
           seed_count=400, scales=(8.0,), rng_seed=0, top_k=20, dedupe_radius=5.0,
           entropy_quantile=0.9, pdf_quantile=0.0, workers=1, quadrant_eta=0.5,
           quadrant_max_iters=50, quadrant_scales=None, shift_min_step=0.1, shift_max_iters=50,
           shift_step_kernel="identity", shift_hist_kernel="identity",
           min_inbounds_fraction=0.1, abmsod_threshold=1e-4, abmsod_max_iters=15,
           abmsod_kernel="gaussian", lambda_min=4.0, lambda_max=0.0):
    """pipeline.cpp:311-402, the reference's own detect() -> (selected detections, visits)."""
    if method == "octant":
        raise OracleError("octant ascent does not exist in the reference (SURVEY 0.4)")
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
    cap = max(top_k, 1)
    out = np.zeros(cap, DET_DTYPE)
    n = C.c_int64(0)
    visits = C.c_uint64(0)
    err = _err()
    _check(lib().sxr_detect(_p(v), nx, ny, nz, C.c_double(low), C.c_double(high), bins,
                            C.byref(P), _p(out), C.c_int64(cap), C.byref(n), C.byref(visits),
                            err, 512), err)
    return out[: min(n.value, cap)].copy(), int(visits.value)


def abmsod_run(vol, low, high, bins, seed, H=None, radius=None, threshold=1e-4, max_iterations=15,
               kernel="gaussian", lambda_min=4.0, lambda_max=0.0, min_inbounds_fraction=0.1,
               target=None, trace=False):
    """abmsod.cpp:43-169 -> (detection record, trace records or None, visits)."""
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
    visits = C.c_uint64(0)
    s = np.zeros(3)
    s[: len(seed)] = seed
    h = np.ascontiguousarray(np.asarray(H, np.float64).reshape(9))
    err = _err()
    _check(lib().sxr_abmsod_run(_p(v), nx, ny, nz, C.c_double(low), C.c_double(high), bins, _p(s),
                                _p(h), C.byref(P), _p(det), _p(tr) if trace else None, cap,
                                C.byref(nt), C.byref(visits), err, 512), err)
    return det[0], (tr[: nt.value].copy() if trace else None), int(visits.value)


def bandwidth_from_moment(outer, wsum, dim, lambda_min, lambda_max):
    H = np.zeros(9)
    o = np.ascontiguousarray(outer, np.float64).reshape(9)
    err = _err()
    _check(lib().sxr_bandwidth_from_moment(_p(o), C.c_double(wsum), int(dim),
                                           C.c_double(lambda_min), C.c_double(lambda_max), _p(H),
                                           err, 512), err)
    return H.reshape(3, 3)


def dedupe_top_k(dets, k, radius):
    d = np.ascontiguousarray(dets, DET_DTYPE)
    out = np.zeros(max(len(d), 1), DET_DTYPE)
    n = lib().sxr_dedupe_top_k(_p(d), C.c_int64(len(d)), int(k), C.c_double(radius), _p(out))
    return out[:n].copy()


def rasterize_window(shape_zyx, center, H):
    nz, ny, nx = shape_zyx
    c = np.ascontiguousarray(center, np.float64)
    h = np.ascontiguousarray(np.asarray(H, np.float64).reshape(9))
    n = lib().sxr_rasterize_window(nx, ny, nz, _p(c), _p(h), None, C.c_int64(0))
    out = np.zeros(max(n, 1), np.uint64)
    lib().sxr_rasterize_window(nx, ny, nz, _p(c), _p(h), _p(out), C.c_int64(n))
    return out[:n]


def hu_moments(img):
    a = np.ascontiguousarray(img, np.float32)
    if a.ndim == 3:
        a = np.ascontiguousarray(a[0])
    out = np.zeros(7)
    err = _err()
    _check(lib().sxr_hu_moments(_p(a), a.shape[1], a.shape[0], _p(out), err, 512), err)
    return out


def hu_template_distance(vol, center, H, tmpl, slices=5):
    v, nx, ny, nz = _vol(vol)
    t = np.ascontiguousarray(tmpl, np.float32)
    if t.ndim == 3:
        t = np.ascontiguousarray(t[0])
    c = np.ascontiguousarray(center, np.float64)
    h = np.ascontiguousarray(np.asarray(H, np.float64).reshape(9))
    return lib().sxr_hu_template_distance(_p(v), nx, ny, nz, _p(c), _p(h), _p(t), t.shape[1],
                                          t.shape[0], int(slices))


def rasterize_windows(shape_zyx, centers, Hs):
    """rasterize_window over many windows on ONE frame -> per-window support counts."""
    nz, ny, nx = shape_zyx
    c = np.ascontiguousarray(centers, np.float64).reshape(-1, 3)
    h = np.ascontiguousarray(np.asarray(Hs, np.float64).reshape(-1, 9))
    counts = np.zeros(max(len(c), 1), np.int64)
    lib().sxr_rasterize_windows.restype = C.c_int64
    lib().sxr_rasterize_windows(nx, ny, nz, _p(c), _p(h), C.c_int64(len(c)), _p(counts))
    return counts[: len(c)]


def hu_template_distances(vol, centers, Hs, tmpl, slices=5):
    """hu_template_distance for many detections with ONE Volume built."""
    v, nx, ny, nz = _vol(vol)
    t = np.ascontiguousarray(tmpl, np.float32)
    c = np.ascontiguousarray(centers, np.float64).reshape(-1, 3)
    h = np.ascontiguousarray(np.asarray(Hs, np.float64).reshape(-1, 9))
    out = np.zeros(max(len(c), 1))
    lib().sxr_hu_template_distances(_p(v), nx, ny, nz, _p(c), _p(h), C.c_int64(len(c)), _p(t),
                                    t.shape[1], t.shape[0], int(slices), _p(out))
    return out[: len(c)]


def load_volume(mhd_path):
    """meta_io.cpp:37-117 -> (volume zyx float32, spacing (3,))."""
    dims = np.zeros(3, np.int32)
    sp = np.zeros(3)
    err = _err()
    path = os.fsencode(mhd_path)
    _check(lib().sxr_load_volume(path, None, C.c_int64(0), _p(dims), _p(sp), err, 512), err)
    nx, ny, nz = (int(d) for d in dims)
    out = np.zeros((nz, ny, nx), np.float32)
    _check(lib().sxr_load_volume(path, _p(out), C.c_int64(out.size), _p(dims), _p(sp), err, 512),
           err)
    return out, sp


def save_volume(vol, mhd_path):
    v, nx, ny, nz = _vol(vol)
    err = _err()
    _check(lib().sxr_save_volume(_p(v), nx, ny, nz, os.fsencode(mhd_path), err, 512), err)


def _text_call(fn, *args):
    n = C.c_int64(0)
    err = _err()
    _check(fn(*args, None, C.c_int64(0), C.byref(n), err, 512), err)
    buf = C.create_string_buffer(n.value + 1)
    _check(fn(*args, buf, C.c_int64(n.value + 1), C.byref(n), err, 512), err)
    return buf.value.decode()


def config_roundtrip(config):
    """config.cpp RunConfig::from_json_text(...).to_json_text()."""
    text = config if isinstance(config, str) else json.dumps(config)
    return _text_call(lib().sxr_config_roundtrip, text.encode())


def detection_report_json(config, vol, dets, wall_time_ms=0.0):
    """report.cpp:28-60."""
    text = config if isinstance(config, str) else json.dumps(config)
    v, nx, ny, nz = _vol(vol)
    d = np.ascontiguousarray(dets, DET_DTYPE)
    return _text_call(lib().sxr_detection_report_json, text.encode(), _p(v), nx, ny, nz, _p(d),
                      C.c_int64(len(d)), C.c_double(wall_time_ms))


def fnv1a64(data):
    b = bytes(data)
    return int(lib().sxr_fnv1a64(b, C.c_size_t(len(b))))
