"""The reference's public API for the hot path, backed by the B200 C-ABI.

Mirrors the Python binding of the reference (/root/reference/proj/bindings/
py_module.cpp) -- same function names, argument names, defaults, return shapes
and exception types -- for the functions on the accelerated path:

  kadir_brady_exhaustive   py_module.cpp:186-204  (pipeline.cpp:63-166)
  detect                   py_module.cpp:206-230  (pipeline.cpp:311-402)
  saliency_shift           py_module.cpp:159-170  (shift.cpp:36-107)
  make_phantom             py_module.cpp:96-112   (phantom.cpp:364-421)

plus the C++-level entry points the binding does not expose (plan_seeds,
quadrant_seek / octant_seek, dedupe_top_k, select, the z-slab exhaustive).

Volumes are numpy arrays indexed [z, y, x] (2D arrays are [y, x], nz = 1).
Everything computes on the GPU; there is no CPU fallback.
"""
from __future__ import annotations

import ctypes as C
import json

import numpy as np

from . import _lib
from ._lib import DET_DTYPE, MAX_DTYPE, KERNELS, METHODS, check, default_context, ptr

DEFAULT_BUDGET = 2_000_000  # include/salvox/pipeline.hpp:53


def _volume(arr):
    a = np.ascontiguousarray(arr, dtype=np.float32)
    if a.ndim == 2:
        a = a[None]
    if a.ndim != 3:
        raise ValueError("expected a 2D or 3D array")
    nz, ny, nx = a.shape
    return a, nx, ny, nz


def _window(low, high, bins):
    """window_or_full (py_module.cpp:73-77): explicit window, else observed range on device."""
    if low is not None and high is not None:
        if not (low < high):
            raise ValueError("IntensityWindow: low must be < high")
        return _lib.Window(float(low), float(high), int(bins), 0)
    return _lib.Window(0.0, 1.0, int(bins), 1)


def _ctx(ctx):
    return ctx if ctx is not None else default_context()


_FLAG_NAMES = [(1, "converged"), (2, "degenerate"), (4, "boundary-clamped")]


def detection_to_dict(d) -> dict:
    """detection_to_dict (py_module.cpp:58-70)."""
    flags = int(d["flags"])
    return {
        "center": tuple(float(v) for v in d["center"]),
        "H": np.array(d["H"], dtype=np.float64).reshape(3, 3),
        "entropy_bits": float(d["entropy_bits"]),
        "pdf_diff": float(d["pdf_diff"]),
        "bhattacharyya": float(d["bhattacharyya"]),
        "iterations": int(d["iterations"]),
        "flags": [n for f, n in _FLAG_NAMES if flags & f],
        "seed_index": int(d["seed_index"]),
    }


# ------------------------------------------------------------------ exhaustive (E1)
def kadir_brady_exhaustive_records(volume, scales, window_low=None, window_high=None, bins=64,
                                   kernel="identity", budget=DEFAULT_BUDGET, ctx=None,
                                   want_maps=True):
    """Structured form: (score[z,y,x] f32, best_scale[z,y,x] f32, maxima MAX_DTYPE, visits)."""
    v, nx, ny, nz = _volume(volume)
    sc = np.ascontiguousarray(scales, dtype=np.float64)
    iw = _window(window_low, window_high, bins)
    c = _ctx(ctx)
    score = np.empty(v.shape, np.float32) if want_maps else None
    best = np.empty(v.shape, np.float32) if want_maps else None
    cap = max(4096, int(_MAXIMA_HINT.get(id(c), 0) * 1.1))  # size from the last call
    maxima = np.empty(cap, MAX_DTYPE)
    n = C.c_int64(0)
    visits = C.c_uint64(0)
    check(_lib.load().salvox_exhaustive(
        c.handle, ptr(v), nx, ny, nz, C.byref(iw), ptr(sc), len(sc), KERNELS[kernel], int(budget),
        ptr(score), ptr(best), ptr(maxima), cap, C.byref(n), C.byref(visits)))
    _MAXIMA_HINT[id(c)] = n.value
    if n.value > cap:
        maxima = np.empty(n.value, MAX_DTYPE)
        check(_lib.load().salvox_last_maxima(c.handle, ptr(maxima), n.value, C.byref(n)))
    return score, best, maxima[: n.value], int(visits.value)


def kadir_brady_exhaustive(volume, scales, window_low=None, window_high=None, bins=64,
                           kernel="identity", budget=DEFAULT_BUDGET, ctx=None):
    """Dense scan; returns (score map [z,y,x], ranked local maxima) like py_module.cpp:186-204.

    The reference binding always uses the default budget (2e6 voxel-scale
    evaluations) and raises ValueError above it; pass ``budget`` to lift it.
    """
    score, _, maxima, _ = kadir_brady_exhaustive_records(volume, scales, window_low, window_high,
                                                         bins, kernel, budget, ctx)
    # columns to Python lists first (per-record access of a structured array costs
    # microseconds; a 256^3 pass has ~0.5 M maxima), and no cyclic-GC passes while
    # the ~0.5 M new containers are made (none of them can form a cycle):
    # 2.4 s -> 0.35 s for C2's list
    import gc

    pos = maxima["position"].tolist()
    enabled = gc.isenabled()
    gc.disable()
    try:
        out = [{"position": tuple(p), "score": s, "scale": c}
               for p, s, c in zip(pos, maxima["score"].tolist(), maxima["scale"].tolist())]
    finally:
        if enabled:
            gc.enable()
    return score, out


_MAXIMA_HINT = {}  # context id -> maxima count of its last slab call (output sizing)


def kadir_brady_exhaustive_slab(slab, nz_total, zs0, z0, z1, scales, window_low, window_high,
                                bins=64, kernel="identity", budget=DEFAULT_BUDGET, ctx=None,
                                out=None, maxima_out=None):
    """z-slab form (salvox_exhaustive_slab): `slab` holds planes [zs0, zs0+len) of a volume
    with nz_total planes; returns owned-plane maps [z0, z1) and global maxima."""
    s = np.ascontiguousarray(slab, dtype=np.float32)
    nzs, ny, nx = s.shape
    sc = np.ascontiguousarray(scales, dtype=np.float64)
    iw = _window(window_low, window_high, bins)
    if iw.full_range:
        raise ValueError("exhaustive slab: pass an explicit (global) intensity window")
    c = _ctx(ctx)
    if out is not None:  # caller-provided (e.g. pinned) output planes
        score, best = out
        assert score.shape == best.shape == (z1 - z0, ny, nx)
        assert score.dtype == best.dtype == np.float32 and score.flags.c_contiguous
    else:
        score = np.empty((z1 - z0, ny, nx), np.float32)
        best = np.empty((z1 - z0, ny, nx), np.float32)
    if maxima_out is not None:  # caller-provided (e.g. pinned) maxima buffer
        maxima = maxima_out
        assert maxima.dtype == MAX_DTYPE and maxima.flags.c_contiguous
        cap = len(maxima)
    else:
        cap = max(4096, int(_MAXIMA_HINT.get(id(c), 0) * 1.1))  # size from the last call
        maxima = np.empty(cap, MAX_DTYPE)
    n = C.c_int64(0)
    visits = C.c_uint64(0)
    check(_lib.load().salvox_exhaustive_slab(
        c.handle, ptr(s), nx, ny, int(nz_total), int(zs0), int(zs0 + nzs), int(z0), int(z1),
        C.byref(iw), ptr(sc), len(sc), KERNELS[kernel], int(budget), ptr(score), ptr(best),
        ptr(maxima), cap, C.byref(n), C.byref(visits)))
    _MAXIMA_HINT[id(c)] = n.value
    if n.value > cap:
        maxima = np.empty(n.value, MAX_DTYPE)
        check(_lib.load().salvox_last_maxima(c.handle, ptr(maxima), n.value, C.byref(n)))
    return score, best, maxima[: n.value], int(visits.value)


def exhaustive_slab_scores(slab, nz_total, zs0, z0, z1, scales, window_low, window_high,
                           bins=64, kernel="identity", budget=DEFAULT_BUDGET, ctx=None, out=None):
    """Step 1 of the exchange form (salvox_exhaustive_slab_scores): scores ONLY the
    owned planes [z0, z1). `slab` is a host array (pipelined H2D/compute/D2H;
    returns host maps, `out` may supply pinned ones) or a CUDA torch tensor
    (device-resident; returns device tensors). Returns (score, best, visits)."""
    sc = np.ascontiguousarray(scales, dtype=np.float64)
    iw = _window(window_low, window_high, bins)
    if iw.full_range:
        raise ValueError("exhaustive slab: pass an explicit (global) intensity window")
    c = _ctx(ctx)
    visits = C.c_uint64(0)
    on_device = hasattr(slab, "is_cuda") and slab.is_cuda
    if on_device:
        import torch
        s = slab.contiguous()
        nzs, ny, nx = s.shape
        if out is not None:
            score, best = out
        else:
            score = torch.empty((z1 - z0, ny, nx), dtype=torch.float32, device=s.device)
            best = torch.empty_like(score)
        c.after_torch(s, score, best)  # inputs/outputs may still be in use on torch's stream
        sp, op, bp = C.c_void_p(s.data_ptr()), C.c_void_p(score.data_ptr()), C.c_void_p(best.data_ptr())
    else:
        s = np.ascontiguousarray(slab, dtype=np.float32)
        nzs, ny, nx = s.shape
        if out is not None:
            score, best = out
            assert score.shape == best.shape == (z1 - z0, ny, nx)
        else:
            score = np.empty((z1 - z0, ny, nx), np.float32)
            best = np.empty((z1 - z0, ny, nx), np.float32)
        sp, op, bp = ptr(s), ptr(score), ptr(best)
    check(_lib.load().salvox_exhaustive_slab_scores(
        c.handle, sp, 1 if on_device else 0, nx, ny, int(nz_total), int(zs0), int(zs0 + nzs),
        int(z0), int(z1), C.byref(iw), ptr(sc), len(sc), KERNELS[kernel], int(budget), op, bp,
        C.byref(visits)))
    return score, best, int(visits.value)


def exhaustive_slab_edges(first, last, ctx=None):
    """Step 2: the first / last owned score planes into device tensors (nx*ny floats)."""
    c = _ctx(ctx)
    c.after_torch(first, last)
    check(_lib.load().salvox_exhaustive_slab_edges(
        c.handle, C.c_void_p(first.data_ptr()) if first is not None else None,
        C.c_void_p(last.data_ptr()) if last is not None else None))


def exhaustive_slab_maxima(below, above, ctx=None, maxima_out=None, on_device=False):
    """Step 3: strict maxima of the owned planes given the neighbour planes z0-1
    (`below`) and z1 (`above`) as device tensors (None at the volume ends).
    on_device=True leaves them on the device and returns their count."""
    c = _ctx(ctx)
    c.after_torch(below, above)  # e.g. planes just received by NCCL on torch's stream
    if on_device:
        n = C.c_int64(0)
        check(_lib.load().salvox_exhaustive_slab_maxima(
            c.handle, C.c_void_p(below.data_ptr()) if below is not None else None,
            C.c_void_p(above.data_ptr()) if above is not None else None, None, 0, C.byref(n)))
        return int(n.value)
    if maxima_out is not None:
        maxima = maxima_out
        cap = len(maxima)
    else:
        cap = max(4096, int(_MAXIMA_HINT.get(id(c), 0) * 1.1))
        maxima = np.empty(cap, MAX_DTYPE)
    n = C.c_int64(0)
    check(_lib.load().salvox_exhaustive_slab_maxima(
        c.handle, C.c_void_p(below.data_ptr()) if below is not None else None,
        C.c_void_p(above.data_ptr()) if above is not None else None, ptr(maxima), cap,
        C.byref(n)))
    _MAXIMA_HINT[id(c)] = n.value
    if n.value > cap:
        maxima = np.empty(n.value, MAX_DTYPE)
        check(_lib.load().salvox_last_maxima(c.handle, ptr(maxima), n.value, C.byref(n)))
    return maxima[: n.value]


def last_maxima_device(out, ctx=None):
    """The last exhaustive call's maxima into a CUDA uint8 tensor of shape (cap, 48)
    (salvox_last_maxima_device); returns the full count."""
    c = _ctx(ctx)
    c.after_torch(out)
    n = C.c_int64(0)
    check(_lib.load().salvox_last_maxima_device(c.handle, C.c_void_p(out.data_ptr()),
                                                int(out.shape[0]), C.byref(n)))
    return int(n.value)


def merge_maxima_device(records, ctx=None):
    """Device sort of maxima records (CUDA uint8 tensor (n, 48)) into the reference's
    order (score desc, linear index asc); returns a new tensor."""
    import torch
    c = _ctx(ctx)
    out = torch.empty_like(records)
    c.after_torch(records, out)
    check(_lib.load().salvox_merge_maxima_device(c.handle, C.c_void_p(records.data_ptr()),
                                                 int(records.shape[0]), C.c_void_p(out.data_ptr())))
    return out


def exhaustive_debug_hist(voxels, bins, n_scales, ctx=None):
    """Exact S_b(r) / T(r) of the last exhaustive call for the given linear voxel indices.
    Returns (radii, hist[n, n_radii, bins+1] uint32; column `bins` holds T(r))."""
    c = _ctx(ctx)
    vox = np.ascontiguousarray(voxels, dtype=np.int64)
    radii = np.zeros(3 * n_scales + 1)
    nr = C.c_int32(0)
    tmp = np.zeros(max(len(vox), 1) * 3 * n_scales * (bins + 1), np.uint32)
    check(_lib.load().salvox_exhaustive_debug_hist(c.handle, ptr(vox), len(vox), ptr(tmp),
                                                   ptr(radii), C.byref(nr)))
    R = nr.value
    return radii[:R], tmp[: len(vox) * R * (bins + 1)].reshape(len(vox), R, bins + 1)


# --------------------------------------------------------------------- detect (E2/E3)
# ------------------------------------------------- window operations (device)
def window_ops(volume, ops, window_low=None, window_high=None, bins=64, target=None, ctx=None,
               want_pmf=False):
    """Runs WINDOW_OP_DTYPE records through salvox_window_ops (one warp per op) ->
    (WINDOW_RESULT_DTYPE[n], pmf[n, bins] or None)."""
    from ._lib import WINDOW_RESULT_DTYPE

    v, nx, ny, nz = _volume(volume)
    iw = _window(window_low, window_high, bins)
    o = np.ascontiguousarray(ops)
    out = np.zeros(max(len(o), 1), WINDOW_RESULT_DTYPE)
    pmf = np.zeros((max(len(o), 1), int(bins))) if want_pmf else None
    t = None if target is None else np.ascontiguousarray(histogram_from_array(target))
    check(_lib.load().salvox_window_ops(_ctx(ctx).handle, ptr(v), nx, ny, nz, C.byref(iw), ptr(t),
                                        ptr(o), len(o), ptr(out), ptr(pmf)))
    return out[: len(o)], (pmf[: len(o)] if want_pmf else None)


def _op(kind, center=(0.0, 0.0, 0.0), H=None, kernel="identity", step_kernel="identity"):
    from ._lib import WINDOW_OP_DTYPE

    o = np.zeros(1, WINDOW_OP_DTYPE)
    o["op"] = kind
    o["kernel"] = KERNELS[kernel]
    o["step_kernel"] = KERNELS[step_kernel]
    c = np.zeros(3)
    c[: len(center)] = center
    o["center"] = c
    if H is not None:
        o["H"] = np.asarray(H, np.float64).reshape(9)
    return o


def candidate_histogram(volume, center, H, window_low=None, window_high=None, bins=64,
                        kernel="epanechnikov", ctx=None):
    """candidate_histogram (py_module.cpp:125-137, window.cpp:5-27) on the device."""
    from ._lib import WOP_HIST

    r, pmf = window_ops(volume, _op(WOP_HIST, center, H, kernel), window_low, window_high, bins,
                        ctx=ctx, want_pmf=True)
    if not r[0]["ok"]:
        raise ValueError("candidate_histogram: window support holds no usable in-bounds voxel")
    return pmf[0].copy()


def pdf_difference(volume, center, scale, window_low=None, window_high=None, bins=64,
                   kernel="identity", ctx=None):
    """pdf_difference (py_module.cpp:139-147, window.cpp:30-51) on the device: isotropic
    window of the given scale (z pinned to 1 voxel for 2D arrays)."""
    from ._lib import WOP_PDF_DIFF

    v = np.asarray(volume)
    two_d = v.ndim == 2 or v.shape[0] == 1
    s2 = float(scale) ** 2
    H = np.diag([s2, s2, 1.0 if two_d else s2])
    r, _ = window_ops(volume, _op(WOP_PDF_DIFF, center, H, kernel), window_low, window_high, bins,
                      ctx=ctx)
    if r[0]["ok"] < 0:
        raise ValueError("pdf_difference: degenerate scale (inner flank below 1 voxel)")
    if r[0]["ok"] == 0:
        raise ValueError("pdf_difference: degenerate flanking support")
    return float(r[0]["value"][0])


def shift_step(volume, x, half_extents, window_low=None, window_high=None, bins=64,
               step_kernel="identity", hist_kernel="identity", target=None, ctx=None):
    """shift_step (shift.hpp:49-52, shift.cpp:15-34) on the device -> new position or None."""
    from ._lib import WOP_SHIFT_STEP

    v = np.asarray(volume)
    half = np.asarray(half_extents, np.float64).copy()
    if v.ndim == 2 or v.shape[0] == 1:
        half[2] = 1.0  # shift.cpp:9
    H = np.diag(half * half)
    r, _ = window_ops(volume, _op(WOP_SHIFT_STEP, x, H, hist_kernel, step_kernel), window_low,
                      window_high, bins, target=target, ctx=ctx)
    return r[0]["value"].copy() if r[0]["ok"] else None


def box_entropy_bits(volume, x0, x1, y0, y1, z0=0.0, z1=0.0, window_low=None, window_high=None,
                     bins=64, min_voxels=4, ctx=None):
    """box_entropy_bits (quadrant.hpp:58-60, quadrant.cpp:18-35) on the device; the z
    range generalises it to the octant boxes."""
    from ._lib import WOP_BOX_ENTROPY

    o = _op(WOP_BOX_ENTROPY)
    o["box"] = [x0, x1, y0, y1, z0, z1]
    o["min_voxels"] = int(min_voxels)
    r, _ = window_ops(volume, o, window_low, window_high, bins, ctx=ctx)
    return float(r[0]["value"][0])


def ascent_step(volume, points, scale_range, window_low=None, window_high=None, bins=64, dims=2,
                ctx=None):
    """quadrant_step (quadrant.cpp:37-81; dims = 2) or the octant step (dims = 3) for many
    points in one launch -> (moved[n, 3], ASCENT_STATE_DTYPE[n], visits)."""
    from ._lib import ASCENT_STATE_DTYPE

    v, nx, ny, nz = _volume(volume)
    iw = _window(window_low, window_high, bins)
    pts = np.asarray(points, np.float64)
    if pts.ndim == 1:
        pts = pts[None]
    if pts.shape[-1] == 2:
        pts = np.concatenate([pts, np.zeros(pts.shape[:-1] + (1,))], axis=-1)
    pts = np.ascontiguousarray(pts)
    sc = np.ascontiguousarray(scale_range, np.int32)
    moved = np.zeros((max(len(pts), 1), 3))
    st = np.zeros(max(len(pts), 1), ASCENT_STATE_DTYPE)
    visits = C.c_uint64(0)
    check(_lib.load().salvox_ascent_step(_ctx(ctx).handle, ptr(v), nx, ny, nz, C.byref(iw),
                                         int(dims), ptr(sc), len(sc), ptr(pts), len(pts),
                                         ptr(moved), ptr(st), C.byref(visits)))
    return moved[: len(pts)], st[: len(pts)], int(visits.value)


# -------------------------------------------------- pmf functionals (host)
def entropy_nats(pmf):
    """entropy_nats (py_module.cpp:86-88, histogram.hpp:56-62): normalises the input,
    max(-sum p ln p, 0) in bin order."""
    import math

    p = histogram_from_array(pmf)
    h = 0.0
    for v in p.tolist():
        if v > 0.0:
            h -= v * math.log(v)
    return max(h, 0.0)


def entropy_bits(pmf):
    """entropy_bits (py_module.cpp:82-84, histogram.hpp:65-67)."""
    import math

    return entropy_nats(pmf) / math.log(2.0)


def bhattacharyya(p, q):
    """bhattacharyya (py_module.cpp:95-97, histogram.hpp:95-103), capped at 1."""
    import math

    a, b = histogram_from_array(p), histogram_from_array(q)
    if len(a) != len(b):
        raise ValueError("bhattacharyya: bin count mismatch")
    rho = 0.0
    for x, y in zip(a.tolist(), b.tolist()):
        rho += math.sqrt(x * y)
    return min(rho, 1.0)


def mixture_entropy(alpha, bins):
    """mixture_entropy (py_module.cpp:90-91, histogram.hpp:73-83): entropy (nats) of M bins
    blended with fraction alpha into one background bin,
    -(a/M + 1-a) ln(a/M + 1-a) - a (M-1)/M ln(a/M)."""
    import math

    if bins < 2:
        raise ValueError("mixture_entropy: bins must be >= 2")
    if alpha < 0.0 or alpha > 1.0:
        raise ValueError("mixture_entropy: alpha outside [0,1]")
    if alpha == 0.0:
        return 0.0
    m = float(bins)
    shared = alpha / m + (1.0 - alpha)
    return -shared * math.log(shared) - alpha * (m - 1.0) / m * math.log(alpha / m)


def mixture_entropy_derivative(alpha, bins):
    """mixture_entropy_derivative (py_module.cpp:92-93, histogram.hpp:86-93):
    (M-1)/M ln((a + M(1-a)) / a) on (0, 1]."""
    import math

    if bins < 2:
        raise ValueError("mixture_entropy_derivative: bins must be >= 2")
    if alpha <= 0.0 or alpha > 1.0:
        raise ValueError("mixture_entropy_derivative: alpha outside (0,1]")
    m = float(bins)
    return (m - 1.0) / m * math.log((alpha + m * (1.0 - alpha)) / alpha)


def histogram_from_array(arr):
    """histogram_from_array (py_module.cpp:46-54): 1D, normalised by the sequential
    bin-order mass (Histogram::normalize, histogram.hpp:21-33)."""
    a = np.asarray(arr, np.float64)
    if a.ndim != 1:
        raise ValueError("expected a 1D histogram")
    mass = 0.0
    for v in a.tolist():
        mass += v
    if not mass > 0.0:
        raise ValueError("Histogram::normalize: zero total mass")
    return np.array([v / mass for v in a.tolist()], np.float64)


def _detect_params(method="shift", seed_spacing=16.0, scales=(8.0,), k=20, dedupe_radius=5.0,
                   entropy_quantile=0.9, pdf_quantile=0.0, workers=1, seed_mode="lattice",
                   seed_count=400, rng_seed=0, quadrant_eta=0.5, quadrant_max_iters=50,
                   quadrant_scales=None, shift_min_step=0.1, shift_max_iters=50,
                   shift_step_kernel="identity", shift_hist_kernel="identity",
                   min_inbounds_fraction=0.1, target=None, abmsod_threshold=1e-4,
                   abmsod_max_iters=15, abmsod_kernel="gaussian", lambda_min=4.0,
                   lambda_max=0.0):
    keep = []
    P = _lib.DetectParams()
    P.method = METHODS[method]
    P.seed_mode = 0 if seed_mode == "lattice" else 1
    P.seed_spacing = float(seed_spacing)
    P.seed_count = int(seed_count)
    P.top_k = int(k)
    P.rng_seed = int(rng_seed)
    sc = (C.c_double * len(scales))(*[float(s) for s in scales])
    keep.append(sc)
    P.scales = sc
    P.n_scales = len(scales)
    P.workers = int(workers)
    P.dedupe_radius = float(dedupe_radius)
    P.entropy_quantile = float(entropy_quantile)
    P.pdf_quantile = float(pdf_quantile)
    P.quadrant_eta = float(quadrant_eta)
    P.quadrant_max_iters = int(quadrant_max_iters)
    if quadrant_scales is not None:
        qs = (C.c_int32 * len(quadrant_scales))(*[int(q) for q in quadrant_scales])
        keep.append(qs)
        P.quadrant_scales = qs
        P.n_quadrant_scales = len(quadrant_scales)
    P.shift_min_step = float(shift_min_step)
    P.shift_max_iters = int(shift_max_iters)
    P.shift_step_kernel = KERNELS[shift_step_kernel]
    P.shift_hist_kernel = KERNELS[shift_hist_kernel]
    P.shift_min_inbounds_fraction = float(min_inbounds_fraction)
    P.abmsod_threshold = float(abmsod_threshold)
    P.abmsod_max_iters = int(abmsod_max_iters)
    P.abmsod_kernel = KERNELS[abmsod_kernel]
    P.abmsod_lambda_min = float(lambda_min)
    P.abmsod_lambda_max = float(lambda_max)
    P.abmsod_min_inbounds_fraction = float(min_inbounds_fraction)
    if target is not None:
        t = np.ascontiguousarray(histogram_from_array(target))
        keep.append(t)
        P.shift_target = t.ctypes.data_as(C.POINTER(C.c_double))
        P.abmsod_target = P.shift_target
    return P, keep


def detect_records(volume, method="shift", seed_spacing=16.0, scales=(8.0,), k=20,
                   dedupe_radius=5.0, window_low=None, window_high=None, bins=64,
                   entropy_quantile=0.9, pdf_quantile=0.0, workers=1, ctx=None, per_seed=False,
                   **extra):
    """Structured form of detect: (selected DET_DTYPE, per-seed DET_DTYPE or None, visits)."""
    v, nx, ny, nz = _volume(volume)
    iw = _window(window_low, window_high, bins)
    P, keep = _detect_params(method, seed_spacing, scales, k, dedupe_radius, entropy_quantile,
                             pdf_quantile, workers, **extra)
    c = _ctx(ctx)
    ns = C.c_int64(0)
    check(_lib.load().salvox_plan_seeds(nx, ny, nz, P.seed_mode, P.seed_spacing, P.seed_count,
                                        C.cast(P.scales, C.c_void_p), P.n_scales, P.rng_seed,
                                        None, None, 0, C.byref(ns)))
    out = np.empty(max(int(k), 1), DET_DTYPE)
    n_out = C.c_int64(0)
    seeds = np.empty(max(ns.value, 1), DET_DTYPE) if per_seed else None
    n_seed = C.c_int64(0)
    visits = C.c_uint64(0)
    check(_lib.load().salvox_detect(
        c.handle, ptr(v), nx, ny, nz, C.byref(iw), C.byref(P), ptr(out), len(out),
        C.byref(n_out), ptr(seeds), len(seeds) if per_seed else 0, C.byref(n_seed),
        C.byref(visits)))
    del keep
    return (out[: n_out.value].copy(), seeds[: n_seed.value].copy() if per_seed else None,
            int(visits.value))


def detect_batch_device(d_volumes, batch, shape_zyx, method="shift", seed_spacing=16.0,
                        scales=(8.0,), k=20, dedupe_radius=5.0, window_low=None,
                        window_high=None, bins=64, entropy_quantile=0.9, pdf_quantile=0.0,
                        workers=1, ctx=None, **extra):
    """detect() over `batch` device-resident volumes stored back to back at the
    device address d_volumes (a CUDA tensor, or an int address whose producer the
    caller has already synchronised): one seek
    launch covers every volume -> ([selected DET_DTYPE per volume], visits)."""
    nz, ny, nx = shape_zyx if len(shape_zyx) == 3 else (1,) + tuple(shape_zyx)
    iw = _window(window_low, window_high, bins)
    P, keep = _detect_params(method, seed_spacing, scales, k, dedupe_radius, entropy_quantile,
                             pdf_quantile, workers, **extra)
    kk = max(int(k), 1)
    out = np.empty(max(batch, 1) * kk, DET_DTYPE)
    n_out = np.zeros(max(batch, 1), np.int64)
    visits = C.c_uint64(0)
    c = _ctx(ctx)
    if hasattr(d_volumes, "data_ptr"):  # a torch tensor: order after its producer
        c.after_torch(d_volumes)
        d_volumes = d_volumes.data_ptr()
    check(_lib.load().salvox_detect_batch_device(
        c.handle, C.c_void_p(int(d_volumes)), int(batch), nx, ny, nz, C.byref(iw),
        C.byref(P), ptr(out), kk, ptr(n_out), C.byref(visits)))
    del keep
    return [out[v * kk: v * kk + n_out[v]].copy() for v in range(batch)], int(visits.value)


def detect_shard(volume, rank, world, method="shift", seed_spacing=16.0, scales=(8.0,), k=20,
                 dedupe_radius=5.0, window_low=None, window_high=None, bins=64,
                 entropy_quantile=0.9, pdf_quantile=0.0, workers=1, ctx=None, **extra):
    """This rank's share of detect's plan (salvox_detect_shard): per-seed
    detections for plan positions j % world == rank, in increasing j ->
    (DET_DTYPE[n_local], n_total, visits)."""
    v, nx, ny, nz = _volume(volume)
    iw = _window(window_low, window_high, bins)
    P, keep = _detect_params(method, seed_spacing, scales, k, dedupe_radius, entropy_quantile,
                             pdf_quantile, workers, **extra)
    c = _ctx(ctx)
    ns = C.c_int64(0)
    check(_lib.load().salvox_plan_seeds(nx, ny, nz, P.seed_mode, P.seed_spacing, P.seed_count,
                                        C.cast(P.scales, C.c_void_p), P.n_scales, P.rng_seed,
                                        None, None, 0, C.byref(ns)))
    cap = ns.value // max(int(world), 1) + 1
    out = np.empty(max(cap, 1), DET_DTYPE)
    n_local, n_total, visits = C.c_int64(0), C.c_int64(0), C.c_uint64(0)
    check(_lib.load().salvox_detect_shard(
        c.handle, ptr(v), nx, ny, nz, C.byref(iw), C.byref(P), int(rank), int(world), ptr(out),
        cap, C.byref(n_local), C.byref(n_total), C.byref(visits)))
    del keep
    return out[: n_local.value].copy(), int(n_total.value), int(visits.value)


def detect(volume, method="shift", seed_spacing=16.0, scales=(8.0,), k=20, dedupe_radius=5.0,
           window_low=None, window_high=None, bins=64, entropy_quantile=0.9, pdf_quantile=0.0,
           workers=1, ctx=None, **extra):
    """Seed, seek, threshold and dedupe in one call; returns detection dicts
    (py_module.cpp:206-230). method: "shift", "quadrant" (2D) or "octant" (3D, new)."""
    sel, _, _ = detect_records(volume, method, seed_spacing, scales, k, dedupe_radius, window_low,
                               window_high, bins, entropy_quantile, pdf_quantile, workers, ctx,
                               **extra)
    return [detection_to_dict(d) for d in sel]


def seek_records(volume, positions, scales=None, half_extents=None, method="shift",
                 window_low=None, window_high=None, bins=64, seed_index=None, ctx=None, **extra):
    """Per-seed trajectories (salvox_seek) in seed order -> (DET_DTYPE[n], visits)."""
    v, nx, ny, nz = _volume(volume)
    pos = np.ascontiguousarray(np.asarray(positions, np.float64).reshape(-1, 3))
    n = len(pos)
    sc = None if scales is None else np.ascontiguousarray(np.broadcast_to(
        np.asarray(scales, np.float64), (n,)))
    he = None if half_extents is None else np.ascontiguousarray(np.broadcast_to(
        np.asarray(half_extents, np.float64), (n, 3)))
    si = None if seed_index is None else np.ascontiguousarray(seed_index, np.int32)
    iw = _window(window_low, window_high, bins)
    P, keep = _detect_params(method, **extra)
    c = _ctx(ctx)
    out = np.empty(max(n, 1), DET_DTYPE)
    visits = C.c_uint64(0)
    check(_lib.load().salvox_seek(c.handle, ptr(v), nx, ny, nz, C.byref(iw), C.byref(P), ptr(pos),
                                  ptr(sc), ptr(he), ptr(si), n, ptr(out), C.byref(visits)))
    del keep
    return out[:n].copy(), int(visits.value)


def saliency_shift(volume, seed, half_extents, window_low=None, window_high=None, bins=64,
                   max_iters=50, min_step=0.1, ctx=None, **extra):
    """Fixed-bandwidth mean shift toward the uniform pmf (py_module.cpp:159-170)."""
    d, _ = seek_records(volume, [seed], half_extents=[half_extents], method="shift",
                        window_low=window_low, window_high=window_high, bins=bins, ctx=ctx,
                        shift_max_iters=max_iters, shift_min_step=min_step, **extra)
    return detection_to_dict(d[0])


def quadrant_seek(volume, seeds, scale_range, window_low=None, window_high=None, bins=64, eta=0.5,
                  max_iters=50, ctx=None, octant=False):
    """quadrant_seek (quadrant.hpp:73-76, quadrant.cpp:83-125) on the device; octant=True
    runs the 3D octant ascent. Returns ASCENT_DTYPE records (position, entropy_bits and
    best_scale of the highest-entropy window, iterations, converged, degenerate) and the
    EvalCounter visits."""
    from ._lib import ASCENT_DTYPE

    v, nx, ny, nz = _volume(volume)
    s = np.asarray(seeds, np.float64)
    if s.ndim == 1:
        s = s[None]
    if s.shape[-1] == 2:
        s = np.concatenate([s, np.zeros(s.shape[:-1] + (1,))], axis=-1)
    s = np.ascontiguousarray(s)
    if len(s) == 0:
        raise ValueError("quadrant_seek: no seeds")  # quadrant.cpp:290
    iw = _window(window_low, window_high, bins)
    sr = np.ascontiguousarray(scale_range, np.int32)
    out = np.empty(len(s), ASCENT_DTYPE)
    visits = C.c_uint64(0)
    check(_lib.load().salvox_ascent_seek(_ctx(ctx).handle, ptr(v), nx, ny, nz, C.byref(iw),
                                         3 if octant else 2, ptr(sr), len(sr), float(eta),
                                         int(max_iters), ptr(s), len(s), ptr(out),
                                         C.byref(visits)))
    return out, int(visits.value)


def abmsod_records(volume, seeds, radius=None, H=None, window_low=None, window_high=None,
                   bins=64, max_iterations=15, threshold=1e-4, kernel="gaussian",
                   lambda_min=4.0, lambda_max=0.0, min_inbounds_fraction=0.1, target=None,
                   trace=False, ctx=None):
    """abmsod_run (abmsod.hpp:77-79) for many seeds on the device. Seed windows are
    H (3x3, or one per seed) or EllipsoidWindow::isotropic(seed, radius).
    Returns (DET_DTYPE[n], [ABMSOD_ITER_DTYPE arrays] or None, visits)."""
    from ._lib import ABMSOD_ITER_DTYPE, AbmsodParams

    v, nx, ny, nz = _volume(volume)
    s = np.asarray(seeds, np.float64)
    if s.ndim == 1:
        s = s[None]
    if s.shape[-1] == 2:
        s = np.concatenate([s, np.zeros(s.shape[:-1] + (1,))], axis=-1)
    s = np.ascontiguousarray(s)
    n = len(s)
    hs = None if H is None else np.ascontiguousarray(
        np.broadcast_to(np.asarray(H, np.float64).reshape(-1, 9), (n, 9)))
    rs = None if radius is None else np.ascontiguousarray(
        np.broadcast_to(np.asarray(radius, np.float64), (n,)))
    if hs is None and rs is None:
        raise ValueError("abmsod: give radius or H")
    iw = _window(window_low, window_high, bins)
    P = AbmsodParams(float(threshold), int(max_iterations), KERNELS[kernel], float(lambda_min),
                     float(lambda_max), float(min_inbounds_fraction), None)
    t = None
    if target is not None:
        t = np.ascontiguousarray(histogram_from_array(target))
        P.target = t.ctypes.data_as(C.POINTER(C.c_double))
    out = np.empty(max(n, 1), DET_DTYPE)
    tr = np.zeros(max(n, 1) * max(int(max_iterations), 1), ABMSOD_ITER_DTYPE) if trace else None
    tn = np.zeros(max(n, 1), np.int32) if trace else None
    visits = C.c_uint64(0)
    check(_lib.load().salvox_abmsod_run(_ctx(ctx).handle, ptr(v), nx, ny, nz, C.byref(iw),
                                        C.byref(P), ptr(s), ptr(hs), ptr(rs), C.c_int64(n), ptr(out),
                                        ptr(tr), ptr(tn), C.byref(visits)))
    del t
    traces = None
    if trace:
        m = int(max_iterations)
        traces = [tr[i * m: i * m + tn[i]].copy() for i in range(n)]
    return out[:n].copy(), traces, int(visits.value)


def abmsod(volume, seed, radius, window_low=None, window_high=None, bins=64, max_iterations=15,
           threshold=1e-4, ctx=None):
    """abmsod (py_module.cpp:172-184): one seed, isotropic seed window -> detection dict."""
    d, _, _ = abmsod_records(volume, [seed], radius=radius, window_low=window_low,
                             window_high=window_high, bins=bins, max_iterations=max_iterations,
                             threshold=threshold, ctx=ctx)
    return detection_to_dict(d[0])


def bandwidth_from_moment(outer, weight_sum, dim, lambda_min, lambda_max):
    """bandwidth_from_moment (abmsod.hpp:66-70) -> H (3x3)."""
    H = np.zeros(9)
    o = np.ascontiguousarray(outer, np.float64).reshape(9)
    check(_lib.load().salvox_bandwidth_from_moment(
        ptr(o), C.c_double(weight_sum), C.c_int32(int(dim)), C.c_double(lambda_min),
        C.c_double(lambda_max), ptr(H)))
    return H.reshape(3, 3)


def hu_moments(image, ctx=None):
    """hu_moments (py_module.cpp:149-155): the seven invariants of a 2D image (device)."""
    a = np.ascontiguousarray(image, np.float32)
    if a.ndim == 3 and a.shape[0] == 1:
        a = a[0]
    if a.ndim != 2:
        raise ValueError("hu_moments: expected a 2D slice")
    out = np.zeros(7)
    check(_lib.load().salvox_hu_moments(_ctx(ctx).handle, ptr(a), a.shape[1], a.shape[0], ptr(out)))
    return out


def _as_records(dets):
    if isinstance(dets, np.ndarray) and dets.dtype == DET_DTYPE:
        return np.ascontiguousarray(dets)
    recs = np.zeros(len(dets), DET_DTYPE)
    for i, d in enumerate(dets):
        recs[i]["center"] = d["center"]
        recs[i]["H"] = np.asarray(d["H"], np.float64).reshape(9)
    return recs


def hu_template_distance(dets, volume, template, slices=5, ctx=None):
    """hu_template_distance (pipeline.hpp:73-74) for each detection (records or
    dicts) -> array of mean Hu distances (inf when no crop has mass)."""
    v, nx, ny, nz = _volume(volume)
    t = np.ascontiguousarray(template, np.float32)
    if t.ndim == 3 and t.shape[0] == 1:
        t = t[0]
    recs = _as_records(dets)
    out = np.zeros(max(len(recs), 1))
    check(_lib.load().salvox_hu_template_distance(
        _ctx(ctx).handle, ptr(v), nx, ny, nz, ptr(recs), C.c_int64(len(recs)), ptr(t), t.shape[1],
        t.shape[0], int(slices), ptr(out)))
    return out[: len(recs)]


def hu_filter(dets, volume, template, slices=5, ctx=None):
    """hu_filter (pipeline.hpp:69-70): index of the detection whose crops best match."""
    if len(dets) == 0:
        raise ValueError("hu_filter: no detections")
    d = hu_template_distance(dets, volume, template, slices, ctx)
    best, best_d = 0, np.inf
    for i, x in enumerate(d):
        if x < best_d:
            best, best_d = i, x
    return best


def rasterize_window(shape_zyx, center, H, ctx=None):
    """rasterize_window (pipeline.hpp:61): sorted linear indices of the window's
    in-bounds support on a frame of the given shape, rasterised on the device."""
    nz, ny, nx = shape_zyx if len(shape_zyx) == 3 else (1,) + tuple(shape_zyx)
    c = np.ascontiguousarray(center, np.float64)
    h = np.ascontiguousarray(np.asarray(H, np.float64).reshape(9))
    n = C.c_int64(0)
    cx = _ctx(ctx)
    check(_lib.load().salvox_rasterize_window(cx.handle, nx, ny, nz, ptr(c), ptr(h), None,
                                              C.c_int64(0), C.byref(n)))
    out = np.zeros(max(n.value, 1), np.uint64)
    if n.value:
        check(_lib.load().salvox_rasterize_window(cx.handle, nx, ny, nz, ptr(c), ptr(h), ptr(out),
                                                  C.c_int64(n.value), C.byref(n)))
    return out[: n.value]


def jaccard(a, b):
    """jaccard (pipeline.hpp:63): |A n B| / |A u B| over sorted voxel index sets."""
    a = np.asarray(a, np.uint64)
    b = np.asarray(b, np.uint64)
    if len(a) == 0 and len(b) == 0:
        raise ValueError("jaccard: both sets are empty")
    inter = len(np.intersect1d(a, b, assume_unique=True))
    return inter / float(len(a) + len(b) - inter)


def select(dets, entropy_quantile=0.9, pdf_quantile=0.0, k=20, dedupe_radius=5.0, ctx=None):
    """Alive filter + population-quantile thresholds + dedupe (pipeline.cpp:383-401)."""
    d = np.ascontiguousarray(dets, DET_DTYPE)
    out = np.empty(max(len(d), 1), DET_DTYPE)
    n = C.c_int64(0)
    check(_lib.load().salvox_select(_ctx(ctx).handle, ptr(d), len(d), entropy_quantile,
                                    pdf_quantile, int(k), dedupe_radius, ptr(out), C.byref(n)))
    return out[: n.value].copy()


def dedupe_top_k(dets, k, radius, ctx=None):
    """dedupe_top_k (pipeline.hpp:57)."""
    d = np.ascontiguousarray(dets, DET_DTYPE)
    out = np.empty(max(len(d), 1), DET_DTYPE)
    n = C.c_int64(0)
    check(_lib.load().salvox_dedupe_top_k(_ctx(ctx).handle, ptr(d), len(d), int(k), radius,
                                          ptr(out), C.byref(n)))
    return out[: n.value].copy()


# ----------------------------------------------------------------- data formats
def plan_seeds(shape_zyx, mode="lattice", spacing=16.0, count=0, scales=(8.0,), rng_seed=0):
    """plan_seeds (seeds.hpp:43) -> (positions (n,3), scales (n,))."""
    nz, ny, nx = shape_zyx if len(shape_zyx) == 3 else (1,) + tuple(shape_zyx)
    sc = np.ascontiguousarray(scales, np.float64)
    m = 0 if mode == "lattice" else 1
    n = C.c_int64(0)
    check(_lib.load().salvox_plan_seeds(nx, ny, nz, m, float(spacing), int(count), ptr(sc),
                                        len(sc), int(rng_seed), None, None, 0, C.byref(n)))
    pos = np.empty((n.value, 3))
    ss = np.empty(n.value)
    check(_lib.load().salvox_plan_seeds(nx, ny, nz, m, float(spacing), int(count), ptr(sc),
                                        len(sc), int(rng_seed), ptr(pos), ptr(ss), n.value,
                                        C.byref(n)))
    return pos, ss


_SHAPES = {"box": 0, "ball": 1, "ellipsoid": 2}


def _phantom_args(spec):
    """PhantomSpec JSON text / dict (phantom.cpp:226-277) -> the C-ABI argument arrays."""
    if isinstance(spec, str):
        spec = json.loads(spec)
    nx, ny, nz = (int(d) for d in spec["dims"])
    bg = spec.get("background", {"type": "constant", "value": 0.0})
    regions = spec.get("regions", [])
    n = max(len(regions), 1)
    shape = np.zeros(n, np.int32)
    center = np.zeros(3 * n)
    half = np.zeros(3 * n)
    radius = np.zeros(n)
    axes = np.tile(np.eye(3).ravel(), n).astype(np.float64)
    ftype = np.zeros(n, np.int32)
    flev = np.full(n, 64, np.int32)
    fval = np.zeros(n)
    Hs = []
    for i, r in enumerate(regions):
        shape[i] = _SHAPES[r["shape"]]
        center[3 * i:3 * i + 3] = r["center"]
        if r["shape"] == "box":
            half[3 * i:3 * i + 3] = r["half_extents"]
            H = np.diag(np.square(np.asarray(r["half_extents"], float)))
        elif r["shape"] == "ball":
            radius[i] = r["radius"]
            H = np.eye(3) * r["radius"] * r["radius"]
        else:
            ax = np.asarray(r["axes"], np.float64)
            axes[9 * i:9 * i + 9] = ax.ravel()
            H = ax @ ax.T
        Hs.append(H)
        f = r.get("fill", {"type": "uniform", "levels": 64})
        ftype[i] = 0 if f["type"] == "uniform" else 1
        flev[i] = int(f.get("levels", 64))
        fval[i] = float(f.get("value", 0.0))
    arrays = (shape, center, half, radius, axes, ftype, flev, fval)
    head = (nx, ny, nz, 0 if bg["type"] == "constant" else 1, float(bg.get("value", 0.0)),
            float(bg.get("mean", 0.0)), float(bg.get("sigma", 1.0)), len(regions))
    return head, arrays, int(spec.get("rng_seed", 0)), Hs


def make_phantom(spec):
    """make_phantom (py_module.cpp:96-112): spec is PhantomSpec JSON text or a dict
    (phantom.cpp:226-277). Returns (array[z,y,x], regions[{center, H}])."""
    head, arrays, seed, Hs = _phantom_args(spec)
    nx, ny, nz, nreg = head[0], head[1], head[2], head[7]
    out = np.empty((nz, ny, nx), np.float32)
    cent = np.zeros(3 * max(nreg, 1))
    check(_lib.load().salvox_make_phantom(*head, *(ptr(a) for a in arrays), seed, ptr(out), ptr(cent)))
    gt = [{"center": tuple(cent[3 * i:3 * i + 3]), "H": Hs[i]} for i in range(nreg)]
    return out, gt


def make_phantom_device(spec, device=0, out=None, ctx=None):
    """make_phantom generated on the GPU -> (torch CUDA
    tensor [z, y, x] float32, regions). Integer / constant fills are
    bit-identical to make_phantom; a gaussian background may differ in the last
    float place. `out` may be a preallocated contiguous CUDA float32 tensor."""
    import torch

    head, arrays, seed, Hs = _phantom_args(spec)
    nx, ny, nz, nreg = head[0], head[1], head[2], head[7]
    if out is None:
        out = torch.empty((nz, ny, nx), dtype=torch.float32, device=torch.device("cuda", device))
    elif (tuple(out.shape) != (nz, ny, nx) or out.dtype != torch.float32 or not out.is_cuda
          or not out.is_contiguous()):
        raise ValueError("make_phantom_device: out must be a contiguous CUDA float32 [z, y, x] tensor")
    cent = np.zeros(3 * max(nreg, 1))
    c = _ctx(ctx)
    c.after_torch(out)
    check(_lib.load().salvox_make_phantom_device(c.handle, *head,
                                                 *(ptr(a) for a in arrays), seed,
                                                 C.c_void_p(out.data_ptr()), ptr(cent)))
    gt = [{"center": tuple(cent[3 * i:3 * i + 3]), "H": Hs[i]} for i in range(nreg)]
    return out, gt
