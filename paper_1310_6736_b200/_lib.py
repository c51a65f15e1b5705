"""ctypes binding of libsalvox_b200.so (the C-ABI declared in include/salvox_capi.h).

The library is built in-tree (``python -m paper_1310_6736_b200.build`` or
``__graft_entry__.build()``). There is no CPU fallback: loading fails loudly if
the .so is missing, and every compute call raises ``SalvoxCudaError`` without a
CUDA device.
"""
from __future__ import annotations

import ctypes as C
import os
import threading

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libsalvox_b200.so")

SALVOX_OK, SALVOX_EINVAL, SALVOX_ECUDA, SALVOX_EUNSUPPORTED, SALVOX_ERUNTIME = 0, 1, 2, 3, 4
KERNELS = {"identity": 0, "epanechnikov": 1, "gaussian": 2}
METHODS = {"quadrant": 0, "shift": 1, "abmsod": 2, "octant": 3}
FLAG_CONVERGED, FLAG_DEGENERATE, FLAG_CLAMPED = 1, 2, 4

# salvox_detection (136 bytes) and salvox_maximum (48 bytes) as numpy records
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
        ("reserved", "<i4"),
    ]
)
ASCENT_DTYPE = np.dtype(
    [("position", "<f8", (3,)), ("entropy_bits", "<f8"), ("best_scale", "<i4"),
     ("iterations", "<i4"), ("converged", "<i4"), ("degenerate", "<i4")]
)
MAX_DTYPE = np.dtype(
    [("position", "<f8", (3,)), ("score", "<f8"), ("scale", "<f8"), ("linear_index", "<i8")]
)
assert DET_DTYPE.itemsize == 136 and MAX_DTYPE.itemsize == 48


class SalvoxError(RuntimeError):
    pass


class SalvoxCudaError(SalvoxError):
    """CUDA / device failure (SALVOX_ECUDA). Raised instead of any CPU fallback."""


class Window(C.Structure):
    _fields_ = [("low", C.c_double), ("high", C.c_double), ("bins", C.c_int32),
                ("full_range", C.c_int32)]


class DetectParams(C.Structure):
    _fields_ = [
        ("method", C.c_int32),
        ("seed_mode", C.c_int32),
        ("seed_spacing", C.c_double),
        ("seed_count", C.c_int32),
        ("top_k", C.c_int32),
        ("rng_seed", C.c_uint64),
        ("scales", C.POINTER(C.c_double)),
        ("n_scales", C.c_int32),
        ("workers", C.c_int32),
        ("dedupe_radius", C.c_double),
        ("entropy_quantile", C.c_double),
        ("pdf_quantile", C.c_double),
        ("quadrant_eta", C.c_double),
        ("quadrant_max_iters", C.c_int32),
        ("n_quadrant_scales", C.c_int32),
        ("quadrant_scales", C.POINTER(C.c_int32)),
        ("shift_min_step", C.c_double),
        ("shift_max_iters", C.c_int32),
        ("shift_step_kernel", C.c_int32),
        ("shift_hist_kernel", C.c_int32),
        ("reserved", C.c_int32),
        ("shift_min_inbounds_fraction", C.c_double),
        ("shift_target", C.POINTER(C.c_double)),
        ("abmsod_threshold", C.c_double),
        ("abmsod_max_iters", C.c_int32),
        ("abmsod_kernel", C.c_int32),
        ("abmsod_lambda_min", C.c_double),
        ("abmsod_lambda_max", C.c_double),
        ("abmsod_min_inbounds_fraction", C.c_double),
        ("abmsod_target", C.POINTER(C.c_double)),
    ]


class AbmsodParams(C.Structure):
    _fields_ = [
        ("threshold", C.c_double),
        ("max_iterations", C.c_int32),
        ("kernel", C.c_int32),
        ("lambda_min", C.c_double),
        ("lambda_max", C.c_double),
        ("min_inbounds_fraction", C.c_double),
        ("target", C.POINTER(C.c_double)),
    ]


# salvox_window_op / salvox_window_result / salvox_ascent_state (include/salvox_capi.h)
WINDOW_OP_DTYPE = np.dtype([("op", "<i4"), ("kernel", "<i4"), ("step_kernel", "<i4"),
                            ("min_voxels", "<i4"), ("center", "<f8", (3,)), ("H", "<f8", (9,)),
                            ("box", "<f8", (6,))])
WINDOW_RESULT_DTYPE = np.dtype([("value", "<f8", (3,)), ("support", "<u8"), ("visits", "<u8"),
                                ("ok", "<i4"), ("pad_", "<i4")])
ASCENT_STATE_DTYPE = np.dtype([("entropy", "<f8", (8,)), ("best_scale", "<i4", (8,)),
                               ("norm_entropy", "<f8", (8,)), ("displacement", "<f8", (3,)),
                               ("degenerate", "<i4"), ("pad_", "<i4")])
WOP_HIST, WOP_SHIFT_STEP, WOP_PDF_DIFF, WOP_BOX_ENTROPY = 0, 1, 2, 3

ABMSOD_ITER_DTYPE = np.dtype([("position", "<f8", (3,)), ("H", "<f8", (9,)),
                              ("bhattacharyya", "<f8"), ("max_bhattacharyya", "<f8"),
                              ("eig_min", "<f8"), ("eig_max", "<f8")])


# Every symbol include/salvox_capi.h declares (checked by tests/test_capi_symbols.py).
EXPORTS = [
    "salvox_last_error", "salvox_version", "salvox_ctx_create", "salvox_ctx_destroy",
    "salvox_ctx_set_stream", "salvox_ctx_wait_stream", "salvox_ctx_launch_count",
    "salvox_exhaustive",
    "salvox_exhaustive_slab", "salvox_exhaustive_device", "salvox_exhaustive_slab_device",
    "salvox_exhaustive_slab_scores", "salvox_exhaustive_slab_edges",
    "salvox_exhaustive_slab_maxima", "salvox_last_maxima", "salvox_last_maxima_device",
    "salvox_last_maps",
    "salvox_merge_maxima_device",
    "salvox_exhaustive_debug_hist", "salvox_detect", "salvox_detect_batch_device",
    "salvox_detect_shard", "salvox_seek",
    "salvox_select", "salvox_dedupe_top_k", "salvox_plan_seeds", "salvox_make_phantom",
    "salvox_make_phantom_device",
    "salvox_ascent_seek", "salvox_ascent_step", "salvox_window_ops", "salvox_abmsod_run",
    "salvox_bandwidth_from_moment",
    "salvox_upload_widen", "salvox_widen_device", "salvox_rasterize_window",
    "salvox_hu_moments", "salvox_hu_template_distance",
]
# include/salvox_bench.h
BENCH_EXPORTS = ["salvox_probe_smem_peak", "salvox_probe_prmt_rate", "salvox_ctx_set_profiling",
                 "salvox_ctx_kernel_time"]

_lib = None
_lock = threading.Lock()


def load():
    """Loads the in-tree shared library (raises if it was not built)."""
    global _lib
    with _lock:
        if _lib is None:
            if not os.path.exists(LIB_PATH):
                raise SalvoxError(
                    f"{LIB_PATH} is missing: build it with `python -m paper_1310_6736_b200.build` "
                    "(there is no CPU fallback)")
            lib = C.CDLL(LIB_PATH)
            _declare(lib)
            _lib = lib
    return _lib


_vp = C.c_void_p
_i32, _i64, _u64, _dbl = C.c_int32, C.c_int64, C.c_uint64, C.c_double
_pi64 = C.POINTER(C.c_int64)
_pu64 = C.POINTER(C.c_uint64)


def _declare(L):
    L.salvox_last_error.restype = C.c_char_p
    L.salvox_version.restype = C.c_int
    L.salvox_ctx_create.argtypes = [C.c_int, C.POINTER(_vp)]
    L.salvox_ctx_destroy.argtypes = [_vp]
    L.salvox_ctx_set_stream.argtypes = [_vp, _vp]
    L.salvox_ctx_wait_stream.argtypes = [_vp, _vp]
    L.salvox_ctx_launch_count.argtypes = [_vp, _pu64]
    L.salvox_exhaustive.argtypes = [_vp, _vp, _i32, _i32, _i32, C.POINTER(Window), _vp, _i32, _i32,
                                    _u64, _vp, _vp, _vp, _i64, _pi64, _pu64]
    L.salvox_exhaustive_slab.argtypes = [_vp, _vp, _i32, _i32, _i32, _i32, _i32, _i32, _i32,
                                         C.POINTER(Window), _vp, _i32, _i32, _u64, _vp, _vp, _vp,
                                         _i64, _pi64, _pu64]
    L.salvox_exhaustive_device.argtypes = [_vp, _vp, _i32, _i32, _i32, C.POINTER(Window), _vp,
                                           _i32, _i32, _u64, _vp, _vp, _pi64]
    L.salvox_exhaustive_slab_device.argtypes = [_vp, _vp, _i32, _i32, _i32, _i32, _i32, _i32,
                                                _i32, C.POINTER(Window), _vp, _i32, _i32, _u64,
                                                _vp, _vp, _pi64]
    L.salvox_exhaustive_slab_scores.argtypes = [_vp, _vp, _i32, _i32, _i32, _i32, _i32, _i32,
                                                _i32, _i32, C.POINTER(Window), _vp, _i32, _i32,
                                                _u64, _vp, _vp, C.POINTER(_u64)]
    L.salvox_exhaustive_slab_edges.argtypes = [_vp, _vp, _vp]
    L.salvox_exhaustive_slab_maxima.argtypes = [_vp, _vp, _vp, _vp, _i64, _pi64]
    L.salvox_last_maxima.argtypes = [_vp, _vp, _i64, _pi64]
    L.salvox_last_maps.argtypes = [_vp, _vp, _vp]
    L.salvox_last_maxima_device.argtypes = [_vp, _vp, _i64, _pi64]
    L.salvox_merge_maxima_device.argtypes = [_vp, _vp, _i64, _vp]
    L.salvox_exhaustive_debug_hist.argtypes = [_vp, _vp, _i32, _vp, _vp, C.POINTER(_i32)]
    L.salvox_detect.argtypes = [_vp, _vp, _i32, _i32, _i32, C.POINTER(Window),
                                C.POINTER(DetectParams), _vp, _i64, _pi64, _vp, _i64, _pi64, _pu64]
    L.salvox_detect_batch_device.argtypes = [_vp, _vp, _i32, _i32, _i32, _i32, C.POINTER(Window),
                                             C.POINTER(DetectParams), _vp, _i64, _vp, _pu64]
    L.salvox_seek.argtypes = [_vp, _vp, _i32, _i32, _i32, C.POINTER(Window),
                              C.POINTER(DetectParams), _vp, _vp, _vp, _vp, _i64, _vp, _pu64]
    L.salvox_ascent_seek.argtypes = [_vp, _vp, _i32, _i32, _i32, C.POINTER(Window), _i32, _vp,
                                     _i32, _dbl, _i32, _vp, _i64, _vp, _pu64]
    L.salvox_ascent_step.argtypes = [_vp, _vp, _i32, _i32, _i32, C.POINTER(Window), _i32, _vp,
                                     _i32, _vp, _i64, _vp, _vp, _pu64]
    L.salvox_window_ops.argtypes = [_vp, _vp, _i32, _i32, _i32, C.POINTER(Window), _vp, _vp, _i64,
                                    _vp, _vp]
    L.salvox_select.argtypes = [_vp, _vp, _i64, _dbl, _dbl, _i32, _dbl, _vp, _pi64]
    L.salvox_dedupe_top_k.argtypes = [_vp, _vp, _i64, _i32, _dbl, _vp, _pi64]
    L.salvox_plan_seeds.argtypes = [_i32, _i32, _i32, _i32, _dbl, _i32, _vp, _i32, _u64, _vp, _vp,
                                    _i64, _pi64]
    L.salvox_make_phantom.argtypes = [_i32, _i32, _i32, _i32, _dbl, _dbl, _dbl, _i32, _vp, _vp,
                                      _vp, _vp, _vp, _vp, _vp, _vp, _u64, _vp, _vp]
    L.salvox_make_phantom_device.argtypes = [_vp, _i32, _i32, _i32, _i32, _dbl, _dbl, _dbl, _i32,
                                             _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _u64, _vp, _vp]
    L.salvox_probe_smem_peak.argtypes = [_vp, C.c_int, C.POINTER(_dbl), C.POINTER(_dbl),
                                         C.POINTER(_dbl)]
    L.salvox_ctx_set_profiling.argtypes = [_vp, C.c_int]
    L.salvox_ctx_kernel_time.argtypes = [_vp, C.POINTER(_dbl), _pi64, C.POINTER(_dbl)]
    for name in EXPORTS + BENCH_EXPORTS:
        if name not in ("salvox_last_error",):
            getattr(L, name).restype = C.c_int
    L.salvox_probe_prmt_rate.argtypes = []
    L.salvox_probe_prmt_rate.restype = _dbl


def check(rc):
    """Maps a C-ABI status to the reference's exception classes."""
    if rc == SALVOX_OK:
        return
    msg = load().salvox_last_error().decode(errors="replace")
    if rc == SALVOX_EINVAL:
        raise ValueError(msg)  # std::invalid_argument (pybind11 maps it to ValueError)
    if rc == SALVOX_EUNSUPPORTED:
        raise NotImplementedError(msg)
    if rc == SALVOX_ECUDA:
        raise SalvoxCudaError(msg)
    raise RuntimeError(msg)


class Context:
    """Owns one salvox_ctx (device streams + buffers)."""

    def __init__(self, device: int = 0):
        self._h = _vp()
        check(load().salvox_ctx_create(int(device), C.byref(self._h)))
        self.device = device

    @property
    def handle(self):
        return self._h

    def set_stream(self, stream_ptr):
        check(load().salvox_ctx_set_stream(self._h, _vp(stream_ptr) if stream_ptr else None))

    def wait_stream(self, stream_ptr):
        """Orders this context's stream after the work queued on `stream_ptr`."""
        check(load().salvox_ctx_wait_stream(self._h, _vp(stream_ptr)))

    def after_torch(self, *tensors):
        """Device-tensor entry points read torch tensors that torch's current stream
        may still be producing (.contiguous(), non_blocking copies, torch.cat, ...):
        order the context's stream after it (no-op when the context is bound to it
        or no tensor is on the GPU)."""
        dev = next((t.device for t in tensors if t is not None and getattr(t, "is_cuda", False)),
                   None)
        if dev is None:
            return
        import torch

        self.wait_stream(torch.cuda.current_stream(dev).cuda_stream)

    def launch_count(self) -> int:
        out = C.c_uint64(0)
        check(load().salvox_ctx_launch_count(self._h, C.byref(out)))
        return int(out.value)

    def set_profiling(self, on: bool):
        check(load().salvox_ctx_set_profiling(self._h, 1 if on else 0))

    def kernel_time(self):
        """(kb_kernel ms total, launches, algorithmic updates) since set_profiling(True)."""
        ms, n, u = C.c_double(0), C.c_int64(0), C.c_double(0)
        check(load().salvox_ctx_kernel_time(self._h, C.byref(ms), C.byref(n), C.byref(u)))
        return ms.value, n.value, u.value

    def probe_smem_peak(self, iters: int = 64):
        """(LDS.U8+ATOMS pair rate, LDS-only rate, ATOMS-only rate) per second."""
        a, b, c = C.c_double(0), C.c_double(0), C.c_double(0)
        check(load().salvox_probe_smem_peak(self._h, int(iters), C.byref(a), C.byref(b),
                                            C.byref(c)))
        return a.value, b.value, c.value

    def probe_prmt_rate(self):
        """ATOMS rate of kb_quad_kernel's walk minus its bin loads (last probe call)."""
        return float(load().salvox_probe_prmt_rate())

    def close(self):
        if self._h:
            load().salvox_ctx_destroy(self._h)
            self._h = _vp()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


_default = {}


def default_context(device: int | None = None) -> Context:
    """Process-global context per device (the reference's free functions are stateless)."""
    if device is None:
        device = int(os.environ.get("LOCAL_RANK", "0")) if "LOCAL_RANK" in os.environ else 0
    with _lock:
        ctx = _default.get(device)
    if ctx is None:
        ctx = Context(device)
        with _lock:
            _default[device] = ctx
    return ctx


def ptr(a: np.ndarray):
    return a.ctypes.data_as(_vp) if a is not None else None
