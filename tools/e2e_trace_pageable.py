"""SALVOX_E2E_TRACE=1 timeline of the exhaustive call with PAGEABLE host buffers
(numpy in, fresh numpy maps out: the copy-back form with pinned staging)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1310_6736_b200 as sx  # noqa: E402
from tests import phantoms  # noqa: E402

ctx = sx.Context(0)
vol = sx.make_phantom_device(phantoms.config_c2(), ctx=ctx)[0].cpu().numpy()
sc = [float(s) for s in range(3, 16)]
for i in range(3):
    t0 = time.perf_counter()
    r = sx.kadir_brady_exhaustive_records(vol, sc, 0.0, 32.0, 32, budget=10**13, ctx=ctx)
    print(f"call {i}: {(time.perf_counter() - t0) * 1e3:.2f} ms", flush=True)

# where the time outside the pipelined body goes
import ctypes as C  # noqa: E402
import numpy as np  # noqa: E402
from paper_1310_6736_b200 import _lib, api  # noqa: E402

lib = _lib.load()
nz, ny, nx = vol.shape
iw = api._window(0.0, 32.0, 32)
scd = np.ascontiguousarray(sc, np.float64)
for touched in (False, True):
    for i in range(3):
        score = np.empty(vol.shape, np.float32)
        best = np.empty(vol.shape, np.float32)
        mx = np.empty(600000, sx.MAX_DTYPE)
        if touched:
            score.fill(0)
            best.fill(0)
            mx.fill(0)
        n = C.c_int64(0)
        visits = C.c_uint64(0)
        t0 = time.perf_counter()
        _lib.check(lib.salvox_exhaustive(ctx.handle, _lib.ptr(vol), nx, ny, nz, C.byref(iw),
                                         _lib.ptr(scd), len(scd), 0, 10**13, _lib.ptr(score),
                                         _lib.ptr(best), _lib.ptr(mx), len(mx), C.byref(n),
                                         C.byref(visits)))
        print(f"raw C call (outputs {'pre-touched' if touched else 'fresh'}): "
              f"{(time.perf_counter() - t0) * 1e3:.2f} ms", flush=True)
