"""C3 shift: time and voxel visits vs max_iters (where does the time go?)."""
import ctypes as C
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_1310_6736_b200 import _lib, api  # noqa: E402
from paper_1310_6736_b200._lib import Context  # noqa: E402
from tests import phantoms  # noqa: E402

ctx = Context(0)
dev = torch.device("cuda", 0)
st = torch.cuda.current_stream(dev)
ctx.set_stream(st.cuda_stream)
cfgs = {"C3": (phantoms.config_c3(), 64, [8.0, 12.0], 16.0),
        "C1": (phantoms.config_c1(), 16, [float(s) for s in range(3, 16)], 8.0)}
for name, (spec, bins, scales, spacing) in cfgs.items():
    vol, _ = api.make_phantom(spec)
    d = torch.from_numpy(vol).to(dev)
    nz, ny, nx = vol.shape
    for mi in (1, 2, 5, 50):
        iw = _lib.Window(0.0, float(bins), bins, 0)
        P, keep = api._detect_params("shift", seed_spacing=spacing, scales=scales, k=20,
                                     dedupe_radius=5.0, shift_max_iters=mi)
        out = np.empty(20, _lib.DET_DTYPE)
        n_out = np.zeros(1, np.int64)
        vis = C.c_uint64(0)

        def run():
            _lib.check(_lib.load().salvox_detect_batch_device(
                ctx.handle, C.c_void_p(d.data_ptr()), 1, nx, ny, nz, C.byref(iw), C.byref(P),
                out.ctypes.data_as(C.c_void_p), 20, n_out.ctypes.data_as(C.c_void_p),
                C.byref(vis)))
        run()
        vis.value = 0
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(st)
        run()
        e1.record(st)
        e1.synchronize()
        ms = e0.elapsed_time(e1)
        print(f"{name} max_iters={mi:3d}: {ms:8.2f} ms  visits {vis.value:.3e}  "
              f"{vis.value / ms / 1e6:.2f} Gvisits/s")
