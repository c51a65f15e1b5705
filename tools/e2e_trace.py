"""Device timeline of the host-buffer exhaustive call at the bench workload (C2,
256^3, pinned volume and maps): SALVOX_E2E_TRACE=1 makes the library print one
line per mark to stderr; also times the same call's host->device volume copy
alone and the whole call, for the e2e budget in DESIGN.md."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1310_6736_b200 as sx  # noqa: E402
from tests import phantoms  # noqa: E402

SCALES = [float(s) for s in range(3, 16)]


def main():
    spec = phantoms.config_c2()
    ctx = sx.Context(0)
    vol = sx.make_phantom_device(spec, ctx=ctx)[0].cpu().numpy()
    nz, ny, nx = vol.shape
    vp = torch.from_numpy(vol).pin_memory()
    outs = tuple(torch.empty(vol.shape, dtype=torch.float32).pin_memory().numpy() for _ in range(2))
    mx = torch.empty((vol.size // 24 + 4096) * sx.MAX_DTYPE.itemsize,
                     dtype=torch.uint8).pin_memory().numpy().view(sx.MAX_DTYPE)
    d = torch.empty(vol.shape, dtype=torch.float32, device="cuda")
    for _ in range(3):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        d.copy_(vp, non_blocking=True)
        torch.cuda.synchronize()
        h2d = (time.perf_counter() - t0) * 1e3
    print(f"H2D of the volume alone: {h2d:.3f} ms ({vol.nbytes / h2d / 1e6:.1f} GB/s)", flush=True)
    for i in range(4):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        r = sx.kadir_brady_exhaustive_slab(vp.numpy(), nz, 0, 0, nz, SCALES, 0.0, 32.0, 32,
                                           budget=10**13, ctx=ctx, out=outs, maxima_out=mx)
        t1 = time.perf_counter()
        print(f"call {i}: {(t1 - t0) * 1e3:.3f} ms, {len(r[2])} maxima", flush=True)


if __name__ == "__main__":
    main()
