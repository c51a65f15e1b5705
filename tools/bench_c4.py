"""C4 (BASELINE.json configs[3]): the 512^3 exhaustive pass on one B200, whole
volume and as the z-slabs a 2/4/8-GPU run would give each rank (the slab
passes run one after another here -- per-rank compute, not a multi-GPU
measurement; the driver's SCALE run measures that). Device-resident, CUDA events."""
import ctypes as C
import json
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_1310_6736_b200 import _lib, api, sharding  # noqa: E402
from paper_1310_6736_b200._lib import Context  # noqa: E402
from tests import phantoms  # noqa: E402

SCALES = [float(s) for s in range(3, 16)]
ctx = Context(0)
dev = torch.device("cuda", 0)
st = torch.cuda.current_stream(dev)
ctx.set_stream(st.cuda_stream)
vol, _ = api.make_phantom(phantoms.config_c4())
nz, ny, nx = vol.shape
d_vol = torch.from_numpy(vol).to(dev)
sc = np.asarray(SCALES, np.float64)
iw = _lib.Window(0.0, 32.0, 32, 0)
R = sharding.halo_radius(SCALES)
evals = float(nx * ny * nz * len(SCALES))
res = {"config": "C4 512^3 exhaustive, 32 bins, scales 3..15", "evals_per_pass": evals}
for world in (1, 2, 4, 8):
    times = []
    for rank in range(world):
        z0, z1, zs0, zs1 = sharding.slab_bounds(nz, world, rank, R)
        d_slab = d_vol[zs0:zs1].contiguous()
        d_score = torch.empty((z1 - z0, ny, nx), dtype=torch.float32, device=dev)
        d_best = torch.empty_like(d_score)
        n = C.c_int64(0)

        def run():
            _lib.check(_lib.load().salvox_exhaustive_slab_device(
                ctx.handle, C.c_void_p(d_slab.data_ptr()), nx, ny, nz, zs0, zs1, z0, z1,
                C.byref(iw), sc.ctypes.data_as(C.c_void_p), len(sc), 0, 10**15,
                C.c_void_p(d_score.data_ptr()), C.c_void_p(d_best.data_ptr()), C.byref(n)))
        run()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(st)
        run()
        e1.record(st)
        e1.synchronize()
        times.append(e0.elapsed_time(e1))
    res[f"slab_ms_x{world}"] = {"max": max(times), "min": min(times),
                                "implied_evals_per_s": evals / (max(times) * 1e-3)}
    # the exchange form (what bench.py runs at N > 1): owned planes only
    # (salvox_exhaustive_slab_scores), the two neighbour planes passed in (as the
    # NCCL exchange delivers them), then maxima left on the device for the
    # all-gather + device merge (not included: ~1 ms over NVLink at N = 8)
    if world > 1:
        times = []
        for rank in range(world):
            z0, z1, zs0, zs1 = sharding.slab_bounds(nz, world, rank, R)
            d_slab = d_vol[zs0:zs1].contiguous()
            d_score = torch.empty((z1 - z0, ny, nx), dtype=torch.float32, device=dev)
            d_best = torch.empty_like(d_score)
            below = d_vol[max(z0 - 1, 0)].contiguous()  # stand-ins with the right shape
            above = d_vol[min(z1, nz - 1)].contiguous()

            def run_x():
                api.exhaustive_slab_scores(d_slab, nz, zs0, z0, z1, SCALES, 0.0, 32.0, 32,
                                           budget=10**15, ctx=ctx, out=(d_score, d_best))
                api.exhaustive_slab_maxima(below if z0 > 0 else None, above if z1 < nz else None,
                                           ctx=ctx, on_device=True)
            run_x()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(st)
            run_x()
            e1.record(st)
            e1.synchronize()
            times.append(e0.elapsed_time(e1))
        res[f"exchange_slab_ms_x{world}"] = {"max": max(times), "min": min(times),
                                             "implied_evals_per_s": evals / (max(times) * 1e-3)}
print(json.dumps(res))
