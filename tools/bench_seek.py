"""Seed-grid detector timings on the BASELINE configs (device-resident volumes).

  C1: 128^3 PET-like phantom, 16 bins, scales 3..15, lattice 8, octant ascent
      (4,096 trajectories) and shift (53,248 seeds)
  C3: 256x256x160 MR phantom, 64 bins, shift, lattice 16 x scales {8, 12}
  C5: batch of 64 x 128^3 C1-style volumes (rng_seed 1310+i, centre jittered by
      Rng(i)), octant, volumes data-parallel (one rank here)
  PAPER PET / MR: ABMSOD (the paper's GPU workload) on the
      paper's shapes: 128x128x34 with 400 random seeds (16 bins) and 256x256x176
      with 700 random seeds (64 bins), seed windows isotropic r = 8 -- the paper
      reports 4.1 s and 7.8 s per volume on a Tesla C2050
Prints one JSON object per config; --cpu adds the oracle's time on all host cores,
--ref the reference's OWN detect() (oracle/_ref, its parallel_for on all host
cores; octant does not exist in the reference).
"""
import argparse
import ctypes as C
import json
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_1310_6736_b200 import _lib, api  # noqa: E402
from paper_1310_6736_b200._lib import Context  # noqa: E402
from tests import phantoms  # noqa: E402

C1_SCALES = [float(s) for s in range(3, 16)]


def c5_specs(n):
    specs = []
    for i in range(n):
        z = i  # splitmix64 jitter in [-8, 8] per axis from Rng(i)
        jit = []
        for _ in range(3):
            z = (z + 0x9E3779B97F4A7C15) & 0xFFFFFFFFFFFFFFFF
            t = z
            t = ((t ^ (t >> 30)) * 0xBF58476D1CE4E5B9) & 0xFFFFFFFFFFFFFFFF
            t = ((t ^ (t >> 27)) * 0x94D049BB133111EB) & 0xFFFFFFFFFFFFFFFF
            t ^= t >> 31
            jit.append(float((t >> 11) * 2.0**-53 * 16.0 - 8.0))
        specs.append(phantoms.config_c1(seed=1310 + i, jitter=jit))
    return specs


def time_batch(ctx, stream, d_vols, batch, shape, window, method, scales, spacing, steps=3,
               **extra):
    nz, ny, nx = shape
    iw = _lib.Window(window[0], window[1], window[2], 0)
    P, keep = api._detect_params(method, seed_spacing=spacing, scales=scales, k=20,
                                 dedupe_radius=5.0, **extra)
    out = np.empty(batch * 20, _lib.DET_DTYPE)
    n_out = np.zeros(batch, np.int64)
    visits = C.c_uint64(0)

    def run():
        _lib.check(_lib.load().salvox_detect_batch_device(
            ctx.handle, C.c_void_p(d_vols.data_ptr()), batch, nx, ny, nz, C.byref(iw), C.byref(P),
            out.ctypes.data_as(C.c_void_p), 20, n_out.ctypes.data_as(C.c_void_p), C.byref(visits)))

    run()
    ts = []
    for _ in range(steps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        run()
        e1.record(stream)
        e1.synchronize()
        ts.append(e0.elapsed_time(e1))
    del keep
    return float(np.mean(ts)), int(n_out.sum())


def ref_ms(vol, low, high, bins, **kw):
    """The reference's own detect() (oracle/_ref) on all host cores, best of 2."""
    from oracle import ref as R
    best = float("inf")
    for _ in range(2):
        t0 = time.perf_counter()
        R.detect(vol, low, high, bins, workers=os.cpu_count() or 1, **kw)
        best = min(best, time.perf_counter() - t0)
    return best * 1e3


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--cpu", action="store_true")
    ap.add_argument("--ref", action="store_true")
    ap.add_argument("--c5", type=int, default=64)
    ap.add_argument("--only", default="", help="substring filter on config names")
    args = ap.parse_args()
    ctx = Context(0)
    dev = torch.device("cuda", 0)
    st = torch.cuda.current_stream(dev)
    ctx.set_stream(st.cuda_stream)
    res = []
    v1, _ = api.make_phantom(phantoms.config_c1())
    d1 = torch.from_numpy(v1).to(dev)
    want = lambda name: args.only.lower() in name.lower()  # noqa: E731
    for method in ("octant", "shift") if want("C1") else ():
        ms, sel = time_batch(ctx, st, d1, 1, v1.shape, (0.0, 16.0, 16), method, C1_SCALES, 8.0)
        r = {"config": f"C1 {method}", "ms_per_volume": ms, "volumes_per_s": 1e3 / ms,
             "selected": sel}
        if args.cpu:
            from oracle import oracle as O
            t0 = time.perf_counter()
            O.detect(v1, 0.0, 16.0, 16, method=method, seed_spacing=8.0, scales=C1_SCALES,
                     top_k=20, dedupe_radius=5.0, workers=os.cpu_count() or 1)
            r["cpu_ms"] = (time.perf_counter() - t0) * 1e3
            r["cpu_cores"] = os.cpu_count()
        if args.ref and method == "shift":
            r["ref_ms"] = ref_ms(v1, 0.0, 16.0, 16, method="shift", seed_spacing=8.0,
                                 scales=C1_SCALES, top_k=20, dedupe_radius=5.0)
            r["ref_cores"] = os.cpu_count()
        res.append(r)
    if want("C3 shift"):
        v3, _ = api.make_phantom(phantoms.config_c3())
        d3 = torch.from_numpy(v3).to(dev)
        ms, sel = time_batch(ctx, st, d3, 1, v3.shape, (0.0, 64.0, 64), "shift", [8.0, 12.0], 16.0)
        r = {"config": "C3 shift", "ms_per_volume": ms, "volumes_per_s": 1e3 / ms,
             "selected": sel}
        if args.ref:
            r["ref_ms"] = ref_ms(v3, 0.0, 64.0, 64, method="shift", seed_spacing=16.0,
                                 scales=[8.0, 12.0], top_k=20, dedupe_radius=5.0)
            r["ref_cores"] = os.cpu_count()
        res.append(r)
    for name, spec, bins, n_seeds, paper_s in (("PAPER PET abmsod", phantoms.paper_pet(), 16, 400, 4.1),
                                               ("PAPER MR abmsod", phantoms.paper_mr(), 64, 700, 7.8)):
        if not want(name):
            continue
        vp, _ = api.make_phantom(spec)
        dp = torch.from_numpy(vp).to(dev)
        kw = dict(seed_mode="random", seed_count=n_seeds, rng_seed=1310)
        ms, sel = time_batch(ctx, st, dp, 1, vp.shape, (0.0, float(bins), bins), "abmsod", [8.0],
                             16.0, **kw)
        r = {"config": name, "shape": list(vp.shape), "seeds": n_seeds, "ms_per_volume": ms,
             "volumes_per_s": 1e3 / ms, "selected": sel, "paper_c2050_s_per_volume": paper_s}
        if args.cpu:
            from oracle import oracle as O
            t0 = time.perf_counter()
            O.detect(vp, 0.0, float(bins), bins, method="abmsod", seed_mode="random",
                     seed_count=n_seeds, rng_seed=1310, scales=[8.0], top_k=20, dedupe_radius=5.0,
                     workers=os.cpu_count() or 1)
            r["cpu_ms"] = (time.perf_counter() - t0) * 1e3
            r["cpu_cores"] = os.cpu_count()
        if args.ref:
            r["ref_ms"] = ref_ms(vp, 0.0, float(bins), bins, method="abmsod", seed_mode="random",
                                 seed_count=n_seeds, rng_seed=1310, scales=[8.0], top_k=20,
                                 dedupe_radius=5.0)
            r["ref_cores"] = os.cpu_count()
        res.append(r)
    if args.c5 > 0 and want("C5"):
        vols = np.stack([api.make_phantom(s)[0] for s in c5_specs(args.c5)])
        dv = torch.from_numpy(vols).to(dev)
        for method in ("octant", "shift"):
            ms, sel = time_batch(ctx, st, dv, args.c5, vols.shape[1:], (0.0, 16.0, 16), method,
                                 C1_SCALES, 8.0, steps=1)
            res.append({"config": f"C5 {method} batch x{args.c5}", "ms_per_batch": ms,
                        "volumes_per_s": args.c5 * 1e3 / ms, "selected": sel})
    for r in res:
        print(json.dumps(r))


if __name__ == "__main__":
    main()
