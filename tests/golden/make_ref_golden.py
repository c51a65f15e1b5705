"""Generates tests/golden/ref_*.npz from the REFERENCE ITSELF.

The reference's own sources are compiled here into oracle/_ref/libsalvox_ref.so
(`make -C oracle ref`; DESIGN.md §4 "Pinning") and run on fixed inputs. The
vectors it returns are frozen here so the GPU parity tests
(tests/test_gpu_reference.py) compare the device path with the reference's
own outputs on a box where /root/reference does not exist. Inputs are rebuilt
from the stored PhantomSpecs (bit-identical Rng on every side), so only specs
and outputs are stored. Run from the repo root (needs /root/reference):

    python tests/golden/make_ref_golden.py
"""
import json
import math
import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)

from oracle import ref as R  # noqa: E402
from tests import phantoms  # noqa: E402

WORKERS = os.cpu_count() or 1


def _oblique_spec():
    th = math.radians(30.0)
    rz = np.array([[math.cos(th), -math.sin(th), 0], [math.sin(th), math.cos(th), 0], [0, 0, 1]])
    return phantoms.ellipsoid_3d(rz @ np.diag([10.0, 7.0, 5.0]), 222, 64)


CASES = {
    # C2 (BASELINE configs[1]) exhaustive pass with all 13 scales on a 40^3 crop of
    # the C2 phantom around its r = 12 ball (crop faces exercise the OOB skips).
    "ref_exh_c2crop": dict(spec=phantoms.config_c2(), crop=[[160, 200], [70, 110], [108, 148]],
                           low=0.0, high=32.0, bins=32, scales=[float(s) for s in range(3, 16)]),
    # the reference's 2D exhaustive square fixture (test_pipeline.cpp:228-236)
    "ref_exh_square2d": dict(spec=phantoms.square_2d(64, 31.0, 31.0, 8, 64, 77), low=0.0,
                             high=64.0, bins=64, scales=[4.0, 6.0, 8.0, 10.0]),
    # shift detect + every seed's saliency_shift (test_pipeline.cpp:296-319 style)
    "ref_det_shift3d": dict(spec=phantoms.ball_3d(32, (16.0, 15.0, 14.0), 6.0, 7), low=0.0,
                            high=64.0, bins=64, method="shift", seed_spacing=8.0,
                            scales=[4.0, 6.0], top_k=8, dedupe_radius=4.0),
    # quadrant detect + every position's quadrant_seek_one (test_pipeline.cpp:356-379)
    "ref_det_quadrant2d": dict(spec=phantoms.square_2d(64, 31.0, 31.0, 8, 64, 77), low=0.0,
                               high=64.0, bins=64, method="quadrant", seed_spacing=16.0,
                               scales=[4.0, 6.0, 8.0, 10.0], top_k=5, dedupe_radius=5.0),
    # ABMSOD with traces on the oblique ellipsoid (test_seek.cpp:516-540 style)
    "ref_abmsod": dict(spec=_oblique_spec(), low=0.0, high=64.0, bins=64, radius=6.0,
                       seeds=[[31.5, 31.5, 31.5], [34.5, 29.5, 32.5], [25.5, 35.5, 28.5]]),
    # full-size seed-grid configs of BASELINE.json through the reference's detect()
    "ref_c3_shift": dict(spec=phantoms.config_c3(), low=0.0, high=64.0, bins=64, method="shift",
                         seed_spacing=16.0, scales=[8.0, 12.0], top_k=20, dedupe_radius=5.0),
    "ref_c1_shift": dict(spec=phantoms.config_c1(), low=0.0, high=16.0, bins=16, method="shift",
                         seed_spacing=8.0, scales=[float(s) for s in range(3, 16)], top_k=20,
                         dedupe_radius=5.0),
}


def crop(vol, box):
    (x0, x1), (y0, y1), (z0, z1) = box
    return np.ascontiguousarray(vol[z0:z1, y0:y1, x0:x1])


def main(only=None):
    meta = {}
    old = os.path.join(HERE, "ref_cases.json")
    if os.path.exists(old):
        meta = json.load(open(old))
    for name, c in CASES.items():
        if only and name not in only:
            meta.setdefault(name, c)
            continue
        t0 = time.time()
        vol, _ = R.make_phantom(c["spec"])
        if "crop" in c:
            vol = crop(vol, c["crop"])
        out = {}
        if name.startswith("ref_exh"):
            s, b, m, v = R.exhaustive(vol, c["low"], c["high"], c["bins"], c["scales"],
                                      budget=10**13)
            nz, ny, nx = vol.shape
            lin = (m[:, 0] + nx * (m[:, 1] + ny * m[:, 2])).astype(np.int64)
            out = dict(score=s, best=b, max_lin=lin, max_score=m[:, 3], max_scale=m[:, 4],
                       visits=np.uint64(v))
        elif name == "ref_abmsod":
            dets, traces, visits = [], [], []
            for sd in c["seeds"]:
                d, tr, v = R.abmsod_run(vol, c["low"], c["high"], c["bins"], sd,
                                        radius=c["radius"], trace=True)
                dets.append(d)
                traces.append(tr)
                visits.append(v)
            out = dict(dets=np.frombuffer(np.array(dets).tobytes(), np.uint8),
                       trace_len=np.array([len(t) for t in traces], np.int32),
                       traces=np.frombuffer(np.concatenate(traces).tobytes(), np.uint8),
                       visits=np.array(visits, np.uint64))
        else:
            sel, v = R.detect(vol, c["low"], c["high"], c["bins"], method=c["method"],
                              seed_spacing=c["seed_spacing"], scales=c["scales"],
                              top_k=c["top_k"], dedupe_radius=c["dedupe_radius"],
                              workers=WORKERS)
            out = dict(selected=np.frombuffer(sel.tobytes(), np.uint8), visits=np.uint64(v))
            if c["method"] == "shift" and vol.size <= 64**3:
                pos, ss = R.plan_seeds(vol.shape, spacing=c["seed_spacing"], scales=c["scales"])
                per, pv = [], 0
                for i, (p, s) in enumerate(zip(pos, ss)):
                    d, vv = R.saliency_shift(vol, c["low"], c["high"], c["bins"], p, [s, s, s])
                    d["seed_index"] = i  # detect() sets it (pipeline.cpp:369)
                    per.append(d)
                    pv += vv
                out["per_seed"] = np.frombuffer(np.array(per).tobytes(), np.uint8)
                out["per_seed_visits"] = np.uint64(pv)
            if c["method"] == "quadrant":
                pos, _ = R.plan_seeds(vol.shape, spacing=c["seed_spacing"], scales=c["scales"])
                rows = []
                for p in pos[:: len(c["scales"])]:
                    r, vv = R.quadrant_seek_one(vol, c["low"], c["high"], c["bins"], p,
                                                [int(round(s)) for s in c["scales"]])
                    rows.append([r.position[0], r.position[1], r.best_scale, r.iterations,
                                 r.entropy_bits, r.converged, r.degenerate, vv])
                out["trajectories"] = np.array(rows, np.float64)
        np.savez_compressed(os.path.join(HERE, name + ".npz"), **out)
        meta[name] = c
        print(f"{name}: {time.time() - t0:.1f} s", flush=True)
    with open(old, "w") as f:
        json.dump(meta, f, indent=1, sort_keys=True)


if __name__ == "__main__":
    main(set(sys.argv[1:]) or None)
