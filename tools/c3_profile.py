"""C3 shift seed grid: per-seed iteration counts (the device's own per-seed
records) and salvox_seek timings of the whole grid vs only its longest
trajectories (same starts), to tell a long-trajectory tail from throughput."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import paper_1310_6736_b200 as sx  # noqa: E402
from tests import phantoms  # noqa: E402

vol, _ = sx.make_phantom(phantoms.config_c3())
pos, scl = sx.plan_seeds(vol.shape, mode="lattice", spacing=16.0, scales=[8.0, 12.0])
win = dict(window_low=0.0, window_high=64.0, bins=64, method="shift")
ctx = sx.Context(0)


def run(idx, reps=3):
    best = 1e9
    for _ in range(reps):
        t0 = time.perf_counter()
        out, vis = sx.seek_records(vol, pos[idx], scales=scl[idx], ctx=ctx, **win)
        best = min(best, time.perf_counter() - t0)
    return best * 1e3, out, vis


allidx = np.arange(len(pos))
ms, out, vis = run(allidx)
it = out["iterations"]
print(f"seeds {len(it)}  iterations mean {it.mean():.2f} max {it.max()}  visits {vis}")
print("iterations histogram:", {int(k): int(v) for k, v in zip(*np.unique(it, return_counts=True))})
print(f"all seeds: {ms:.2f} ms (host call incl. upload)")
order = np.argsort(-it, kind="stable")
for n in (1, 16, 148, 592):
    m, _, _ = run(order[:n])
    print(f"longest {n:4d} seeds: {m:.2f} ms (iterations >= {it[order[n - 1]]})")
m, _, _ = run(order[-1:])
print(f"shortest 1 seed: {m:.2f} ms (upload + binning + launch: the fixed part)")
m, _, _ = run(order[len(order) // 2:])
print(f"shortest half: {m:.2f} ms")
for s in (8.0, 12.0):
    sel = np.where(scl == s)[0]
    m, _, _ = run(sel)
    print(f"scale {s}: {len(sel)} seeds {m:.2f} ms, mean iterations {it[sel].mean():.2f}")
