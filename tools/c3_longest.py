"""Latency of ONE long C3 trajectory (the critical path of the seed grid): the
longest seed (50 iterations) alone vs the shortest seed alone (the fixed part:
upload + binning + launch); prints their difference in ms."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import paper_1310_6736_b200 as sx  # noqa: E402
from tests import phantoms  # noqa: E402

import torch  # noqa: E402

v0, _ = sx.make_phantom(phantoms.config_c3())
vol = torch.from_numpy(v0).pin_memory().numpy()  # pinned: a fast, steady upload
pos, scl = sx.plan_seeds(vol.shape, mode="lattice", spacing=16.0, scales=[8.0, 12.0])
win = dict(window_low=0.0, window_high=64.0, bins=64, method="shift")
ctx = sx.Context(0)
out, _ = sx.seek_records(vol, pos, scales=scl, ctx=ctx, **win)
it = out["iterations"]
lo, hi = int(np.argmin(it)), int(np.argmax(it))


def t(i, reps=15):
    best = 1e9
    for _ in range(reps):
        t0 = time.perf_counter()
        sx.seek_records(vol, pos[i:i + 1], scales=scl[i:i + 1], ctx=ctx, **win)
        best = min(best, time.perf_counter() - t0)
    return best * 1e3


a, b = t(hi), t(lo)
print(f"longest seed ({it[hi]} iterations, scale {scl[hi]}): {a:.2f} ms; shortest: {b:.2f} ms; "
      f"trajectory latency {a - b:.2f} ms")

# the whole grid in plan order vs sorted longest-trajectory-first (an oracle ordering:
# the upper bound of what predicting trajectory lengths could buy)
order = np.argsort(-it, kind="stable")


def grid(idx, reps=7):
    best = 1e9
    for _ in range(reps):
        t0 = time.perf_counter()
        sx.seek_records(vol, pos[idx], scales=scl[idx], ctx=ctx, **win)
        best = min(best, time.perf_counter() - t0)
    return best * 1e3


print(f"grid, plan order: {grid(np.arange(len(pos))) - b:.2f} ms; longest-first: "
      f"{grid(order) - b:.2f} ms (fixed part removed)")
