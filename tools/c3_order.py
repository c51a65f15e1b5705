"""Can a cheap first step predict C3 trajectory lengths? Runs the grid with
shift_max_iters = K (the probe), orders the seeds by the probe's outcome
(unconverged first, then by first-step length), and times the full grid in
that order vs plan order vs the oracle longest-first order."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1310_6736_b200 as sx  # noqa: E402
from tests import phantoms  # noqa: E402

v0, _ = sx.make_phantom(phantoms.config_c3())
vol = torch.from_numpy(v0).pin_memory().numpy()
pos, scl = sx.plan_seeds(vol.shape, mode="lattice", spacing=16.0, scales=[8.0, 12.0])
win = dict(window_low=0.0, window_high=64.0, bins=64, method="shift")
ctx = sx.Context(0)


def grid(idx, reps=7, **kw):
    best, out = 1e9, None
    for _ in range(reps):
        t0 = time.perf_counter()
        out, _ = sx.seek_records(vol, pos[idx], scales=scl[idx], ctx=ctx, **win, **kw)
        best = min(best, time.perf_counter() - t0)
    return best * 1e3, out


t_one, _ = grid(np.arange(1))
t_plan, full = grid(np.arange(len(pos)))
it = full["iterations"]
print(f"plan order {t_plan - t_one:.2f} ms")
t_or, _ = grid(np.argsort(-it, kind="stable"))
print(f"oracle longest-first {t_or - t_one:.2f} ms")
for K in (1, 2, 3):
    t_probe, pr = grid(np.arange(len(pos)), shift_max_iters=K)
    step = np.linalg.norm(pr["center"] - np.clip(pos, 0, None), axis=1)
    conv = (pr["flags"] & 1) != 0  # SALVOX_FLAG_CONVERGED
    key = np.where(conv, 0.0, 1.0)
    # unconverged first; within them longer cumulative movement first
    order = np.lexsort((-step, -key))
    t_ord, _ = grid(order)
    rc = np.corrcoef(np.argsort(np.argsort(-it, kind="stable")), np.argsort(order))[0, 1]
    print(f"K={K}: probe {t_probe - t_one:.2f} ms, predicted order {t_ord - t_one:.2f} ms, "
          f"unconverged {int((~conv).sum())}, rank corr {rc:.2f}")
