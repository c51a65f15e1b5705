"""C1 octant seed grid (4,096 trajectories, scales 3..15): iteration histogram
from the device's own records, and salvox_ascent_seek timings of the whole
grid vs its longest trajectory alone vs the shortest (the fixed part), with a
pinned volume."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1310_6736_b200 as sx  # noqa: E402
from tests import phantoms  # noqa: E402

v0, _ = sx.make_phantom(phantoms.config_c1())
vol = torch.from_numpy(v0).pin_memory().numpy()
pos, _ = sx.plan_seeds(vol.shape, mode="lattice", spacing=8.0, scales=[3.0])
scales = list(range(3, 16))
ctx = sx.Context(0)


def run(idx, reps=7):
    best, out = 1e9, None
    for _ in range(reps):
        t0 = time.perf_counter()
        out, _ = sx.quadrant_seek(vol, pos[idx], scales, 0.0, 16.0, 16, ctx=ctx, octant=True)
        best = min(best, time.perf_counter() - t0)
    return best * 1e3, out


t_all, out = run(np.arange(len(pos)))
it = out["iterations"]
print(f"trajectories {len(it)}, iterations mean {it.mean():.2f} max {it.max()}")
print("histogram:", {int(k): int(v) for k, v in zip(*np.unique(it, return_counts=True))})
lo, hi = int(np.argmin(it)), int(np.argmax(it))
t_lo, _ = run(np.array([lo]))
t_hi, _ = run(np.array([hi]))
print(f"grid {t_all - t_lo:.2f} ms, longest alone {t_hi - t_lo:.2f} ms (fixed part {t_lo:.2f} ms)")
