import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_1310_6736_b200 as sx
from oracle import oracle as O
from tests import phantoms
np.set_printoptions(precision=17)
axes = phantoms.rot_z(45.0) @ np.diag([9.0, 4.0, 4.0])
vol, _ = O.make_phantom(phantoms.ellipsoid_3d(axes, 333, 48))
kw = dict(seed_spacing=12.0, scales=[5.0, 7.0], k=5, dedupe_radius=5.0)
sel, seeds, visits = sx.detect_records(vol, "abmsod", window_low=0, window_high=64, bins=64, per_seed=True, **kw)
O.set_log_mode(7)
rsel, rseeds, rv = O.detect(vol, 0, 64, 64, method="abmsod", seed_spacing=12.0, scales=[5.0, 7.0], top_k=5, dedupe_radius=5.0)
pos, sc = sx.plan_seeds(vol.shape, spacing=12.0, scales=[5.0, 7.0])
bad = 0
for i in range(len(seeds)):
    g, r = seeds[i], rseeds[i]
    diff = [f for f in ["center", "H", "iterations", "flags", "entropy_bits", "pdf_diff", "bhattacharyya", "seed_index"] if not np.array_equal(g[f], r[f])]
    if diff:
        bad += 1
        if bad <= 4:
            print(i, pos[i], sc[i], diff, g["iterations"], r["iterations"], g["flags"], r["flags"])
            print("  g", g["center"], g["H"][:3]); print("  r", r["center"], r["H"][:3])
            raw, tr, _ = sx.abmsod_records(vol, [pos[i]], radius=sc[i], window_low=0, window_high=64, trace=True)
            rr, rtr, _ = O.abmsod_run(vol, 0, 64, 64, pos[i], radius=sc[i], trace=True)
            print("  raw==ref", np.array_equal(raw[0]["center"], rr["center"]), "raw==detect", np.array_equal(raw[0]["center"], g["center"]))
print("bad", bad, "of", len(seeds), visits, rv)
