import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_1310_6736_b200 as sx
from oracle import oracle as O
from tests import phantoms
np.set_printoptions(precision=17)
axes = phantoms.rot_z(45.0) @ np.diag([9.0, 4.0, 4.0])
vol, _ = O.make_phantom(phantoms.ellipsoid_3d(axes, 222, 64))
c = np.array([31.5] * 3)
seeds = [c, c + [2.0, 1.0, 0.0], c + [-5.0, 3.5, 2.25], [0.0, 0.0, 0.0], [63.0, 10.0, 31.5]]
gpu, traces, visits = sx.abmsod_records(vol, seeds, radius=6.0, window_low=0, window_high=64, trace=True)
O.set_log_mode(7)
for i, s in enumerate(seeds):
    r, rt, v = O.abmsod_run(vol, 0, 64, 64, s, radius=6.0, trace=True)
    print("seed", i, "iters", gpu[i]["iterations"], r["iterations"], "flags", gpu[i]["flags"], r["flags"])
    for k in range(min(len(traces[i]), len(rt))):
        a, b = traces[i][k], rt[k]
        same_p = np.array_equal(a["position"], b["position"])
        same_h = np.array_equal(a["H"], b["H"])
        print("  it", k, "pos", same_p, "H", same_h, "bhat", a["bhattacharyya"] == b["bhattacharyya"])
        if not (same_p and same_h):
            print("   gpu pos", a["position"], "\n   ref pos", b["position"])
            print("   gpu H", a["H"], "\n   ref H", b["H"])
            break
# direct eigen test via bandwidth_from_moment C-ABI (host) vs oracle
rng = np.random.default_rng(3)
