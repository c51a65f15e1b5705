import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_1310_6736_b200 as sx
from oracle import oracle as O
from tests.test_gpu_fuzz import _case
np.set_printoptions(precision=17)
for seed in range(12):
    rng = np.random.default_rng(1000 + seed)
    vol, two_d, bins = _case(rng)
    methods = ["shift", "abmsod"] + (["quadrant"] if two_d else ["octant"])
    method = methods[seed % len(methods)]
    lo, hi = float(np.floor(vol.min())), float(np.ceil(vol.max()) + 1.0)
    scales = sorted({float(s) for s in rng.integers(2, 7, size=int(rng.integers(1, 4)))})
    kw = dict(seed_spacing=float(rng.integers(4, 9)), scales=scales, k=int(rng.integers(3, 9)),
              dedupe_radius=float(rng.uniform(2.0, 6.0)))
    extra = {}
    if method == "shift":
        extra = dict(shift_hist_kernel=str(rng.choice(["identity", "epanechnikov", "gaussian"])),
                     shift_step_kernel=str(rng.choice(["identity", "gaussian"])),
                     shift_max_iters=int(rng.integers(1, 30)))
    if rng.random() < 0.3:
        extra.update(seed_mode="random", seed_count=int(rng.integers(5, 40)), rng_seed=int(rng.integers(0, 1000)))
    sel, seeds, visits = sx.detect_records(vol, method, window_low=lo, window_high=hi, bins=bins, per_seed=True, **kw, **extra)
    okw = dict(kw); okw["top_k"] = okw.pop("k")
    O.set_log_mode(7)
    rsel, rseeds, rv = O.detect(vol, lo, hi, bins, method=method, **okw, **extra)
    O.set_log_mode(0)
    ok = seeds.tobytes() == rseeds.tobytes()
    print(seed, method, vol.shape, bins, scales, kw, extra, "OK" if ok else "MISMATCH", visits == rv)
    if not ok:
        nbad = 0
        for i in range(len(seeds)):
            g, r = seeds[i], rseeds[i]
            diff = [f for f in ["center", "H", "iterations", "flags", "entropy_bits", "pdf_diff", "bhattacharyya", "seed_index"] if not np.array_equal(g[f], r[f])]
            if diff:
                nbad += 1
                if nbad <= 2:
                    print("   seed", i, diff, "it", g["iterations"], r["iterations"], "fl", g["flags"], r["flags"])
                    for f in diff[:3]:
                        print("     ", f, g[f], r[f])
        print("   bad", nbad, "of", len(seeds))
