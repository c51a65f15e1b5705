import time, numpy as np, torch, sys
sys.path.insert(0, '.')
import paper_1310_6736_b200 as sx
from tests import phantoms
ctx = sx.Context(0)
vol = sx.make_phantom_device(phantoms.config_c2(), ctx=ctx)[0].cpu().numpy()
sc = [float(s) for s in range(3, 16)]
for k in ["identity", "epanechnikov"]:
    ts = []
    for i in range(3):
        t0 = time.perf_counter()
        r = sx.kadir_brady_exhaustive_records(vol, sc, 0.0, 32.0, 32, kernel=k, budget=10**13, ctx=ctx)
        ts.append(time.perf_counter() - t0)
    print(k, "C2 host-buffer call ms", [round(t * 1e3, 1) for t in ts], "maxima", len(r[2]), flush=True)
