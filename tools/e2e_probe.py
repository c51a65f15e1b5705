import sys, os, time
sys.path.insert(0, '/root/repo')
os.chdir('/root/repo')
import numpy as np, torch
import paper_1310_6736_b200 as sx
from paper_1310_6736_b200 import api
from tests import phantoms
vol, _ = api.make_phantom(phantoms.config_c2())
ctx = sx.Context(0)
vp = torch.from_numpy(vol).pin_memory().numpy()
o1 = torch.empty(vol.shape, dtype=torch.float32).pin_memory().numpy()
o2 = torch.empty(vol.shape, dtype=torch.float32).pin_memory().numpy()
sc = [float(s) for s in range(3, 16)]
for i in range(4):
    t0 = time.perf_counter()
    r = api.kadir_brady_exhaustive_slab(vp, 256, 0, 0, 256, sc, 0, 32, 32, budget=10**12, ctx=ctx, out=(o1, o2))
    t1 = time.perf_counter()
    print("slab call ms", (t1 - t0) * 1e3, len(r[2]))
# plan cost: tiny volume
small = np.zeros((40, 40, 40), np.float32)
for i in range(3):
    t0 = time.perf_counter()
    api.kadir_brady_exhaustive_slab(small, 40, 0, 0, 40, sc, 0, 32, 32, budget=10**12, ctx=ctx)
    print("small call ms", (time.perf_counter() - t0) * 1e3)
