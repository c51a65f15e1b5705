import sys, time, numpy as np, torch
sys.path.insert(0, '.')
import paper_1310_6736_b200 as sx
from tests import phantoms
ctx = sx.Context(0)
vol = sx.make_phantom_device(phantoms.config_c2(), ctx=ctx)[0].cpu().numpy()
vp = torch.from_numpy(vol).pin_memory().numpy()
outs = tuple(torch.empty(vol.shape, dtype=torch.float32).pin_memory().numpy() for _ in range(2))
mx = torch.empty((vol.size // 24 + 4096) * sx.MAX_DTYPE.itemsize, dtype=torch.uint8).pin_memory().numpy().view(sx.MAX_DTYPE)
sc = [float(s) for s in range(3, 16)]
ts = []
for i in range(40):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    sx.kadir_brady_exhaustive_slab(vp, 256, 0, 0, 256, sc, 0.0, 32.0, 32, budget=10**13, ctx=ctx, out=outs, maxima_out=mx)
    ts.append((time.perf_counter() - t0) * 1e3)
ts = np.array(ts[3:])
print("e2e ms: mean %.2f median %.2f min %.2f max %.2f" % (ts.mean(), np.median(ts), ts.min(), ts.max()))
print(" ".join("%.1f" % t for t in ts))
