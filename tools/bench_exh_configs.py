"""Exhaustive-pass throughput beyond the bench's C2 line: device-resident scores
(exhaustive_slab_scores on a CUDA tensor, maps only), CUDA-event timed, best of
3 after a warm-up. Configs: C1 (128^3, 16 bins), C2 identity and Epanechnikov,
C2 at 64 bins (the 65-bin kb_kernel path), a 2D 2048^2 image (kb_kernel 2D).
Prints one JSON object."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1310_6736_b200 as sx  # noqa: E402
from paper_1310_6736_b200 import api  # noqa: E402
from tests import phantoms  # noqa: E402

SC = [float(s) for s in range(3, 16)]


def run(vol, low, high, bins, scales, kernel="identity"):
    dev = torch.device("cuda", 0)
    st = torch.cuda.current_stream(dev)
    ctx = sx.Context(0)
    ctx.set_stream(st.cuda_stream)
    d = torch.from_numpy(vol).to(dev)
    nz = vol.shape[0]
    kw = dict(kernel=kernel, budget=10**15, ctx=ctx)
    api.exhaustive_slab_scores(d, nz, 0, 0, nz, scales, low, high, bins, **kw)
    best = 1e9
    for _ in range(3):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(st)
        api.exhaustive_slab_scores(d, nz, 0, 0, nz, scales, low, high, bins, **kw)
        e1.record(st)
        e1.synchronize()
        best = min(best, e0.elapsed_time(e1))
    ctx.close()
    evals = vol.size * len(scales)
    return {"ms": best, "evals_per_s": evals / (best * 1e-3), "voxels": int(vol.size),
            "scales": len(scales), "bins": bins, "kernel": kernel}


def main():
    res = {}
    c1, _ = api.make_phantom(phantoms.config_c1())
    res["C1 128^3 16 bins"] = run(c1, 0.0, 16.0, 16, SC)
    c2 = sx.make_phantom_device(phantoms.config_c2())[0].cpu().numpy()
    res["C2 256^3 32 bins"] = run(c2, 0.0, 32.0, 32, SC)
    res["C2 256^3 32 bins Epanechnikov"] = run(c2, 0.0, 32.0, 32, SC, kernel="epanechnikov")
    res["C2 256^3 64 bins"] = run(c2, 0.0, 32.0, 64, SC)
    rng = np.random.default_rng(7)
    img = np.clip(rng.normal(16.0, 5.0, size=(1, 2048, 2048)), 0, 31.9).astype(np.float32)
    res["2D 2048^2 32 bins"] = run(img, 0.0, 32.0, 32, SC)
    print(json.dumps(res))


if __name__ == "__main__":
    main()
