"""Times the C3 seed-grid detector (bench.py's secondary line) on its own."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402
from paper_1310_6736_b200._lib import Context  # noqa: E402

ctx = Context(0)
dev = torch.device("cuda", 0)
st = torch.cuda.current_stream(dev)
ctx.set_stream(st.cuda_stream)
fl = torch.empty(256 * 2**20, dtype=torch.uint8, device=dev)
print(bench.bench_seed_grid(ctx, dev, st, fl, steps=3))
