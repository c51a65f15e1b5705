"""Functional check of the multi-rank exhaustive orchestration on ONE GPU (gloo,
ranks share the device; no timing): exhaustive_sharded's device path -- owned
planes only, boundary-plane exchange, device all-gather + merge -- must give the
single-call maps and maxima byte for byte. Run under torchrun with 2-4 ranks."""
import os
import sys

import numpy as np
import torch
import torch.distributed as dist

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1310_6736_b200 import api, sharding  # noqa: E402
from paper_1310_6736_b200._lib import Context  # noqa: E402
from tests import phantoms  # noqa: E402

dist.init_process_group("gloo")
rank, world = dist.get_rank(), dist.get_world_size()
dev = torch.device("cuda", 0)
torch.cuda.set_device(dev)
ctx = Context(0)
spec = phantoms.ball_3d(48, (20.0, 25.0, 23.0), 9.0, 31, levels=32,
                        background={"type": "gaussian", "mean": 8.0, "sigma": 2.0})
vol, _ = api.make_phantom(spec)
scales = [3.0, 4.0, 5.0, 6.0, 7.0]
s, b, (z0, z1), merged, _ = sharding.exhaustive_sharded(vol, scales, 0.0, 32.0, 32, budget=10**12,
                                                        device=dev, ctx=ctx)
ref_s, ref_b, ref_m, _ = api.kadir_brady_exhaustive_slab(vol, vol.shape[0], 0, 0, vol.shape[0],
                                                         scales, 0.0, 32.0, 32, budget=10**12,
                                                         ctx=ctx)
ok = (np.array_equal(s, ref_s[z0:z1]) and np.array_equal(b, ref_b[z0:z1])
      and np.array_equal(merged, ref_m))
print(f"rank {rank}/{world} planes [{z0},{z1}) maxima {len(merged)} == single call: {ok}", flush=True)
dist.barrier()
dist.destroy_process_group()
sys.exit(0 if ok else 1)
