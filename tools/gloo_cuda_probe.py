"""Functional probe: can gloo move CUDA tensors (all_gather, P2P) between two
processes on ONE GPU? Used only to smoke-test the N>1 host orchestration of
bench.py/sharding on a 1-GPU box (no timing)."""
import os
import torch
import torch.distributed as dist

dist.init_process_group("gloo")
r = dist.get_rank()
dev = torch.device("cuda", 0)
x = torch.full((4,), float(r), device=dev)
outs = [torch.empty_like(x) for _ in range(dist.get_world_size())]
dist.all_gather(outs, x)
peer = 1 - r
y = torch.empty_like(x)
ops = [dist.P2POp(dist.isend, x, peer), dist.P2POp(dist.irecv, y, peer)]
for w in dist.batch_isend_irecv(ops):
    w.wait()
print(r, [o.tolist() for o in outs], y.tolist(), flush=True)
dist.destroy_process_group()
