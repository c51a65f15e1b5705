"""Multi-GPU z-slab sharding of the exhaustive pass.

One process per GPU (torch.distributed, NCCL over NVLink on the box; gloo in the
CPU tests). Rank g owns planes [z_g, z_{g+1}); it bins the planes
[z_g - R - 1, z_{g+1} + R + 1) (halo R = max scale + 1), scores its owned planes
plus one neighbour plane each side (so strict 26-neighbour maxima are decided
locally, no score exchange) and selects its maxima. The only collective is ONE
all-gather of the per-slab maxima records (fixed-capacity tensors: counts first,
then the padded records), followed by a merge in the reference's stable order
(score descending, linear index ascending -- pipeline.cpp:163-164), so every
N-GPU result is byte-identical to the 1-GPU one.
"""
from __future__ import annotations

import math

import numpy as np

from ._lib import MAX_DTYPE


def halo_radius(scales) -> int:
    """R = floor(max radius) with radii {s-1, s, s+1} (pipeline.cpp:76-84)."""
    return int(math.floor(max(scales) + 1.0))


def slab_bounds(nz: int, world: int, rank: int, R: int):
    """Owned planes [z0, z1) and the planes [zs0, zs1) the rank must read."""
    z0 = nz * rank // world
    z1 = nz * (rank + 1) // world
    zs0 = max(0, z0 - R - 1)
    zs1 = min(nz, z1 + R + 1)
    return z0, z1, zs0, zs1


def merge_maxima(parts) -> np.ndarray:
    """Concatenate per-slab maxima and restore the reference's stable_sort order."""
    parts = [p for p in parts if len(p)]
    if not parts:
        return np.zeros(0, MAX_DTYPE)
    m = np.concatenate(parts)
    order = np.lexsort((m["linear_index"], -m["score"]))
    return m[order]


def _pack(maxima: np.ndarray) -> np.ndarray:
    out = np.zeros((len(maxima), 6), np.float64)
    if len(maxima):
        out[:, 0:3] = maxima["position"]
        out[:, 3] = maxima["score"]
        out[:, 4] = maxima["scale"]
        out[:, 5] = maxima["linear_index"].astype(np.float64)  # exact: < 2^53
    return out


def _unpack(a: np.ndarray) -> np.ndarray:
    m = np.zeros(len(a), MAX_DTYPE)
    if len(a):
        m["position"] = a[:, 0:3]
        m["score"] = a[:, 3]
        m["scale"] = a[:, 4]
        m["linear_index"] = a[:, 5].astype(np.int64)
    return m


def allgather_maxima(local: np.ndarray, group=None, device=None) -> np.ndarray:
    """The one collective: all-gather of every rank's maxima, then the stable merge."""
    import torch
    import torch.distributed as dist

    world = dist.get_world_size(group)
    dev = device if device is not None else torch.device("cpu")
    cnt = torch.tensor([len(local)], dtype=torch.int64, device=dev)
    cnts = [torch.zeros_like(cnt) for _ in range(world)]
    dist.all_gather(cnts, cnt, group=group)
    cap = max(int(c.item()) for c in cnts)
    buf = torch.zeros((max(cap, 1), 6), dtype=torch.float64, device=dev)
    if len(local):
        buf[: len(local)] = torch.from_numpy(_pack(local)).to(dev)
    bufs = [torch.zeros_like(buf) for _ in range(world)]
    dist.all_gather(bufs, buf, group=group)
    parts = [_unpack(b[: int(c.item())].cpu().numpy()) for b, c in zip(bufs, cnts)]
    return merge_maxima(parts)


def exhaustive_sharded(volume: np.ndarray, scales, window_low, window_high, bins=64,
                       budget=None, group=None, device=None, compute=None, ctx=None, out=None):
    """kadir_brady_exhaustive over z-slabs, one per rank.

    Returns (owned score planes, owned best_scale planes, (z0, z1), merged maxima,
    visits of this rank). `compute(slab, nz, zs0, z0, z1)` may replace the
    device call (the CPU multi-process tests inject the oracle there). `out`
    optionally supplies (score, best) host buffers for the owned planes (e.g. pinned).
    """
    import torch.distributed as dist

    from . import api

    vol = np.asarray(volume, np.float32)
    if vol.ndim == 2:
        vol = vol[None]
    nz = vol.shape[0]
    world = dist.get_world_size(group) if dist.is_initialized() else 1
    rank = dist.get_rank(group) if dist.is_initialized() else 0
    R = halo_radius(scales)
    z0, z1, zs0, zs1 = slab_bounds(nz, world, rank, R)
    if z1 <= z0:
        score = np.zeros((0,) + vol.shape[1:], np.float32)
        best, local, visits = score.copy(), np.zeros(0, MAX_DTYPE), 0
    elif compute is not None:
        score, best, local, visits = compute(vol[zs0:zs1], nz, zs0, z0, z1)
    else:
        score, best, local, visits = api.kadir_brady_exhaustive_slab(
            vol[zs0:zs1], nz, zs0, z0, z1, scales, window_low, window_high, bins,
            budget=budget if budget is not None else api.DEFAULT_BUDGET, ctx=ctx, out=out)
    # one rank: the slab call already returns the reference's stable order
    merged = allgather_maxima(local, group, device) if world > 1 else local
    return score, best, (z0, z1), merged, visits
