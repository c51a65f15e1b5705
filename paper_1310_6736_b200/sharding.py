"""Multi-GPU sharding: z-slabs for the exhaustive pass,
seed interleave for the seed-grid detector.

One process per GPU (torch.distributed, NCCL over NVLink on the box; gloo in the
CPU tests). Rank g owns planes [z_g, z_{g+1}); it bins the planes
[z_g - R - 1, z_{g+1} + R + 1) (halo R = max scale + 1), scores its owned planes
only (whole 8-plane tile layers), swaps one boundary score plane with each
neighbour (exchange_edges: NCCL send/recv) so strict 26-neighbour maxima are
decided locally, and selects its maxima. ONE all-gather of the per-slab maxima
records (counts first, then the padded records) and a merge in the reference's
stable order (score descending, linear index ascending -- pipeline.cpp:163-164)
give every rank the 1-GPU list. (Byte-identity with the 1-GPU call is tested on
CPU with gloo and on one GPU with the ranks' slabs run one after another and
gloo staging; a real multi-GPU NCCL run has not been available.)

detect_sharded replicates the volume and gives rank g the plan positions
j % N == g (interleaved for balance: neighbouring seeds have similar
trajectory lengths). ONE all-gather of the fixed-size detection records
restores plan order; the population-quantile thresholds and the dedupe then
run once on the whole population (pipeline.cpp:383-401), so the selection is
byte-identical to the 1-GPU detect.

detect_batch_sharded (C5, replicas only) gives rank g a contiguous block of a
batch of volumes, runs it through one batch seek launch and all-gathers the
fixed-capacity per-volume selections once.
"""
from __future__ import annotations

import math

import numpy as np

from ._lib import DET_DTYPE, MAX_DTYPE


def collective_device(group=None, device=None):
    """Where a collective's tensors must live: NCCL moves device memory only
    (the given device, else the current CUDA device), gloo host memory only."""
    import torch
    import torch.distributed as dist

    if dist.get_backend(group) == "nccl":
        if device is not None and torch.device(device).type == "cuda":
            return torch.device(device)
        return torch.device("cuda", torch.cuda.current_device())
    return torch.device("cpu")


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
    dev = collective_device(group, device)
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


def exchange_edges(first, last, group=None):
    """The neighbour-plane exchange of the z-slab split: rank g sends its first
    owned score plane to g-1 and its last to g+1 and receives plane z0-1 (from
    g-1's last) and plane z1 (from g+1's first). Point-to-point over the process
    group (NCCL send/recv on the box, gloo in the CPU tests). Returns
    (below, above), None at the volume ends."""
    import torch
    import torch.distributed as dist

    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    if first.is_cuda and dist.get_backend(group) != "nccl":
        # gloo cannot send device memory: stage through the host (functional
        # multi-process tests on one GPU; the product path is NCCL)
        b, a = exchange_edges(first.cpu(), last.cpu(), group)
        return (b.to(first.device) if b is not None else None,
                a.to(first.device) if a is not None else None)
    below = torch.empty_like(first) if rank > 0 else None
    above = torch.empty_like(last) if rank < world - 1 else None
    ops = []
    if rank > 0:
        ops.append(dist.P2POp(dist.isend, first, rank - 1, group))
        ops.append(dist.P2POp(dist.irecv, below, rank - 1, group))
    if rank < world - 1:
        ops.append(dist.P2POp(dist.isend, last, rank + 1, group))
        ops.append(dist.P2POp(dist.irecv, above, rank + 1, group))
    if ops:
        for w in dist.batch_isend_irecv(ops):
            w.wait()
    return below, above


def allgather_maxima_device(n_local, group=None, device=None, ctx=None):
    """The maxima all-gather kept on the device: every rank's records (left on
    the device by the slab maxima call) are all-gathered as raw 48-byte rows over
    NCCL and sorted into the reference's order by salvox_merge_maxima_device --
    no host round trip, no host sort. Returns a CUDA uint8 tensor (n, 48)."""
    import torch
    import torch.distributed as dist

    from . import api

    world = dist.get_world_size(group)
    # gloo cannot move device memory: its collectives run on host copies
    # (functional multi-process tests on one GPU; the product path is NCCL)
    coll = device if dist.get_backend(group) == "nccl" else torch.device("cpu")
    cnt = torch.tensor([n_local], dtype=torch.int64, device=coll)
    cnts = [torch.zeros_like(cnt) for _ in range(world)]
    dist.all_gather(cnts, cnt, group=group)
    counts = [int(c) for c in torch.cat(cnts).cpu().tolist()]
    # rows past each rank's count are never read: no fill needed. The context
    # orders its stream after torch's (Context.after_torch) before writing it.
    buf = torch.empty((max(max(counts), 1), MAX_DTYPE.itemsize), dtype=torch.uint8, device=device)
    api.last_maxima_device(buf, ctx=ctx)
    buf_c = buf if coll == device else buf.cpu()
    bufs = [torch.empty_like(buf_c) for _ in range(world)]
    dist.all_gather(bufs, buf_c, group=group)
    cat = torch.cat([b[:c] for b, c in zip(bufs, counts)]).to(device)
    return api.merge_maxima_device(cat, ctx=ctx)  # ordered after the gather on torch's stream


def exhaustive_exchange(volume, scales, window_low, window_high, bins=64, budget=None, group=None,
                        device=None, ctx=None, out=None, maxima_out=None, d_slab=None):
    """kadir_brady_exhaustive over z-slabs with the neighbour-plane exchange: each
    rank scores only its owned planes (whole 8-plane tile layers), swaps one
    boundary plane with each neighbour, then selects its maxima; ONE all-gather
    merges them. `d_slab` (a CUDA tensor holding planes [zs0, zs1)) makes the
    call device-resident; otherwise the rank's planes of the host `volume` go up
    pipelined. Returns what exhaustive_sharded returns."""
    import torch
    import torch.distributed as dist

    from . import api

    world = dist.get_world_size(group) if dist.is_initialized() else 1
    rank = dist.get_rank(group) if dist.is_initialized() else 0
    nz = volume.shape[0] if volume is not None else None
    if nz is None:
        raise ValueError("exhaustive_exchange: pass the volume (host) for its shape")
    R = halo_radius(scales)
    z0, z1, zs0, zs1 = slab_bounds(nz, world, rank, R)
    ny, nx = volume.shape[1], volume.shape[2]
    bud = budget if budget is not None else api.DEFAULT_BUDGET
    src = d_slab if d_slab is not None else volume[zs0:zs1]
    score, best, visits = api.exhaustive_slab_scores(src, nz, zs0, z0, z1, scales, window_low,
                                                     window_high, bins, budget=bud, ctx=ctx,
                                                     out=out)
    dev = device if device is not None else torch.device("cuda", torch.cuda.current_device())
    first = torch.empty((ny, nx), dtype=torch.float32, device=dev)
    last = torch.empty_like(first)
    api.exhaustive_slab_edges(first, last, ctx=ctx)
    # NCCL's wait orders torch's stream; the maxima call orders the context's
    # stream after it (Context.after_torch), so no host synchronisation here
    below, above = exchange_edges(first, last, group) if world > 1 else (None, None)
    if world == 1:
        merged = api.exhaustive_slab_maxima(below, above, ctx=ctx, maxima_out=maxima_out)
        return score, best, (z0, z1), merged, visits
    n_local = api.exhaustive_slab_maxima(below, above, ctx=ctx, on_device=True)
    merged_d = allgather_maxima_device(n_local, group, dev, ctx=ctx)
    if d_slab is not None:  # device-resident call: the merged list stays on the device
        return score, best, (z0, z1), merged_d, visits
    n = merged_d.shape[0]
    if maxima_out is not None and len(maxima_out) >= n:
        host = torch.from_numpy(maxima_out.view(np.uint8).reshape(-1, MAX_DTYPE.itemsize)[:n])
        host.copy_(merged_d)  # one DMA into the caller's (pinned) buffer
        merged = maxima_out[:n]
    else:
        merged = merged_d.cpu().numpy().reshape(-1).view(MAX_DTYPE)
    return score, best, (z0, z1), merged, visits


def exhaustive_sharded(volume: np.ndarray, scales, window_low, window_high, bins=64,
                       budget=None, group=None, device=None, compute=None, ctx=None, out=None,
                       maxima_out=None):
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
    if world > 1 and compute is None and device is not None and vol.shape[0] >= world:
        # the device path: owned planes only, boundary-plane exchange, device merge
        return exhaustive_exchange(vol, scales, window_low, window_high, bins, budget, group,
                                   device, ctx=ctx, out=out, maxima_out=maxima_out)
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
            budget=budget if budget is not None else api.DEFAULT_BUDGET, ctx=ctx, out=out,
            maxima_out=maxima_out)
    # one rank: the slab call already returns the reference's stable order
    merged = allgather_maxima(local, group, device) if world > 1 else local
    return score, best, (z0, z1), merged, visits


def interleave_detections(parts, n_total: int) -> np.ndarray:
    """Plan order from per-rank shards: position j = rank + world * i."""
    world = len(parts)
    out = np.zeros(n_total, DET_DTYPE)
    for r, p in enumerate(parts):
        out[r::world] = p[: len(range(r, n_total, world))]
    return out


def allgather_detections(local: np.ndarray, n_total: int, group=None, device=None) -> np.ndarray:
    """The one collective of the sharded detector: all-gather of the raw
    136-byte detection records (padded to the largest shard)."""
    import torch
    import torch.distributed as dist

    world = dist.get_world_size(group)
    dev = collective_device(group, device)
    cap = (n_total + world - 1) // world
    raw = np.zeros((max(cap, 1), DET_DTYPE.itemsize), np.uint8)
    if len(local):
        raw[: len(local)] = np.ascontiguousarray(local).view(np.uint8).reshape(len(local), -1)
    buf = torch.from_numpy(raw).to(dev)
    bufs = [torch.zeros_like(buf) for _ in range(world)]
    dist.all_gather(bufs, buf, group=group)
    parts = [np.ascontiguousarray(b.cpu().numpy()).view(DET_DTYPE).reshape(-1) for b in bufs]
    return interleave_detections(parts, n_total)


def detect_sharded(volume: np.ndarray, method="shift", seed_spacing=16.0, scales=(8.0,), k=20,
                   dedupe_radius=5.0, window_low=None, window_high=None, bins=64,
                   entropy_quantile=0.9, pdf_quantile=0.0, group=None, device=None,
                   compute=None, select=None, ctx=None, **extra):
    """detect() with the seeds interleaved over the ranks (volume replicated).

    Returns (selected detections, per-seed detections in plan order, total
    visits). `compute(rank, world) -> (local, n_total, visits)` and
    `select(all_dets) -> selected` may replace the device calls (the CPU
    multi-process tests inject the oracle there).
    """
    import torch
    import torch.distributed as dist

    from . import api

    world = dist.get_world_size(group) if dist.is_initialized() else 1
    rank = dist.get_rank(group) if dist.is_initialized() else 0
    if compute is None:
        def compute(r, w):
            return api.detect_shard(volume, r, w, method, seed_spacing, scales, k, dedupe_radius,
                                    window_low, window_high, bins, entropy_quantile,
                                    pdf_quantile, ctx=ctx, **extra)
    local, n_total, visits = compute(rank, world)
    if world > 1:
        all_dets = allgather_detections(local, n_total, group, device)
        dev = collective_device(group, device)
        v = torch.tensor([visits], dtype=torch.int64, device=dev)
        dist.all_reduce(v, group=group)
        visits = int(v.item())
    else:
        all_dets = local
    if select is None:
        def select(d):
            return api.select(d, entropy_quantile, pdf_quantile, k, dedupe_radius, ctx=ctx)
    return select(all_dets), all_dets, visits


def batch_bounds(batch: int, world: int, rank: int):
    """Contiguous block of volumes [b0, b1) of a batch for one rank."""
    return batch * rank // world, batch * (rank + 1) // world


def detect_batch_sharded(volumes, method="shift", seed_spacing=16.0, scales=(8.0,), k=20,
                         dedupe_radius=5.0, window_low=None, window_high=None, bins=64,
                         entropy_quantile=0.9, pdf_quantile=0.0, group=None, device=None,
                         compute=None, ctx=None, **extra):
    """detect() over a batch of volumes (replicas only): rank r
    runs the contiguous block batch_bounds(B, world, r) through ONE device call
    (salvox_detect_batch_device over the block uploaded back to back), then one
    all-gather of fixed-capacity (k records + count per volume) buffers gives
    every rank the whole batch's selections in volume order.

    `volumes`: host array (B, nz, ny, nx) or (B, ny, nx). Returns
    ([selected DET_DTYPE per volume], total visits). `compute(b0, b1) ->
    ([selected per volume], visits)` may replace the device call (the CPU
    multi-process tests inject the oracle there).
    """
    import torch
    import torch.distributed as dist

    from . import api

    vols = np.asarray(volumes, np.float32)
    B = vols.shape[0]
    world = dist.get_world_size(group) if dist.is_initialized() else 1
    rank = dist.get_rank(group) if dist.is_initialized() else 0
    b0, b1 = batch_bounds(B, world, rank)
    kk = max(int(k), 1)
    if compute is None:
        def compute(a, b):
            if b <= a:
                return [], 0
            dev = (torch.device(device) if device is not None else
                   torch.device("cuda", torch.cuda.current_device()))
            d = torch.from_numpy(np.ascontiguousarray(vols[a:b])).to(dev, non_blocking=True)
            return api.detect_batch_device(d, b - a, vols.shape[1:], method, seed_spacing, scales,
                                           kk, dedupe_radius, window_low, window_high, bins,
                                           entropy_quantile, pdf_quantile, ctx=ctx, **extra)
    local, visits = compute(b0, b1)
    if world == 1:
        return list(local), int(visits)
    cap = (B + world - 1) // world  # largest block
    rec = np.zeros((cap, kk), DET_DTYPE)
    cnt = np.zeros(cap, np.int64)
    for i, sel in enumerate(local):
        rec[i, : len(sel)] = sel[:kk]
        cnt[i] = len(sel)
    dev = collective_device(group, device)
    raw = torch.from_numpy(rec.view(np.uint8).reshape(cap, -1).copy()).to(dev)
    meta = torch.from_numpy(np.concatenate([cnt, [visits]]).astype(np.int64)).to(dev)
    raws = [torch.zeros_like(raw) for _ in range(world)]
    metas = [torch.zeros_like(meta) for _ in range(world)]
    dist.all_gather(raws, raw, group=group)
    dist.all_gather(metas, meta, group=group)
    out, total = [], 0
    for r in range(world):
        a, b = batch_bounds(B, world, r)
        rr = np.ascontiguousarray(raws[r].cpu().numpy()).view(DET_DTYPE).reshape(cap, kk)
        mm = metas[r].cpu().numpy()
        out += [rr[i, : int(mm[i])].copy() for i in range(b - a)]
        total += int(mm[cap])
    return out, total
