"""Multi-process (world_size 2, gloo, CPU) tests of the sharding host logic:
slab bounds + halo, the one all-gather of per-slab maxima and the stable merge;
the seed interleave of the detector, its one all-gather of detection records
and the global selection.
The per-slab compute is injected (the oracle stands in for the device kernel,
which cannot run here); the merged result must equal the single-process one."""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

from tests import phantoms

SCALES = [2.0, 3.0, 4.0]


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _oracle_slab(vol_full, bins):
    from oracle import oracle as O
    from paper_1310_6736_b200 import sharding

    def compute(slab, nz, zs0, z0, z1):
        # score the planes [z0-1, z1+1) of the slab with the oracle, select maxima of [z0, z1)
        zc0, zc1 = max(0, z0 - 1), min(nz, z1 + 1)
        s, b, v = O.exhaustive(slab, 0, bins, bins, SCALES, budget=10**12, mode="exact",
                               threads=2, z_range=(zc0 - zs0, zc1 - zs0))
        pos, sc, scale, lin = O.local_maxima(s, b)
        keep = (pos[:, 2] + zs0 >= z0) & (pos[:, 2] + zs0 < z1)
        m = np.zeros(int(keep.sum()), sharding.MAX_DTYPE)
        m["position"] = pos[keep] + [0, 0, zs0]
        m["score"] = sc[keep]
        m["scale"] = scale[keep]
        ny, nx = slab.shape[1:]
        m["linear_index"] = lin[keep] + zs0 * ny * nx
        return s[z0 - zs0:z1 - zs0], b[z0 - zs0:z1 - zs0], m, v
    return compute


def _worker(rank, world, port, vol, bins, out):
    import torch.distributed as dist

    from paper_1310_6736_b200 import sharding

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        s, b, (z0, z1), merged, _ = sharding.exhaustive_sharded(
            vol, SCALES, 0, bins, bins, compute=_oracle_slab(vol, bins))
        out[rank] = (z0, z1, s, merged)
    finally:
        dist.destroy_process_group()


def test_slab_bounds_cover_and_halo():
    from paper_1310_6736_b200 import sharding

    for nz, world in [(256, 8), (34, 4), (5, 8), (1, 2)]:
        R = sharding.halo_radius([3.0, 15.0])
        owned = []
        for r in range(world):
            z0, z1, zs0, zs1 = sharding.slab_bounds(nz, world, r, R)
            owned += list(range(z0, z1))
            assert zs0 == max(0, z0 - R - 1) and zs1 == min(nz, z1 + R + 1)
        assert owned == list(range(nz))


def test_two_rank_gloo_matches_single_process(oracle):
    from paper_1310_6736_b200 import sharding

    bins = 16
    vol, _ = oracle.make_phantom(phantoms.ball_3d(18, (9.0, 8.0, 9.0), 4.0, 21, levels=bins,
                                                 background={"type": "gaussian", "mean": 4.0,
                                                             "sigma": 1.5}))
    s_ref, b_ref, _ = oracle.exhaustive(vol, 0, bins, bins, SCALES, budget=10**12, mode="exact",
                                        threads=4)
    pos, sc, scale, lin = oracle.local_maxima(s_ref, b_ref)
    mgr = mp.Manager()
    out = mgr.dict()
    port = _free_port()
    ctx = mp.get_context("spawn")
    procs = [ctx.Process(target=_worker, args=(r, 2, port, vol, bins, out)) for r in range(2)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(120)
        assert p.exitcode == 0
    planes = []
    for r in range(2):
        z0, z1, s, merged = out[r]
        planes.append((z0, s))
        assert np.array_equal(merged["linear_index"], lin)  # identical on every rank
        assert np.array_equal(merged["score"], sc)
        assert np.array_equal(merged["scale"], scale)
    full = np.concatenate([s for _, s in sorted(planes, key=lambda t: t[0])])
    assert np.array_equal(full, s_ref)


def test_merge_is_stable_order():
    from paper_1310_6736_b200 import sharding

    a = np.zeros(3, sharding.MAX_DTYPE)
    a["score"] = [5.0, 3.0, 3.0]
    a["linear_index"] = [10, 4, 20]
    b = np.zeros(2, sharding.MAX_DTYPE)
    b["score"] = [5.0, 3.0]
    b["linear_index"] = [2, 11]
    m = sharding.merge_maxima([a, b])
    assert list(m["linear_index"]) == [2, 10, 4, 11, 20]


DET_KW = dict(method="shift", seed_spacing=8.0, scales=[3.0, 5.0], top_k=6, dedupe_radius=4.0)


def _det_volume(oracle):
    vol, _ = oracle.make_phantom(phantoms.ball_3d(24, (12.0, 10.0, 13.0), 5.0, 33))
    return vol


def _det_worker(rank, world, port, vol, out):
    import torch.distributed as dist

    from oracle import oracle as O
    from paper_1310_6736_b200 import sharding

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        def compute(r, w):  # the oracle stands in for salvox_detect_shard
            _, per_seed, _ = O.detect(vol, 0, 64, 64, **DET_KW)
            return per_seed[r::w].copy(), len(per_seed), 1000 + r

        def select(d):
            return O.select(d, 0.9, 0.0, DET_KW["top_k"], DET_KW["dedupe_radius"])

        sel, all_dets, visits = sharding.detect_sharded(vol, compute=compute, select=select)
        out[rank] = (sel.tobytes(), all_dets.tobytes(), visits)
    finally:
        dist.destroy_process_group()


def test_two_rank_gloo_detect_matches_single_process(oracle):
    from paper_1310_6736_b200 import sharding

    vol = _det_volume(oracle)
    sel_ref, seeds_ref, _ = oracle.detect(vol, 0, 64, 64, **DET_KW)
    assert len(seeds_ref) > 8 and len(sel_ref) > 0
    mgr = mp.Manager()
    out = mgr.dict()
    port = _free_port()
    ctx = mp.get_context("spawn")
    procs = [ctx.Process(target=_det_worker, args=(r, 2, port, vol, out)) for r in range(2)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(120)
        assert p.exitcode == 0
    for r in range(2):
        sel_b, all_b, visits = out[r]
        assert all_b == seeds_ref.tobytes()   # plan order restored, byte for byte
        assert sel_b == sel_ref.tobytes()     # global thresholds + dedupe
        assert visits == 2001


def test_interleave_detections_ragged():
    from paper_1310_6736_b200 import sharding

    d = np.zeros(7, sharding.DET_DTYPE)
    d["seed_index"] = np.arange(7)
    parts = [np.concatenate([d[r::3], np.zeros(1, sharding.DET_DTYPE)]) for r in range(3)]
    assert list(sharding.interleave_detections(parts, 7)["seed_index"]) == list(range(7))


@pytest.mark.parametrize("world", [1, 2, 4, 8])
def test_bench_weak_scaling_slabs(world):
    """bench.py's N-rank volume (weak scaling): N x 256^3 voxels, every rank's
    owned slab holds exactly 256^3 voxels; N=1 is C2, N=8 the 512^3 C4 spec."""
    import bench
    from paper_1310_6736_b200 import sharding
    from tests import phantoms

    spec = bench.weak_spec(world)
    nx, ny, nz = spec["dims"]
    assert nx * ny * nz == world * 256 ** 3
    if world == 1:
        assert spec == phantoms.config_c2()
    if world == 8:
        assert spec == phantoms.config_c4()
    for r in spec["regions"]:  # every region lies inside the volume
        assert all(0 <= c < d for c, d in zip(r["center"], spec["dims"]))
    R = sharding.halo_radius(bench.SCALES)
    for rank in range(world):
        z0, z1, zs0, zs1 = sharding.slab_bounds(nz, world, rank, R)
        assert (z1 - z0) * nx * ny == 256 ** 3
        assert zs0 == max(0, z0 - R - 1) and zs1 == min(nz, z1 + R + 1)


def _exchange_worker(rank, world, port, vol, bins, out):
    """The exchange form of the slab split (sharding.exhaustive_exchange): owned
    planes only, one boundary plane each way (sharding.exchange_edges), maxima
    with the received planes, one all-gather. The oracle stands in for the
    device scoring and maxima."""
    import torch
    import torch.distributed as dist

    from oracle import oracle as O
    from paper_1310_6736_b200 import sharding

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        nz, ny, nx = vol.shape
        R = sharding.halo_radius(SCALES)
        z0, z1, zs0, zs1 = sharding.slab_bounds(nz, world, rank, R)
        s, _, _ = O.exhaustive(vol[zs0:zs1], 0, bins, bins, SCALES, budget=10**12, mode="exact",
                               threads=2, z_range=(z0 - zs0, z1 - zs0))
        own = s[z0 - zs0:z1 - zs0]
        below, above = sharding.exchange_edges(torch.from_numpy(own[0].copy()),
                                               torch.from_numpy(own[-1].copy()))
        ext = [own]
        if below is not None:
            ext.insert(0, below.numpy()[None])
        if above is not None:
            ext.append(above.numpy()[None])
        ext = np.concatenate(ext)
        e0 = z0 - (1 if below is not None else 0)
        pos, sc, scale, lin = O.local_maxima(ext, np.zeros_like(ext))
        keep = (pos[:, 2] + e0 >= z0) & (pos[:, 2] + e0 < z1)
        m = np.zeros(int(keep.sum()), sharding.MAX_DTYPE)
        m["position"] = pos[keep] + [0, 0, e0]
        m["score"] = sc[keep]
        m["linear_index"] = lin[keep] + e0 * ny * nx
        merged = sharding.allgather_maxima(m)
        out[rank] = (z0, z1, own, merged)
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_exchange_gloo_matches_single_process(oracle, world):
    """Each rank scores only its owned planes and receives the two neighbour
    planes: the merged maxima equal the single-process ones (3 ranks: a middle
    rank exchanges both ways)."""
    bins = 16
    vol, _ = oracle.make_phantom(phantoms.ball_3d(18, (9.0, 8.0, 9.0), 4.0, 21, levels=bins,
                                                 background={"type": "gaussian", "mean": 4.0,
                                                             "sigma": 1.5}))
    s_ref, b_ref, _ = oracle.exhaustive(vol, 0, bins, bins, SCALES, budget=10**12, mode="exact",
                                        threads=4)
    pos, sc, scale, lin = oracle.local_maxima(s_ref, b_ref)
    mgr = mp.Manager()
    out = mgr.dict()
    port = _free_port()
    ctx = mp.get_context("spawn")
    procs = [ctx.Process(target=_exchange_worker, args=(r, world, port, vol, bins, out))
             for r in range(world)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(120)
        assert p.exitcode == 0
    planes = []
    for r in range(world):
        z0, z1, s, merged = out[r]
        planes.append((z0, s))
        assert np.array_equal(merged["linear_index"], lin)
        assert np.array_equal(merged["score"], sc)
    full = np.concatenate([s for _, s in sorted(planes, key=lambda t: t[0])])
    assert np.array_equal(full, s_ref)


BATCH_KW = dict(method="shift", seed_spacing=8.0, scales=[3.0, 5.0], top_k=4, dedupe_radius=4.0)


def _batch_volumes(oracle, n=5):
    return np.stack([oracle.make_phantom(phantoms.ball_3d(
        20, (8.0 + i, 10.0, 11.0 - i), 4.0, 40 + i))[0] for i in range(n)])


def _batch_worker(rank, world, port, vols, out):
    import torch.distributed as dist

    from oracle import oracle as O
    from paper_1310_6736_b200 import sharding

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        def compute(a, b):  # the oracle stands in for salvox_detect_batch_device
            sels, vis = [], 0
            for v in vols[a:b]:
                s, _, n = O.detect(v, 0, 64, 64, **BATCH_KW)
                sels.append(s)
                vis += n
            return sels, vis

        sels, visits = sharding.detect_batch_sharded(vols, k=BATCH_KW["top_k"], compute=compute)
        out[rank] = ([s.tobytes() for s in sels], visits)
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_batch_replicas_gloo_match_single_process(oracle, world):
    """C5 (replicas only): each rank runs a contiguous block of the batch, one
    all-gather of fixed-capacity per-volume selections; every rank ends with the
    whole batch in volume order, byte-identical to one process."""
    vols = _batch_volumes(oracle)
    ref, ref_vis = [], 0
    for v in vols:
        s, _, n = oracle.detect(v, 0, 64, 64, **BATCH_KW)
        ref.append(s.tobytes())
        ref_vis += n
    assert any(len(r) for r in ref)
    mgr = mp.Manager()
    out = mgr.dict()
    port = _free_port()
    ctx = mp.get_context("spawn")
    procs = [ctx.Process(target=_batch_worker, args=(r, world, port, vols, out))
             for r in range(world)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(180)
        assert p.exitcode == 0
    for r in range(world):
        sels, visits = out[r]
        assert sels == ref and visits == ref_vis


def test_batch_bounds_cover():
    from paper_1310_6736_b200 import sharding

    for B, world in [(64, 8), (5, 3), (2, 4)]:
        blocks = [sharding.batch_bounds(B, world, r) for r in range(world)]
        assert [i for a, b in blocks for i in range(a, b)] == list(range(B))
