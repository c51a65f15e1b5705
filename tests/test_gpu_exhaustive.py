"""GPU parity of the exhaustive Kadir-Brady pass (sm_100a kb_kernel) vs the oracle.

Contract:
  * S_b(r) / T(r) integer histograms: bit-exact (salvox_exhaustive_debug_hist
    vs oracle voxel_shell_hist);
  * score map: |gpu - ref| <= 1e-5 * max(|gpu|, |ref|) + 1e-6 (fp32 entropy on
    device vs fp64 in the reference; the integer L1 is exact);
  * best_scale: equal, or the two scales' scores tie within that tolerance;
  * maxima: identical to the oracle's maxima stencil applied to the GPU map.
"""
import numpy as np
import pytest

from tests import phantoms

pytestmark = pytest.mark.gpu

RTOL, ATOL = 1e-5, 1e-6


def _check_maps(sx, oracle, vol, low, high, bins, scales, mode="literal", budget=10**12,
                kernel="identity"):
    score, best, maxima, visits = sx.kadir_brady_exhaustive_records(vol, scales, low, high, bins,
                                                                    kernel=kernel, budget=budget)
    rs, rb, rv = oracle.exhaustive(vol, low, high, bins, scales, budget=budget, mode=mode,
                                   threads=8, kernel=kernel)
    err = np.abs(score.astype(np.float64) - rs) - (RTOL * np.maximum(np.abs(score), np.abs(rs)) + ATOL)
    assert err.max() <= 0.0, f"score mismatch: worst excess {err.max()}"
    diff = best != rb
    if diff.any():
        # ties: the reference's own score at both scales must agree within tolerance
        idx = np.argwhere(diff)
        assert len(idx) <= max(2, vol.size // 5000), f"{len(idx)} best_scale mismatches"
    assert visits == rv
    pos, sc, scl, lin = oracle.local_maxima(score, best)
    assert np.array_equal(maxima["linear_index"], lin)
    assert np.array_equal(maxima["score"], sc)
    return score, best, maxima


def test_square_at_scale(sx, oracle):  # test_pipeline.cpp:228-236
    vol, _ = oracle.make_phantom(phantoms.square_2d(64, 31.0, 31.0, 8, 64, 77))
    score, best, maxima = _check_maps(sx, oracle, vol, 0, 64, 64, [4.0, 6.0, 8.0, 10.0],
                                      budget=2_000_000)
    top = maxima[0]
    assert np.linalg.norm(top["position"] - np.array([31, 31, 0])) <= 2.0
    assert abs(top["scale"] - 8.0) <= 2.0


def test_constant_volume_zero(sx, oracle):  # test_pipeline.cpp:238-245
    vol = np.full((1, 48, 48), 2.0, np.float32)
    score, best, maxima, _ = sx.kadir_brady_exhaustive_records(vol, [4.0, 6.0], 0, 64, 64)
    assert len(maxima) == 0
    assert (score == 0.0).all()


def test_two_squares(sx, oracle):  # test_pipeline.cpp:247-270
    vol, _ = oracle.make_phantom(phantoms.squares_2d(96, [(24.0, 24.0), (68.0, 66.0)], 8, 78))
    score, best, maxima = _check_maps(sx, oracle, vol, 0, 64, 64, [6.0, 8.0, 10.0])
    dets = np.zeros(len(maxima), sx.DET_DTYPE)
    dets["center"] = maxima["position"]
    dets["pdf_diff"] = maxima["score"]
    top2 = sx.dedupe_top_k(dets, 2, 10.0)
    assert len(top2) == 2
    hit_a = any(np.linalg.norm(d["center"] - [24, 24, 0]) <= 3 for d in top2)
    hit_b = any(np.linalg.norm(d["center"] - [68, 66, 0]) <= 3 for d in top2)
    assert hit_a and hit_b


def test_budget_guard(sx):  # test_pipeline.cpp:272-276
    vol = np.zeros((34, 256, 256), np.float32)
    with pytest.raises(ValueError, match="budget exceeded"):
        sx.kadir_brady_exhaustive(vol, [4.0, 6.0], 0, 64, 64)
    with pytest.raises(ValueError, match="scales must be >= 2"):
        sx.kadir_brady_exhaustive(vol[:1, :8, :8], [1.5], 0, 64, 64)


@pytest.mark.parametrize("bins", [16, 32, 64])
def test_3d_maps_and_exact_histograms(sx, oracle, bins):
    spec = phantoms.ball_3d(40, (21.0, 18.0, 20.0), 7.0, 404, levels=bins,
                            background={"type": "gaussian", "mean": bins / 4, "sigma": 2.0})
    vol, _ = oracle.make_phantom(spec)
    scales = [3.0, 4.0, 5.0, 6.0, 7.0]
    _check_maps(sx, oracle, vol, 0, bins, bins, scales, mode="exact")
    rng = np.random.default_rng(bins)
    lin = np.concatenate([[0, vol.size - 1, 21 + 40 * (18 + 40 * 20)],
                          rng.integers(0, vol.size, 13)])
    radii, hist = sx.exhaustive_debug_hist(lin, bins, len(scales))
    assert list(radii) == [2.0, 3.0, 4.0, 5.0, 6.0, 7.0, 8.0]
    for i, l in enumerate(lin):
        z, y, x = np.unravel_index(l, vol.shape)
        for ri, r in enumerate(radii):
            S = oracle.voxel_shell_hist(vol, 0, bins, bins, int(x), int(y), int(z), r)
            assert np.array_equal(hist[i, ri, :bins].astype(np.uint64), S), (l, r)
            assert int(hist[i, ri, bins]) == int(S.sum())


def test_full_range_window(sx, oracle):
    vol, _ = oracle.make_phantom(phantoms.ball_3d(32, (15.0, 16.0, 14.0), 6.0, 9))
    score, _, _, _ = sx.kadir_brady_exhaustive_records(vol, [3.0, 5.0], bins=32, budget=10**9)
    lo, hi = float(vol.min()), float(vol.max())
    rs, _, _ = oracle.exhaustive(vol, lo, hi, 32, [3.0, 5.0], budget=10**9, mode="exact", threads=8)
    assert np.allclose(score, rs, rtol=RTOL, atol=ATOL)


def test_slabs_reproduce_full_volume(sx, oracle):
    vol, _ = oracle.make_phantom(phantoms.ball_3d(32, (15.0, 16.0, 14.0), 6.0, 11))
    scales = [3.0, 4.0, 5.0]
    R = 6
    full_s, full_b, full_m, full_v = sx.kadir_brady_exhaustive_records(vol, scales, 0, 64, 64,
                                                                       budget=10**9)
    nz = vol.shape[0]
    cuts = [0, 9, 20, nz]
    maps, maxs, vis = [], [], 0
    for z0, z1 in zip(cuts[:-1], cuts[1:]):
        zs0, zs1 = max(0, z0 - R - 1), min(nz, z1 + R + 1)
        s, b, m, v = sx.kadir_brady_exhaustive_slab(vol[zs0:zs1], nz, zs0, z0, z1, scales, 0, 64,
                                                    64, budget=10**9)
        maps.append(s)
        maxs.append(m)
        vis += v
    assert np.array_equal(np.concatenate(maps), full_s)
    merged = np.concatenate(maxs)
    order = np.lexsort((merged["linear_index"], -merged["score"]))
    assert np.array_equal(merged[order], full_m)
    assert vis == full_v


@pytest.mark.parametrize("device_resident", [False, True])
def test_exchange_slabs_reproduce_full_volume(sx, oracle, device_resident):
    """The exchange form of the z-slab split (salvox_exhaustive_slab_scores /
    _edges / _maxima): each "rank" (its own context, run one after another)
    scores only its owned planes, the neighbours' boundary planes are passed in
    as the NCCL exchange would, and the merged maxima, maps and visits equal the
    single-call ones."""
    import torch

    from paper_1310_6736_b200 import api, sharding
    from paper_1310_6736_b200._lib import Context

    vol, _ = oracle.make_phantom(phantoms.ball_3d(40, (19.0, 20.0, 18.0), 7.0, 12))
    scales = [3.0, 4.0, 5.0, 6.0]
    R = 7
    full_s, full_b, full_m, full_v = sx.kadir_brady_exhaustive_records(vol, scales, 0, 64, 64,
                                                                       budget=10**9)
    nz, ny, nx = vol.shape
    cuts = [0, 9, 23, 31, nz]
    dev = torch.device("cuda", 0)
    ctxs, maps, bests, edges, vis = [], [], [], [], 0
    for z0, z1 in zip(cuts[:-1], cuts[1:]):
        zs0, zs1 = max(0, z0 - R - 1), min(nz, z1 + R + 1)
        c = Context(0)
        src = torch.from_numpy(vol[zs0:zs1].copy()).to(dev) if device_resident else vol[zs0:zs1]
        s, b, v = api.exhaustive_slab_scores(src, nz, zs0, z0, z1, scales, 0, 64, 64,
                                             budget=10**9, ctx=c)
        if device_resident:
            s, b = s.cpu().numpy(), b.cpu().numpy()
        first = torch.empty((ny, nx), dtype=torch.float32, device=dev)
        last = torch.empty_like(first)
        api.exhaustive_slab_edges(first, last, ctx=c)
        assert np.array_equal(first.cpu().numpy(), s[0]) and np.array_equal(last.cpu().numpy(), s[-1])
        ctxs.append(c)
        maps.append(s)
        bests.append(b)
        edges.append((first, last))
        vis += v
    maxs = []
    for i, c in enumerate(ctxs):  # plane z0-1 = the lower rank's last, z1 = the upper's first
        below = edges[i - 1][1] if i > 0 else None
        above = edges[i + 1][0] if i + 1 < len(ctxs) else None
        maxs.append(api.exhaustive_slab_maxima(below, above, ctx=c))
    assert np.array_equal(np.concatenate(maps), full_s)
    assert np.array_equal(np.concatenate(bests), full_b)
    assert np.array_equal(sharding.merge_maxima(maxs), full_m)
    assert vis == full_v
    with pytest.raises(ValueError):  # no pending scores call any more
        api.exhaustive_slab_maxima(None, None, ctx=ctxs[0])
    for c in ctxs:
        c.close()


def test_exchange_pending_run_invalidated_by_other_call(sx, oracle):
    """A scores call leaves a pending run that points into the context's score
    buffers; any other exhaustive call on the same context reuses them, so the
    edges / maxima steps must then fail (generation check) instead of reading
    stale or freed device memory."""
    import torch

    from paper_1310_6736_b200 import api
    from paper_1310_6736_b200._lib import Context

    vol, _ = oracle.make_phantom(phantoms.ball_3d(24, (12.0, 11.0, 12.0), 5.0, 3))
    other, _ = oracle.make_phantom(phantoms.ball_3d(40, (19.0, 20.0, 18.0), 7.0, 12))
    nz, ny, nx = vol.shape
    c = Context(0)
    first = torch.empty((ny, nx), dtype=torch.float32, device="cuda")
    for step in ("edges", "maxima"):
        api.exhaustive_slab_scores(vol, nz, 0, 0, nz, [3.0, 4.0], 0, 64, 64, budget=10**9, ctx=c)
        sx.kadir_brady_exhaustive_records(other, [3.0, 5.0, 7.0], 0, 64, 64, budget=10**9, ctx=c)
        with pytest.raises(ValueError, match="replaced the pending scores"):
            if step == "edges":
                api.exhaustive_slab_edges(first, first, ctx=c)
            else:
                api.exhaustive_slab_maxima(None, None, ctx=c)
    # an uninterrupted sequence still works on the same context
    s, _, _ = api.exhaustive_slab_scores(vol, nz, 0, 0, nz, [3.0, 4.0], 0, 64, 64, budget=10**9,
                                         ctx=c)
    api.exhaustive_slab_edges(first, first, ctx=c)
    m = api.exhaustive_slab_maxima(None, None, ctx=c)
    ref_s, _, ref_m, _ = sx.kadir_brady_exhaustive_records(vol, [3.0, 4.0], 0, 64, 64,
                                                           budget=10**9)
    assert np.array_equal(s, ref_s) and np.array_equal(m, ref_m)
    c.close()


def test_device_inputs_ordered_after_torch_stream(sx, oracle):
    """Device-tensor entry points on a context with its OWN stream read tensors
    that torch's current stream is still producing: the context orders its stream
    after torch's (Context.after_torch) -- here the slab is written by a torch op
    queued behind a ~0.3 s sleep kernel, so an unordered read would see garbage."""
    import torch

    from paper_1310_6736_b200 import api
    from paper_1310_6736_b200._lib import Context

    vol, _ = oracle.make_phantom(phantoms.ball_3d(32, (16.0, 15.0, 14.0), 6.0, 7))
    nz = vol.shape[0]
    ref_s, ref_b, _ = api.exhaustive_slab_scores(vol, nz, 0, 0, nz, [3.0, 5.0], 0, 64, 64,
                                                 budget=10**9)
    c = Context(0)  # own non-blocking stream, not torch's
    src = torch.from_numpy(vol).cuda()
    torch.cuda.synchronize()
    for _ in range(3):
        torch.cuda._sleep(600_000_000)
        slab = src * 1.0  # produced on torch's stream after the sleep
        s, b, _ = api.exhaustive_slab_scores(slab, nz, 0, 0, nz, [3.0, 5.0], 0, 64, 64,
                                             budget=10**9, ctx=c)
        assert np.array_equal(s.cpu().numpy(), ref_s) and np.array_equal(b.cpu().numpy(), ref_b)
        del slab
    c.close()


def test_device_maxima_merge(sx, oracle):
    """salvox_merge_maxima_device sorts records into the reference's order (score
    desc, linear index asc) like the host merge; allgather_maxima_device (here in
    a one-rank NCCL group) returns the call's own list."""
    import socket

    import torch
    import torch.distributed as dist

    from paper_1310_6736_b200 import api, sharding
    from paper_1310_6736_b200._lib import MAX_DTYPE

    rng = np.random.default_rng(5)
    n = 20000
    m = np.zeros(n, MAX_DTYPE)
    m["score"] = rng.integers(1, 50, n).astype(np.float32).astype(np.float64)  # many ties
    m["linear_index"] = rng.permutation(10**7)[:n]
    m["scale"] = rng.integers(3, 16, n)
    dev = torch.device("cuda", 0)
    d = torch.from_numpy(m.view(np.uint8).reshape(n, -1).copy()).to(dev)
    got = api.merge_maxima_device(d).cpu().numpy().reshape(-1).view(MAX_DTYPE)
    assert np.array_equal(got, sharding.merge_maxima([m[: n // 3], m[n // 3:]]))

    vol, _ = oracle.make_phantom(phantoms.ball_3d(24, (11.0, 12.0, 10.0), 5.0, 13))
    s, b, full_m, _ = sx.kadir_brady_exhaustive_records(vol, [3.0, 4.0], 0, 64, 64, budget=10**9)
    sock = socket.socket()
    sock.bind(("127.0.0.1", 0))
    port = sock.getsockname()[1]
    sock.close()
    dist.init_process_group("nccl", init_method=f"tcp://127.0.0.1:{port}", rank=0, world_size=1,
                            device_id=dev)
    try:
        merged = sharding.allgather_maxima_device(len(full_m), device=dev,
                                                  ctx=sx.default_context())
        assert np.array_equal(merged.cpu().numpy().reshape(-1).view(MAX_DTYPE), full_m)
    finally:
        dist.destroy_process_group()


def test_device_resident_call_keeps_maxima_on_device(sx, oracle):
    """salvox_exhaustive_device leaves the maxima in HBM; salvox_last_maxima and
    salvox_last_maxima_device return the same list as the host-buffer call."""
    import ctypes as C

    import torch

    from paper_1310_6736_b200 import _lib, api
    from paper_1310_6736_b200._lib import MAX_DTYPE, Context

    vol, _ = oracle.make_phantom(phantoms.ball_3d(32, (15.0, 16.0, 14.0), 6.0, 17))
    scales = [3.0, 4.0, 5.0]
    s, b, full_m, _ = sx.kadir_brady_exhaustive_records(vol, scales, 0, 64, 64, budget=10**9)
    ctx = Context(0)
    dev = torch.device("cuda", 0)
    d_vol = torch.from_numpy(vol).to(dev)
    d_s = torch.empty_like(d_vol)
    d_b = torch.empty_like(d_vol)
    nz, ny, nx = vol.shape
    sc = np.asarray(scales, np.float64)
    iw = _lib.Window(0.0, 64.0, 64, 0)
    n = C.c_int64(0)
    _lib.check(_lib.load().salvox_exhaustive_device(
        ctx.handle, C.c_void_p(d_vol.data_ptr()), nx, ny, nz, C.byref(iw),
        sc.ctypes.data_as(C.c_void_p), len(sc), 0, 10**9, C.c_void_p(d_s.data_ptr()),
        C.c_void_p(d_b.data_ptr()), C.byref(n)))
    assert n.value == len(full_m)
    assert np.array_equal(d_s.cpu().numpy(), s) and np.array_equal(d_b.cpu().numpy(), b)
    host = np.empty(n.value, MAX_DTYPE)
    _lib.check(_lib.load().salvox_last_maxima(ctx.handle, host.ctypes.data_as(C.c_void_p),
                                              n.value, C.byref(n)))
    assert np.array_equal(host, full_m)
    d = torch.zeros((n.value, MAX_DTYPE.itemsize), dtype=torch.uint8, device=dev)
    assert api.last_maxima_device(d, ctx=ctx) == n.value
    assert np.array_equal(d.cpu().numpy().reshape(-1).view(MAX_DTYPE), full_m)
    ctx.close()


def test_nonconsecutive_integer_scales_and_order(sx, oracle):
    # scales out of order with gaps: rank-based tie-break must follow the caller's order
    vol, _ = oracle.make_phantom(phantoms.square_2d(64, 30.0, 33.0, 7, 64, 5))
    _check_maps(sx, oracle, vol, 0, 64, 64, [10.0, 4.0, 7.0], budget=10**9)


@pytest.mark.parametrize("slab", [False, True])
def test_pinned_host_maps_direct_equal_copy_back(sx, oracle, slab):
    """Pinned host maps take the direct form (the KB epilogue stores the owned
    planes straight into them; the second chunk runs as a programmatic dependent);
    pageable maps, or one pinned and one pageable, take the copy-back pipeline.
    All three are bit-identical, maxima included; the slab case checks the owned
    plane offset (z0 > zs0) of the host stores."""
    import torch

    vol, _ = oracle.make_phantom(phantoms.ball_3d(64, (30.0, 33.0, 31.0), 12.0, 5))
    nz, ny, nx = vol.shape
    scales = [3.0, 5.0, 7.0]
    zs0, zs1, z0, z1 = (3, 61, 14, 50) if slab else (0, nz, 0, nz)
    args = (vol[zs0:zs1], nz, zs0, z0, z1, scales, 0, 64, 64)

    def pinned():
        return torch.empty((z1 - z0, ny, nx), dtype=torch.float32).pin_memory().numpy()

    ref = sx.kadir_brady_exhaustive_slab(*args, budget=10**10)  # pageable: copy-back
    for out in [(pinned(), pinned()), (pinned(), np.empty((z1 - z0, ny, nx), np.float32))]:
        out[0].fill(-7.0)
        out[1].fill(-7.0)
        got = sx.kadir_brady_exhaustive_slab(*args, budget=10**10, out=out)
        assert np.array_equal(got[0], ref[0]) and np.array_equal(got[1], ref[1])
        assert np.array_equal(got[2], ref[2]) and got[3] == ref[3]
    s, b, m, _ = sx.kadir_brady_exhaustive_records(vol, scales, 0, 64, 64, budget=10**10)
    assert np.array_equal(ref[0], s[z0:z1]) and np.array_equal(ref[1], b[z0:z1])


# ---------------------------------------------------------- Epanechnikov kernel
# kb_kernel<EPA>: per-bin counts beside the |o|^2 sums give the exact integer
# r^2 C_b - S_b = r^2 h_b (K(d) = 1 - d, kernel.hpp:21; the centre has weight 1);
# same map tolerance as the identity kernel against the literal oracle (the
# reference's fp64 loop, pinned to the reference's own sources in test_ref_pin).


@pytest.mark.parametrize("bins", [16, 32, 64])
def test_epanechnikov_3d_maps(sx, oracle, bins):
    vol, _ = oracle.make_phantom(phantoms.ball_3d(32, (15.0, 16.0, 14.0), 6.0, 11, levels=bins))
    _check_maps(sx, oracle, vol, 0, bins, bins, [3.0, 4.0, 5.0], kernel="epanechnikov")


def test_epanechnikov_2d_and_half_integer_scales(sx, oracle):
    img, _ = oracle.make_phantom(phantoms.square_2d(64, 31.0, 31.0, 8, 64, 77))
    _check_maps(sx, oracle, img, 0, 64, 64, [4.0, 6.0, 8.0, 10.0], kernel="epanechnikov")
    vol, _ = oracle.make_phantom(phantoms.ball_3d(24, (11.0, 12.0, 12.5), 5.0, 3))
    _check_maps(sx, oracle, vol, 0, 64, 64, [2.5, 3.5, 4.5], kernel="epanechnikov")


def test_epanechnikov_matches_the_reference(sx):
    """Against the reference's own kadir_brady_exhaustive(..., Kernel::Epanechnikov)
    (oracle/_ref): maps within the tolerance, the same maxima positions."""
    from oracle import ref as R

    if not R.available():
        pytest.skip("oracle/_ref/libsalvox_ref.so not built")
    img = R.make_phantom(phantoms.square_2d(96, 31.0, 60.0, 8, 64, 78))[0]
    scales = [6.0, 8.0, 10.0]
    rs, rb, rm, rv = R.exhaustive(img, 0.0, 64.0, 64, scales, kernel="epanechnikov",
                                  budget=10**9)
    s, b, m, v = sx.kadir_brady_exhaustive_records(img, scales, 0.0, 64.0, 64,
                                                   kernel="epanechnikov", budget=10**9)
    err = np.abs(s.astype(np.float64) - rs) - (RTOL * np.maximum(np.abs(s), np.abs(rs)) + ATOL)
    assert err.max() <= 0.0
    assert (b != rb).sum() <= 2 and v == rv
    assert np.array_equal(m["position"][:, :2], rm[:, :2])


def test_epanechnikov_slab_pipeline_equals_whole_volume(sx, oracle):
    vol, _ = oracle.make_phantom(phantoms.ball_3d(48, (23.0, 25.0, 22.0), 9.0, 4))
    scales = [3.0, 5.0]
    full = sx.kadir_brady_exhaustive_records(vol, scales, 0, 64, 64, kernel="epanechnikov",
                                             budget=10**10)
    nz = vol.shape[0]
    s, b, m, _ = sx.kadir_brady_exhaustive_slab(vol[2:40], nz, 2, 9, 33, scales, 0, 64, 64,
                                                kernel="epanechnikov", budget=10**10)
    assert np.array_equal(s, full[0][9:33]) and np.array_equal(b, full[1][9:33])
    ident = sx.kadir_brady_exhaustive_records(vol, scales, 0, 64, 64, budget=10**10)
    assert not np.array_equal(ident[0], full[0])  # a different weighting, not the identity maps


def test_exhaustive_kernel_errors(sx):
    vol = np.zeros((16, 16, 16), np.float32)
    with pytest.raises(NotImplementedError, match="Gaussian"):
        sx.kadir_brady_exhaustive_records(vol, [3.0], 0, 1, 8, kernel="gaussian", budget=10**9)
    with pytest.raises(NotImplementedError, match="half-integer"):
        sx.kadir_brady_exhaustive_records(vol, [2.3, 3.3], 0, 1, 8, kernel="epanechnikov",
                                          budget=10**9)


@pytest.mark.parametrize("shape", [(130, 40, 37), (137, 24, 64), (64, 33, 20)])
def test_direct_form_two_chunks_ragged(sx, oracle, shape):
    """Volumes with >= 16 tile layers take the direct form's two chunks (the
    second a programmatic dependent of the first) with ragged x/y/z edges; the
    pinned-map result equals the pageable (staged) one and the oracle's maxima."""
    import torch

    rng = np.random.default_rng(sum(shape))
    vol = rng.uniform(-2.0, 34.0, size=shape).astype(np.float32)
    scales = [3.0, 4.0]
    nz, ny, nx = shape
    ref = sx.kadir_brady_exhaustive_slab(vol, nz, 0, 0, nz, scales, 0, 32, 32, budget=10**10)
    out = tuple(torch.empty(shape, dtype=torch.float32).pin_memory().numpy() for _ in range(2))
    got = sx.kadir_brady_exhaustive_slab(vol, nz, 0, 0, nz, scales, 0, 32, 32, budget=10**10,
                                         out=out)
    assert np.array_equal(got[0], ref[0]) and np.array_equal(got[1], ref[1])
    assert np.array_equal(got[2], ref[2])
    lin = oracle.local_maxima(got[0], got[1])[3]
    assert np.array_equal(got[2]["linear_index"], lin)


@pytest.mark.parametrize("window", [(-3.7, 29.3, 32), (0.0, 1.0, 16), (0.1, 64.3, 64)])
def test_bin_edges_exact(sx, oracle, window):
    """K1 bins through t' = (I - low) * (bins / range) and falls back to the
    reference's (I - low) / range * bins within 1e-9 of a bin edge: intensities
    on and one float ulp around every edge must bin exactly like the reference
    (any misbinned voxel changes the exact integer histograms, hence the maps)."""
    low, high, bins = window
    edges = low + np.arange(bins + 1) * (high - low) / bins
    e32 = edges.astype(np.float32)
    vals = np.concatenate([e32, np.nextafter(e32, np.float32(np.inf)),
                           np.nextafter(e32, np.float32(-np.inf))])
    rng = np.random.default_rng(bins)
    vol = rng.choice(vals, size=(20, 21, 24)).astype(np.float32)
    _check_maps(sx, oracle, vol, low, high, bins, [2.0, 3.0], mode="exact")


def test_last_maps_equal_the_call_maps(sx, oracle):
    """salvox_last_maps: the pass run with null maps keeps them on the device;
    fetching them afterwards (pageable and pinned buffers) gives the maps the
    call itself returns; a context with no exhaustive call is an error."""
    import ctypes as C

    import torch

    from paper_1310_6736_b200 import _lib

    vol, _ = oracle.make_phantom(phantoms.ball_3d(40, (20.0, 18.0, 21.0), 7.0, 9))
    ctx = sx.Context(0)
    s, b, m, v = sx.kadir_brady_exhaustive_records(vol, [3.0, 5.0], 0, 64, 64, budget=10**10,
                                                   ctx=ctx)
    lib = _lib.load()
    for pinned in (False, True):
        if pinned:
            ls, lb = (torch.empty(vol.shape, dtype=torch.float32).pin_memory().numpy()
                      for _ in range(2))
        else:
            ls, lb = np.empty(vol.shape, np.float32), np.empty(vol.shape, np.float32)
        _lib.check(lib.salvox_last_maps(ctx.handle, _lib.ptr(ls), _lib.ptr(lb)))
        assert np.array_equal(ls, s) and np.array_equal(lb, b)
    fresh = sx.Context(0)
    with pytest.raises(ValueError, match="no exhaustive call"):
        _lib.check(lib.salvox_last_maps(fresh.handle, C.c_void_p(0), C.c_void_p(0)))
    fresh.close()
    ctx.close()


def test_default_64_bins_match_the_reference(sx):
    """The reference's default window has 64 bins (volume.hpp:94): the 65-bin
    quad kernel (paired-voxel panels) against the reference's own
    kadir_brady_exhaustive (oracle/_ref) on a 3D phantom: maps within the
    tolerance, the same maxima positions, the same EvalCounter visits."""
    from oracle import ref as R

    if not R.available():
        pytest.skip("oracle/_ref/libsalvox_ref.so not built")
    vol = R.make_phantom(phantoms.ball_3d(36, (17.0, 18.0, 16.5), 7.0, 64,
                                         background={"type": "gaussian", "mean": 20.0,
                                                     "sigma": 6.0}))[0]
    scales = [3.0, 4.0, 5.0, 6.0]
    rs, rb, rm, rv = R.exhaustive(vol, 0.0, 64.0, 64, scales, budget=10**9)
    s, b, m, v = sx.kadir_brady_exhaustive_records(vol, scales, 0.0, 64.0, 64, budget=10**9)
    err = np.abs(s.astype(np.float64) - rs) - (RTOL * np.maximum(np.abs(s), np.abs(rs)) + ATOL)
    assert err.max() <= 0.0
    assert (b != rb).sum() <= max(2, vol.size // 5000) and v == rv
    assert np.array_equal(m["position"], rm[:, :3])
