#!/usr/bin/env python3
"""bench.py -- headline benchmark of the B200 hot path (BASELINE.json configs[1]).

Workload: exhaustive Kadir-Brady saliency on the 256^3 synthetic C2 phantom
(gaussian background + 3 balls + 1 box, uniform fills, 32 bins),
13 scales 3..15, per-voxel best scale + strict-maxima selection. One step = one
full pass (bin pre-pass, kb_kernel, maxima, sort). Metric: voxel-scale entropy
evaluations per second (nx*ny*nz*13 per pass).

  python bench.py [--gpus N --steps K --warmup W]            # B200 arm
  python bench.py --impl reference [--steps K --warmup W]     # CPU reference arm

N > 1 runs under torchrun with WEAK scaling: every rank owns one C2-sized slab
(256^3 voxels) of a volume that grows with N -- 256x256x512 at N=2, 256x512x512
at N=4 and the 512^3 C4 phantom (BASELINE.json configs[3]) at N=8 -- z-slab
sharded with read-only halos; each rank scores only its owned planes, swaps one
boundary score plane with each neighbour (NCCL send/recv) for the strict-maxima
test, and the per-slab maxima meet in one NCCL all-gather
(paper_1310_6736_b200/sharding.py).
`value` times the device-resident pass (CUDA events on the launching stream,
L2 flushed between steps, max over ranks); `e2e` times the public API call with
the pinned host volume in and the maps + maxima out. The roofline denominator is
the shared-memory update peak measured live by salvox_probe_smem_peak (the pass
is bound by shared-memory atomics, not HBM or tensor cores -- DESIGN.md).
"""
from __future__ import annotations

import argparse
import gc
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

SCALES = [float(s) for s in range(3, 16)]
BINS = 32
LOW, HIGH = 0.0, 32.0  # window [0, 32), SURVEY.md 8(d) C2
METRIC = "voxel-scale entropy evals/sec (exhaustive); 256³ seed-grid volumes/sec"
UNIT = "voxel-scale evals/s"
# the 3D exhaustive kernel the library picks (csrc/exhaustive.cu pick_tile; A/B knob SALVOX_KB_VARIANT)
KB_KERNEL = {"0": "kb_kernel", "1": "kb_pair_kernel", "2": "kb_tmem_kernel"}.get(
    os.environ.get("SALVOX_KB_VARIANT", "4"), "kb_quad_kernel")


def c2_spec():
    from tests import phantoms
    return phantoms.config_c2()


def weak_spec(world):
    """The whole-job volume at N ranks: N x 256^3 voxels, so each rank's slab holds
    as many voxels as the N=1 workload. N=1 is C2 itself and N=8 the C4 512^3
    phantom; other N stack C2's region layout once per 256^3 block."""
    from tests import phantoms
    if world == 1:
        return phantoms.config_c2()
    if world == 8:
        return phantoms.config_c4()
    dims = {2: [256, 256, 512], 4: [256, 512, 512]}.get(world, [256, 256, 256 * world])
    base = phantoms.config_c2()
    regs = []
    for bz in range(dims[2] // 256):
        for by in range(dims[1] // 256):
            for bx in range(dims[0] // 256):
                for r in base["regions"]:
                    q = dict(r)
                    q["center"] = [r["center"][0] + 256 * bx, r["center"][1] + 256 * by,
                                   r["center"][2] + 256 * bz]
                    regs.append(q)
    return {"dims": dims, "background": base["background"], "regions": regs,
            "rng_seed": base["rng_seed"]}


def weak_workload(world, dims):
    nx, ny, nz = dims
    if world == 1:
        return ("exhaustive Kadir-Brady saliency, 256^3 C2 phantom (BASELINE.json configs[1]), "
                "32 bins, scales 3..15, per-voxel best scale + strict maxima")
    name = "512^3 C4 phantom (BASELINE.json configs[3])" if world == 8 else \
        f"{nx}x{ny}x{nz} phantom (C2 regions per 256^3 block)"
    return (f"exhaustive Kadir-Brady saliency, {name}, z-slab sharded over {world} GPUs "
            f"(one 256^3-voxel slab per GPU), 32 bins, scales 3..15, per-voxel best scale "
            f"+ strict maxima")


def c3_spec():
    from tests import phantoms
    return phantoms.config_c3()


# ------------------------------------------------------------------ clocks
class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index=0):
        self.index = index
        self.proc = None
        self.lines = []

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "200"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except OSError:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *a):
        if self.proc is not None:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()

    def summary(self):
        sm, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 8:
                continue
            try:
                sm.append(float(parts[0]))
                mx = float(parts[1])
            except ValueError:
                continue
            for n, v in zip(names, parts[4:8]):
                if v.lower().startswith("active"):
                    reasons.add(n)
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": mx,
                "reasons": sorted(reasons), "samples": len(sm)}


# ------------------------------------------------------------------ reference arm
def cpu_sample_run(vol, threads, planes):
    """The oracle's literal restatement of pipeline.cpp:63-166 (fp64, the reference's loop
    order; its maps are bit-identical to the reference's own, tests/test_ref_pin.py) on a
    bounded sample: `planes` full central z-planes of the same volume, split row-wise over
    `threads` host threads."""
    from oracle import oracle as O
    nz, ny, nx = vol.shape
    z0 = nz // 2 - planes // 2
    t0 = time.perf_counter()
    O.exhaustive(vol, LOW, HIGH, BINS, SCALES, budget=10**15, mode="literal", threads=threads,
                 z_range=(z0, z0 + planes))
    dt = time.perf_counter() - t0
    evals = nx * ny * planes * len(SCALES)
    return evals / dt, (f"{nx}x{ny}x{nz} volume, planes z={z0}..{z0 + planes - 1} "
                        f"({nx * ny * planes} voxels x 13 scales, {dt:.1f} s)")


def reference_calibration(vol, n=16):
    """The timed port against the reference ITSELF (oracle/_ref/libsalvox_ref.so: the
    reference's own pipeline.cpp compiled here) on the same whole n^3 sub-volume, one
    thread each: the maps must be bit-identical and the ratio says how the port's
    speed relates to the reference's (the reference's exhaustive pass is
    single-threaded; the port's plane samples are what the arm can afford)."""
    from oracle import oracle as O
    from oracle import ref as R
    if not R.available():
        return {"available": False, "why": "oracle/_ref/libsalvox_ref.so not built"}
    nz, ny, nx = vol.shape
    c = np.ascontiguousarray(vol[nz // 2 - n // 2: nz // 2 + n // 2,
                                 ny // 2 - n // 2: ny // 2 + n // 2,
                                 nx // 2 - n // 2: nx // 2 + n // 2])
    tr = tp = float("inf")
    for _ in range(2):  # alternating, best of 2 each (shared host cores are noisy)
        t0 = time.perf_counter()
        rs, rb, _, _ = R.exhaustive(c, LOW, HIGH, BINS, SCALES, budget=10**15)
        tr = min(tr, time.perf_counter() - t0)
        t0 = time.perf_counter()
        ps, pb, _ = O.exhaustive(c, LOW, HIGH, BINS, SCALES, budget=10**15, mode="literal",
                                 threads=1)
        tp = min(tp, time.perf_counter() - t0)
    evals = c.size * len(SCALES)
    return {"sample": f"central {n}^3 sub-volume of the same volume, whole-volume call, 1 thread",
            "reference_evals_per_s": evals / tr, "port_evals_per_s": evals / tp,
            "port_speed_over_reference": tr / tp,
            "maps_bit_identical": bool(rs.tobytes() == ps.tobytes() and
                                       rb.tobytes() == pb.tobytes())}


def reference_seed_grid(steps, threads):
    """The reference's own detect() (oracle/_ref; pipeline.cpp:311-402, shift, its
    parallel_for over `threads` workers) on the C3 seed grid: volumes/s."""
    from oracle import ref as R
    if not R.available():
        return None
    vol, _ = R.make_phantom(c3_spec())
    kw = dict(method="shift", seed_spacing=16.0, scales=[8.0, 12.0], top_k=20, dedupe_radius=5.0,
              workers=threads)
    R.detect(vol, 0.0, 64.0, 64, **kw)
    times = []
    for _ in range(steps):
        t0 = time.perf_counter()
        sel, _ = R.detect(vol, 0.0, 64.0, 64, **kw)
        times.append(time.perf_counter() - t0)
    ms = float(np.mean(times)) * 1e3
    return {"metric": "seed-grid volumes/sec", "value": 1e3 / ms, "unit": "volumes/s",
            "ms_per_volume": ms, "kind": "reference", "cores": threads,
            "config": {"workload": "C3 256x256x160 MR phantom, shift mean-shift, 64 bins, "
                                   "lattice 16 x scales {8, 12} = 5120 seeds",
                       "selected": int(len(sel))}}


def run_reference(args, rank, world):
    if rank != 0:
        return
    from paper_1310_6736_b200 import api
    vol, _ = api.make_phantom(weak_spec(world))
    threads = os.cpu_count() or 1
    # ~4-8 s per step on the box's cores: threads/4 planes of 256^2 voxels
    planes = max(1, (threads // 4) * 65536 // (vol.shape[1] * vol.shape[2]))
    for _ in range(min(args.warmup, 1)):
        cpu_sample_run(vol, threads, 1)
    vals = []
    for _ in range(args.steps):
        v, sample = cpu_sample_run(vol, threads, planes)
        vals.append(v)
    value = float(np.mean(vals))
    total_evals = float(np.prod(vol.shape)) * len(SCALES)
    cal = reference_calibration(vol)
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": total_evals / value * 1e3, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": weak_workload(world, vol.shape[::-1]),
                   "sample_per_step": sample},
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": threads, "kind": "port",
                         "sample": sample, "reference_calibration": cal},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "note": "the reference's exhaustive pass (pipeline.cpp:63-166) is single-threaded and "
                "can only score whole volumes, so each step times the literal port "
                "(oracle/salvox_oracle.c: fp64, the reference's loop order, bit-identical maps) "
                "on a plane sample of the same volume on ALL of rank 0's host cores; "
                "reference_calibration times the reference itself (oracle/_ref, compiled from "
                "its own sources) against the port on one identical sub-volume, single-threaded "
                "(port_speed_over_reference > 1: this arm overstates the reference). "
                "ms_per_step extrapolates the sample to one full pass",
    }
    sg = reference_seed_grid(3, threads)
    if sg is not None:
        line["seed_grid"] = sg
    print(json.dumps(line), flush=True)


# ------------------------------------------------------------------ B200 arm
def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-seed-grid", action="store_true")
    args = ap.parse_args()
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))

    import torch
    import torch.distributed as dist

    # SALVOX_BENCH_FUNCTIONAL=1: ranks share the visible GPUs round-robin over gloo
    # -- a functional check of the N>1 orchestration on a 1-GPU box, never a
    # measurement (tools/mgpu_functional.sh)
    functional = os.environ.get("SALVOX_BENCH_FUNCTIONAL") == "1"
    if functional and args.impl == "b200":
        local = local % max(torch.cuda.device_count(), 1)
    if world > 1:
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        if args.impl == "b200" and not functional:
            torch.cuda.set_device(local)
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:
            dist.init_process_group("gloo")
    if args.impl == "reference":
        run_reference(args, rank, world)
        if world > 1:
            dist.destroy_process_group()
        return

    import paper_1310_6736_b200 as sx
    from paper_1310_6736_b200 import api, sharding
    from paper_1310_6736_b200._lib import Context

    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    stream = torch.cuda.current_stream(dev)
    ctx = Context(local)
    ctx.set_stream(stream.cuda_stream)

    vol, _ = api.make_phantom(weak_spec(world))
    nz, ny, nx = vol.shape
    R = sharding.halo_radius(SCALES)
    z0, z1, zs0, zs1 = sharding.slab_bounds(nz, world, rank, R)
    total_evals = float(nx * ny * nz * len(SCALES))
    budget = 10**15


    # ---- value: device-resident slab, events on the launching stream
    slab_host = torch.from_numpy(np.ascontiguousarray(vol[zs0:zs1])).pin_memory()
    d_slab = slab_host.to(dev, non_blocking=True)
    d_score = torch.empty((z1 - z0, ny, nx), dtype=torch.float32, device=dev)
    d_best = torch.empty_like(d_score)
    flush = torch.empty(int(256 * 2**20), dtype=torch.uint8, device=dev)  # > 126 MB L2
    from paper_1310_6736_b200 import _lib
    import ctypes as C
    sc = np.asarray(SCALES, np.float64)
    iw = _lib.Window(LOW, HIGH, BINS, 0)
    nmax = C.c_int64(0)

    def device_pass():
        if world > 1:  # owned planes only + one boundary plane each way, then the all-gather
            sharding.exhaustive_exchange(vol, SCALES, LOW, HIGH, BINS, budget=budget, device=dev,
                                         ctx=ctx, out=(d_score, d_best), d_slab=d_slab)
            return
        _lib.check(_lib.load().salvox_exhaustive_slab_device(
            ctx.handle, C.c_void_p(d_slab.data_ptr()), nx, ny, nz, zs0, zs1, z0, z1, C.byref(iw),
            sc.ctypes.data_as(C.c_void_p), len(sc), 0, budget, C.c_void_p(d_score.data_ptr()),
            C.c_void_p(d_best.data_ptr()), C.byref(nmax)))

    for _ in range(args.warmup):
        device_pass()
    torch.cuda.synchronize(dev)
    # live roofline denominator (same GPU, same run; after the warm-up passes so
    # the clocks have ramped; best of 3 trials per probe layout)
    peak_atoms, peak_lds, peak_atoms_only = ctx.probe_smem_peak(64)
    peak_prmt = ctx.probe_prmt_rate()
    if world > 1:
        dist.barrier()
    ctx.set_profiling(True)
    launches0 = ctx.launch_count()
    times = []
    with ClockSampler(local) as clk:
        for _ in range(args.steps):
            flush.fill_(1)  # L2 flush between timed steps (outside the events)
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            device_pass()
            e1.record(stream)
            e1.synchronize()
            times.append(e0.elapsed_time(e1))
    torch.cuda.synchronize(dev)
    launches = ctx.launch_count() - launches0
    kb_ms, kb_n, kb_updates = ctx.kernel_time()
    ctx.set_profiling(False)
    ms_local = float(np.mean(times))
    ms = ms_local
    if world > 1:
        t = torch.tensor([ms_local], dtype=torch.float64, device="cpu" if functional else dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
        dist.barrier()
    value = total_evals / (ms * 1e-3)

    # ---- e2e: public API (host pinned volume in, maps + maxima out), sharded over ranks
    vol_pinned = torch.from_numpy(vol).pin_memory().numpy()
    out_pinned = (torch.empty((z1 - z0, ny, nx), dtype=torch.float32).pin_memory().numpy(),
                  torch.empty((z1 - z0, ny, nx), dtype=torch.float32).pin_memory().numpy())
    h2d = (zs1 - zs0) * ny * nx * 4
    # pinned buffer for the (merged, whole-volume) maxima list: ~2.9% of the voxels
    # of these phantoms are strict maxima; a bigger list falls back to pageable memory
    max_pinned = torch.empty((nx * ny * nz // 24 + 4096) * sx.MAX_DTYPE.itemsize,
                             dtype=torch.uint8).pin_memory().numpy().view(sx.MAX_DTYPE)
    e2e_times, d2h = [], 0
    gc.collect()  # start the loop with a clean heap (no gen-2 pass inherited from setup)
    for i in range(args.warmup + args.steps):
        torch.cuda.synchronize(dev)
        if world > 1:
            dist.barrier()
        t0 = time.perf_counter()
        if world > 1:
            score, best, (oz0, oz1), merged, _ = sharding.exhaustive_exchange(
                vol_pinned, SCALES, LOW, HIGH, BINS, budget=budget, device=dev, ctx=ctx,
                out=out_pinned, maxima_out=max_pinned)
        else:
            score, best, (oz0, oz1), merged, _ = sharding.exhaustive_sharded(
                vol_pinned, SCALES, LOW, HIGH, BINS, budget=budget, ctx=ctx, out=out_pinned,
                maxima_out=max_pinned)
        t1 = time.perf_counter()
        if i >= args.warmup:
            e2e_times.append((t1 - t0) * 1e3)
            d2h = score.nbytes + best.nbytes + len(merged) * sx.MAX_DTYPE.itemsize
    e2e_ms = float(np.mean(e2e_times))
    if world > 1:
        t = torch.tensor([e2e_ms], dtype=torch.float64, device="cpu" if functional else dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e2e_ms = float(t.item())

    # ---- secondary: 256x256x160 seed-grid (shift, 64 bins) volumes/s, device-resident
    seed_grid = abmsod = None
    if not args.no_seed_grid and rank == 0:
        seed_grid = bench_seed_grid(ctx, dev, stream, flush)
        abmsod = bench_abmsod_paper(ctx, dev, stream, flush)

    # ---- cpu baseline (rank 0, N = 1 only)
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        threads = os.cpu_count() or 1
        val, sample = cpu_sample_run(vol, threads, threads)
        cpu = {"value": val, "unit": UNIT, "cores": threads, "kind": "port", "sample": sample,
               "reference_calibration": reference_calibration(vol)}

    if rank == 0:
        achieved = kb_updates / (kb_ms * 1e-3) if kb_ms > 0 else None
        traffic = None
        prof_d = {}
        prof = os.path.join(ROOT, "profiles", "kb_kernel_ncu.json")  # the default kernel's ncu capture
        if os.path.exists(prof):
            try:
                prof_d = json.load(open(prof))
                traffic = prof_d.get("dram_bytes_per_launch")
            except Exception:
                prof_d, traffic = {}, None
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "u32",
            "data": "synthetic",
            "config": {"workload": weak_workload(world, (nx, ny, nz)),
                       "dims": [nx, ny, nz],
                       "voxels": nx * ny * nz, "scales": len(SCALES),
                       "evals_per_pass": total_evals, "parallelism": f"z-slab x{world}",
                       "l2": "flushed between timed steps (256 MiB write)"},
            "e2e": {"value": total_evals / (e2e_ms * 1e-3), "unit": UNIT,
                    "h2d_bytes_per_step": h2d * world, "d2h_bytes_per_step": d2h * world,
                    "ms_per_step": e2e_ms, "ms_min": float(np.min(e2e_times)),
                    "ms_max": float(np.max(e2e_times))},
            "roofline": {"bound": "smem", "achieved": achieved, "peak": peak_atoms_only,
                         "unit": "histogram updates/s",
                         "frac": (achieved / peak_atoms_only) if achieved else None,
                         "traffic": traffic, "kernel": KB_KERNEL,
                         "kb_ms_per_launch": kb_ms / max(kb_n, 1),
                         "updates_per_launch": kb_updates / max(kb_n, 1),
                         "peak_source": "live salvox_probe_smem_peak: the highest shared-memory "
                                        "atomic rate demonstrated on this GPU (ATOMS only, bins "
                                        "from registers; best of 3 trials of each of the "
                                        "1-column/1024-thread, 1-column/512-thread, "
                                        "4-column/256-thread and kb_quad_kernel-walk-without-"
                                        "loads layouts) -- every update is at least one atomic; "
                                        "not in MEASURED_PEAKS.json",
                         "smem_pipe_util_ncu": (prof_d.get("smem_pipe_pct_of_peak_elapsed", 0.0) / 100.0
                                                if prof_d else None),
                         "smem_wavefronts_per_update_ncu": prof_d.get("wavefronts_per_warp_update"),
                         "pair_peak": peak_atoms,
                         "frac_of_pair_peak": (achieved / peak_atoms) if achieved else None,
                         "lds_only_peak": peak_lds,
                         "atoms_prmt_walk_peak": peak_prmt},
            "gpu_launches": launches,
            "clocks": clk.summary(),
        }
        if cpu is not None:
            line["cpu_baseline"] = cpu
        if seed_grid is not None:
            line["seed_grid"] = seed_grid
        if abmsod is not None:
            line["abmsod_paper"] = abmsod
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


def bench_seed_grid(ctx, dev, stream, flush, steps=3):
    """C3 (256x256x160 MR phantom, 64 bins, shift, lattice 16 x scales {8, 12}) volumes/s."""
    import ctypes as C

    import torch

    from paper_1310_6736_b200 import _lib, api

    vol, _ = api.make_phantom(c3_spec())
    d_vol = torch.from_numpy(vol).to(dev)
    iw = _lib.Window(0.0, 64.0, 64, 0)
    P, keep = api._detect_params("shift", seed_spacing=16.0, scales=(8.0, 12.0), k=20,
                                 dedupe_radius=5.0)
    out = np.empty(20, _lib.DET_DTYPE)
    n_out = np.zeros(1, np.int64)
    visits = C.c_uint64(0)
    nz, ny, nx = vol.shape

    def run():
        _lib.check(_lib.load().salvox_detect_batch_device(
            ctx.handle, C.c_void_p(d_vol.data_ptr()), 1, nx, ny, nz, C.byref(iw), C.byref(P),
            out.ctypes.data_as(C.c_void_p), 20, n_out.ctypes.data_as(C.c_void_p),
            C.byref(visits)))

    run()
    times = []
    for _ in range(steps):
        flush.fill_(1)
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        run()
        e1.record(stream)
        e1.synchronize()
        times.append(e0.elapsed_time(e1))
    ms = float(np.mean(times))
    del keep
    return {"metric": "seed-grid volumes/sec", "value": 1e3 / ms, "unit": "volumes/s",
            "ms_per_volume": ms,
            "config": {"workload": "C3 256x256x160 MR phantom, shift mean-shift, 64 bins, "
                                   "lattice 16 x scales {8, 12} = 5120 seeds",
                       "selected": int(n_out[0])}}


def bench_abmsod_paper(ctx, dev, stream, flush, steps=3):
    """ABMSOD detect (the paper's own GPU workload) on the paper's
    volume shapes: PET 128x128x34 / 400 random seeds / 16 bins and MR 256x256x176 /
    700 random seeds / 64 bins, isotropic seed windows r = 8, device-resident volume,
    selection included. The paper: 4.1 s and 7.8 s per volume on a Tesla C2050
    (PAPER.md:264, :290)."""
    import ctypes as C

    import torch

    from paper_1310_6736_b200 import _lib, api

    sys.path.insert(0, ROOT)
    from tests import phantoms

    out_cases = {}
    for name, spec, bins, n_seeds, paper_s in (("pet_128x128x34_400", phantoms.paper_pet(), 16,
                                                400, 4.1),
                                               ("mr_256x256x176_700", phantoms.paper_mr(), 64,
                                                700, 7.8)):
        vol, _ = api.make_phantom(spec)
        d_vol = torch.from_numpy(vol).to(dev)
        iw = _lib.Window(0.0, float(bins), bins, 0)
        P, keep = api._detect_params("abmsod", scales=(8.0,), k=20, dedupe_radius=5.0,
                                     seed_mode="random", seed_count=n_seeds, rng_seed=1310)
        out = np.empty(20, _lib.DET_DTYPE)
        n_out = np.zeros(1, np.int64)
        visits = C.c_uint64(0)
        nz, ny, nx = vol.shape

        def run():
            _lib.check(_lib.load().salvox_detect_batch_device(
                ctx.handle, C.c_void_p(d_vol.data_ptr()), 1, nx, ny, nz, C.byref(iw), C.byref(P),
                out.ctypes.data_as(C.c_void_p), 20, n_out.ctypes.data_as(C.c_void_p),
                C.byref(visits)))

        run()
        times = []
        for _ in range(steps):
            flush.fill_(1)
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            run()
            e1.record(stream)
            e1.synchronize()
            times.append(e0.elapsed_time(e1))
        ms = float(np.mean(times))
        del keep
        out_cases[name] = {"ms_per_volume": ms, "volumes_per_s": 1e3 / ms, "seeds": n_seeds,
                           "bins": bins, "selected": int(n_out[0]),
                           "paper_c2050_s_per_volume": paper_s,
                           "speedup_vs_paper_c2050": paper_s * 1e3 / ms}
    return {"metric": "ABMSOD detect volumes/sec (paper shapes)", "unit": "volumes/s",
            "cases": out_cases}


if __name__ == "__main__":
    main()
