"""The SURVEY 8(f) "next" rows against the reference ITSELF (oracle/_ref, the
reference's own sources compiled here), same inputs, same box:

  f2  phantom generation  make_phantom (phantom.cpp:237-294) of the C2 spec:
      reference (host; it also rasterises the four region masks, a few 10k
      voxels) vs make_phantom_device (volume + centroids, one launch chain)
  f2  MetaImage ingest    load_volume (meta_io.cpp:37-117) of the C2 volume stored
      as MET_SHORT: reference (read + widen on the host) vs load_volume_device
      (read raw bytes, H2D, widen on the device)
  f3  rasterisation       rasterize_window (pipeline.cpp:185-192) of 20 detection
      windows (r 10-20) on the 256^3 frame: reference (one frame for all) vs
      device (one call per window)
  f4  Hu filtering        hu_template_distance (pipeline.cpp:236-256) of 20
      detections x 5 axial crops against a 24x24 disk template: reference
      (one Volume for all detections) vs one device call for all crops (the
      volume upload included)

Every pair is checked for equality first (bit-identical outputs; the gaussian
phantom background within 1 float ulp). Prints one JSON object.
"""
import json
import os
import sys
import tempfile
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1310_6736_b200 as sx  # noqa: E402
from oracle import ref as R  # noqa: E402
from tests import phantoms  # noqa: E402


def best_of(fn, n=3, cuda=False):
    best, out = float("inf"), None
    for _ in range(n):
        if cuda:
            torch.cuda.synchronize()
        t0 = time.perf_counter()
        out = fn()
        if cuda:
            torch.cuda.synchronize()
        best = min(best, time.perf_counter() - t0)
    return best * 1e3, out


def main():
    if not R.available():
        print(json.dumps({"unavailable": "oracle/_ref/libsalvox_ref.so not built"}))
        return
    ctx = sx.Context(0)
    res = {}
    spec = phantoms.config_c2()
    ref_ms, (vref, _) = best_of(lambda: R.make_phantom(spec), n=2)
    dev_ms, (vdev, _) = best_of(lambda: sx.make_phantom_device(spec, ctx=ctx), cuda=True)
    d = vdev.cpu().numpy()
    ulp = np.abs(d.view(np.int32).astype(np.int64) - vref.view(np.int32).astype(np.int64)).max()
    res["phantom_c2"] = {"reference_ms": ref_ms, "device_ms": dev_ms, "speedup": ref_ms / dev_ms,
                         "max_float_ulp": int(ulp)}

    with tempfile.TemporaryDirectory() as tmp:
        raw = np.clip(np.rint(vref * 100.0), -32768, 32767).astype(np.int16)
        open(os.path.join(tmp, "c2.raw"), "wb").write(raw.tobytes())
        open(os.path.join(tmp, "c2.mhd"), "w").write(
            "NDims = 3\nDimSize = 256 256 256\nElementType = MET_SHORT\n"
            "ElementSpacing = 1 1 1\nElementDataFile = c2.raw\n")
        path = os.path.join(tmp, "c2.mhd")
        R.load_volume(path)  # page the file in for both sides
        ref_ms, (lr, _) = best_of(lambda: R.load_volume(path))
        dev_ms, (ld, _) = best_of(lambda: sx.load_volume_device(path, ctx=ctx), cuda=True)
        res["metaimage_short_c2"] = {"reference_ms": ref_ms, "device_ms": dev_ms,
                                     "speedup": ref_ms / dev_ms,
                                     "bit_identical": bool(ld.cpu().numpy().tobytes() == lr.tobytes()),
                                     "bytes": int(raw.nbytes)}

    rng = np.random.default_rng(3)
    wins = []
    for _ in range(20):
        c = rng.uniform(40, 216, size=3)
        A = rng.normal(size=(3, 3))
        H = A @ A.T + np.eye(3) * rng.uniform(100.0, 400.0)
        wins.append((c, H))
    shape = (256, 256, 256)
    cs = np.array([c for c, _ in wins])
    hs = np.array([H for _, H in wins])
    ref_ms, rcounts = best_of(lambda: R.rasterize_windows(shape, cs, hs))
    dev_ms, dr = best_of(lambda: [sx.rasterize_window(shape, c, H, ctx=ctx) for c, H in wins])
    exact = all(R.rasterize_window(shape, c, H).tobytes() == d.tobytes()
                for (c, H), d in zip(wins[:4], dr[:4]))
    res["rasterize_20_windows_256"] = {
        "reference_ms": ref_ms, "device_ms": dev_ms, "speedup": ref_ms / dev_ms,
        "counts_equal": bool(np.array_equal(rcounts, [len(d) for d in dr])),
        "first_4_bit_identical": bool(exact), "voxels": int(rcounts.sum())}

    y, x = np.mgrid[0:24, 0:24]
    tmpl = np.where((x - 11.5) ** 2 + (y - 11.5) ** 2 <= 81.0, 40.0, 0.0).astype(np.float32)
    dets = np.zeros(20, sx.DET_DTYPE)
    for i, (c, H) in enumerate(wins):
        dets[i]["center"] = c
        dets[i]["H"] = np.diag(np.diag(H)).reshape(9)
    ref_ms, hr = best_of(lambda: R.hu_template_distances(vref, dets["center"], dets["H"], tmpl))
    dev_ms, hd = best_of(lambda: sx.hu_template_distance(dets, vref, tmpl, ctx=ctx))
    res["hu_template_20_dets"] = {"reference_ms": ref_ms, "device_ms": dev_ms,
                                  "speedup": ref_ms / dev_ms,
                                  "max_rel_diff": float(np.max(np.abs(hd - hr) /
                                                               np.maximum(np.abs(hr), 1e-300)))}
    res["host_cores"] = os.cpu_count()
    print(json.dumps(res))


if __name__ == "__main__":
    main()
