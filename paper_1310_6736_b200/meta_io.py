"""MetaImage IO mirroring the reference's load_volume / save_volume
(src/meta_io.cpp:37-147, bindings/py_module.cpp:99-107): same accepted headers,
same error messages (RuntimeError for std::runtime_error). load_volume_device
keeps the payload at its native width across PCIe and widens it on the GPU
(salvox_upload_widen)."""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

from . import _lib

_TYPES = {"MET_UCHAR": (np.uint8, 0), "MET_SHORT": (np.int16, 1), "MET_USHORT": (np.uint16, 2),
          "MET_FLOAT": (np.float32, 3)}


def read_header(path):
    """Parses the .mhd header -> (dims (nx, ny, nz), spacing, ElementType, raw path)."""
    try:
        text = open(path).read()
    except OSError:
        raise RuntimeError("load_volume: cannot open " + str(path)) from None
    kv = {}
    for line in text.splitlines():
        if "=" not in line:
            continue
        k, v = line.split("=", 1)
        kv[k.strip()] = v.strip()
    ndims = int(kv.get("NDims", "3"))
    if ndims not in (2, 3):
        raise RuntimeError(f"load_volume: unsupported NDims {ndims}")
    if "DimSize" not in kv:
        raise RuntimeError("load_volume: missing DimSize")
    parts = kv["DimSize"].split()
    if len(parts) < ndims:
        raise RuntimeError("load_volume: bad DimSize")
    dims = [int(parts[i]) for i in range(ndims)] + [1] * (3 - ndims)
    spacing = [1.0, 1.0, 1.0]
    if "ElementSpacing" in kv:
        sp = kv["ElementSpacing"].split()
        if len(sp) < ndims:
            raise RuntimeError("load_volume: bad ElementSpacing")
        for i in range(ndims):
            spacing[i] = float(sp[i])
    if kv.get("BinaryDataByteOrderMSB", "false").lower() != "false":
        raise RuntimeError("load_volume: big-endian payloads are not supported")
    if kv.get("CompressedData", "false").lower() != "false":
        raise RuntimeError("load_volume: compressed payloads are not supported")
    if "ElementType" not in kv:
        raise RuntimeError("load_volume: missing ElementType")
    etype = kv["ElementType"]
    if etype not in _TYPES:
        raise RuntimeError("load_volume: unsupported ElementType " + etype)
    if "ElementDataFile" not in kv:
        raise RuntimeError("load_volume: missing ElementDataFile")
    if kv["ElementDataFile"].lower() == "local":
        raise RuntimeError("load_volume: inline (LOCAL) payloads are not supported")
    raw = os.path.join(os.path.dirname(os.path.abspath(path)), kv["ElementDataFile"])
    return tuple(dims), tuple(spacing), etype, raw


def _payload(path):
    dims, spacing, etype, raw = read_header(path)
    dt, code = _TYPES[etype]
    try:
        size = os.path.getsize(raw)
    except OSError:
        raise RuntimeError("load_volume: cannot open raw file " + raw) from None
    n = dims[0] * dims[1] * dims[2]
    if size != n * np.dtype(dt).itemsize:
        raise RuntimeError(f"load_volume: raw size mismatch, header implies "
                           f"{n * np.dtype(dt).itemsize} bytes but {os.path.basename(raw)} "
                           f"has {size}")
    data = np.fromfile(raw, dtype=dt, count=n)
    return dims, spacing, code, data


def load_volume(path):
    """load_volume (py_module.cpp:99-102) -> (array[z, y, x] float32, spacing)."""
    dims, spacing, _, data = _payload(path)
    return data.astype(np.float32).reshape(dims[2], dims[1], dims[0]), spacing


def load_volume_device(path, device=0, ctx=None):
    """load_volume with the payload widened on the GPU -> (torch CUDA tensor
    [z, y, x] float32, spacing). Bit-identical to load_volume."""
    import torch

    from .api import _ctx

    dims, spacing, code, data = _payload(path)
    out = torch.empty((dims[2], dims[1], dims[0]), dtype=torch.float32,
                      device=torch.device("cuda", device))
    c = _ctx(ctx)
    c.after_torch(out)
    raw = np.ascontiguousarray(data)
    _lib.check(_lib.load().salvox_upload_widen(c.handle, C.c_int32(code),
                                               raw.ctypes.data_as(C.c_void_p),
                                               C.c_int64(raw.size), C.c_void_p(out.data_ptr())))
    return out, spacing


def save_volume(volume, path, spacing=(1.0, 1.0, 1.0)):
    """save_volume (meta_io.cpp:119-147): little-endian MET_FLOAT .mhd/.raw pair."""
    v = np.ascontiguousarray(volume, dtype=np.float32)
    if v.ndim == 2:
        v = v[None]
    nz, ny, nx = v.shape
    root, _ = os.path.splitext(str(path))
    raw = root + ".raw"
    try:
        v.tofile(raw)
    except OSError:
        raise RuntimeError("save_volume: cannot write " + raw) from None

    def g(x):  # operator<< of a double (default stream precision 6)
        return f"{x:g}"

    with open(path, "w") as f:
        f.write("ObjectType = Image\nNDims = 3\nBinaryData = True\n"
                "BinaryDataByteOrderMSB = False\nCompressedData = False\n"
                f"DimSize = {nx} {ny} {nz}\n"
                f"ElementSpacing = {g(spacing[0])} {g(spacing[1])} {g(spacing[2])}\n"
                f"ElementType = MET_FLOAT\nElementDataFile = {os.path.basename(raw)}\n")
