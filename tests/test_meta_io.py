"""MetaImage IO (reference tests/test_volume.cpp:67-160 ported) on CPU, and the
on-device payload widening (salvox_upload_widen) bit-identical to the host
widening on the GPU."""
import os

import numpy as np
import pytest


def _write(dirp, name, header, payload):
    with open(os.path.join(dirp, name + ".raw"), "wb") as f:
        f.write(payload)
    p = os.path.join(dirp, name + ".mhd")
    with open(p, "w") as f:
        f.write(header)
    return p


def test_roundtrip_and_sizes(sx, tmp_path):  # test_volume.cpp:67-99
    rng = np.random.default_rng(17)
    v = rng.uniform(-100.0, 100.0, size=(5, 7, 9)).astype(np.float32)
    p = str(tmp_path / "roundtrip.mhd")
    sx.save_volume(v, p, spacing=(0.5, 0.75, 2.0))
    r, sp = sx.load_volume(p)
    assert r.shape == v.shape and np.array_equal(r, v)
    assert sp == (0.5, 0.75, 2.0)
    one = np.full((1, 1, 1), 42.0, np.float32)
    sx.save_volume(one, str(tmp_path / "one.mhd"))
    assert os.path.getsize(tmp_path / "one.raw") == 4
    assert sx.load_volume(str(tmp_path / "one.mhd"))[0][0, 0, 0] == 42.0
    sx.save_volume(np.zeros((34, 128, 128), np.float32), str(tmp_path / "large.mhd"))
    assert os.path.getsize(tmp_path / "large.raw") == 128 * 128 * 34 * 4


def test_widening_and_errors(sx, tmp_path):  # test_volume.cpp:101-160
    d = str(tmp_path)
    p = _write(d, "uc", "NDims = 3\nDimSize = 4 4 2\nElementType = MET_UCHAR\n"
               "ElementSpacing = 1 1 1\nBinaryDataByteOrderMSB = False\nElementDataFile = uc.raw\n",
               bytes(32))
    v, _ = sx.load_volume(p)
    assert v.shape == (2, 4, 4) and not v.any()
    p = _write(d, "sh", "NDims = 2\nDimSize = 2 2\nElementType = MET_SHORT\nElementDataFile = sh.raw\n",
               np.array([-5, 0, 7, 3000], np.int16).tobytes())
    v, _ = sx.load_volume(p)
    assert v.shape == (1, 2, 2) and v[0, 0, 0] == -5.0 and v[0, 1, 1] == 3000.0
    p = _write(d, "bad", "NDims = 3\nDimSize = 10 10 10\nElementType = MET_UCHAR\n"
               "ElementDataFile = bad.raw\n", bytes(999))
    with pytest.raises(RuntimeError, match="size mismatch"):
        sx.load_volume(p)
    with pytest.raises(RuntimeError):
        sx.load_volume(str(tmp_path / "nope.mhd"))
    p = _write(d, "dbl", "NDims = 3\nDimSize = 1 1 1\nElementType = MET_DOUBLE\n"
               "ElementDataFile = dbl.raw\n", bytes(8))
    with pytest.raises(RuntimeError, match="unsupported ElementType"):
        sx.load_volume(p)
    p = _write(d, "be", "NDims = 3\nDimSize = 1 1 1\nElementType = MET_FLOAT\n"
               "BinaryDataByteOrderMSB = True\nElementDataFile = be.raw\n", bytes(4))
    with pytest.raises(RuntimeError, match="big-endian"):
        sx.load_volume(p)


@pytest.mark.gpu
@pytest.mark.parametrize("etype,dt", [("MET_UCHAR", np.uint8), ("MET_SHORT", np.int16),
                                      ("MET_USHORT", np.uint16), ("MET_FLOAT", np.float32)])
def test_device_widening_bit_identical(sx, tmp_path, etype, dt):
    rng = np.random.default_rng(5)
    info = np.iinfo(dt) if np.issubdtype(dt, np.integer) else None
    shape = (37, 61, 53)  # odd sizes: the kernel's 4-wide tail
    if info is not None:
        data = rng.integers(info.min, info.max, size=shape, endpoint=True).astype(dt)
    else:
        data = rng.normal(0, 1000, size=shape).astype(dt)
    p = _write(str(tmp_path), "v", f"NDims = 3\nDimSize = {shape[2]} {shape[1]} {shape[0]}\n"
               f"ElementType = {etype}\nElementDataFile = v.raw\n", data.tobytes())
    host, sp = sx.load_volume(p)
    dev, sp2 = sx.load_volume_device(p)
    assert sp == sp2
    assert dev.cpu().numpy().tobytes() == host.tobytes()
