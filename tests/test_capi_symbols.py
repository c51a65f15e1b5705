"""The C-ABI boundary (include/*.h) on CPU: the in-tree library loads, exports every
declared symbol, and fails loudly (no CPU fallback) when no CUDA device exists."""
import ctypes
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _declared():
    names = []
    for h in ("salvox_capi.h", "salvox_bench.h"):
        text = open(os.path.join(ROOT, "include", h)).read()
        names += re.findall(r"^SALVOX_API\s+[\w\s\*]+?\b(salvox_\w+)\(", text, flags=re.M)
    return names


def test_library_exports_every_declared_symbol(sx):
    lib = sx._lib.load()
    names = _declared()
    assert len(names) >= 20
    for n in names:
        assert hasattr(lib, n), n
    assert set(names) == set(sx._lib.EXPORTS + sx._lib.BENCH_EXPORTS)
    assert lib.salvox_version() >= 100


def test_struct_layouts_match_header(sx, tmp_path):
    """ctypes / numpy mirrors have the C compiler's sizes and field offsets."""
    import subprocess

    src = tmp_path / "sizes.c"
    src.write_text("""
#include <stdio.h>
#include <stddef.h>
#include "salvox_capi.h"
int main(void) {
  printf("%zu %zu %zu %zu %zu %zu %zu %zu %zu %zu %zu %zu %zu %zu %zu %zu\\n", sizeof(salvox_window),
         sizeof(salvox_detection), sizeof(salvox_maximum), sizeof(salvox_detect_params),
         offsetof(salvox_detect_params, shift_target), offsetof(salvox_detection, flags),
         offsetof(salvox_detect_params, quadrant_scales),
         offsetof(salvox_detect_params, abmsod_target), sizeof(salvox_abmsod_params),
         offsetof(salvox_abmsod_params, target), sizeof(salvox_abmsod_iter),
         sizeof(salvox_window_op), offsetof(salvox_window_op, box), sizeof(salvox_window_result),
         sizeof(salvox_ascent_state), offsetof(salvox_ascent_state, displacement));
  return 0;
}
""")
    exe = tmp_path / "sizes"
    subprocess.run(["gcc", "-I", os.path.join(ROOT, "include"), str(src), "-o", str(exe)],
                   check=True)
    got = [int(v) for v in subprocess.run([str(exe)], capture_output=True, text=True,
                                          check=True).stdout.split()]
    P = sx._lib.DetectParams
    A = sx._lib.AbmsodParams
    assert got == [ctypes.sizeof(sx._lib.Window), sx.DET_DTYPE.itemsize, sx.MAX_DTYPE.itemsize,
                   ctypes.sizeof(P), P.shift_target.offset, sx.DET_DTYPE.fields["flags"][1],
                   P.quadrant_scales.offset, P.abmsod_target.offset, ctypes.sizeof(A),
                   A.target.offset, sx._lib.ABMSOD_ITER_DTYPE.itemsize,
                   sx._lib.WINDOW_OP_DTYPE.itemsize, sx._lib.WINDOW_OP_DTYPE.fields["box"][1],
                   sx._lib.WINDOW_RESULT_DTYPE.itemsize, sx._lib.ASCENT_STATE_DTYPE.itemsize,
                   sx._lib.ASCENT_STATE_DTYPE.fields["displacement"][1]]


def test_no_cpu_fallback_without_gpu(sx):
    import torch

    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    with pytest.raises(sx.SalvoxCudaError, match="no CPU fallback"):
        sx.Context(0)
