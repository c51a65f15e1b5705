"""The reference's OWN C++ test suite against the B200 drop-in API.

tests/cpp/Makefile compiles /root/reference/proj/tests/test_{volume,entropy,
seek,pipeline,cli}.cpp unmodified (where they lie) against include/salvox/*.hpp
+ cpp/libsalvox_host.so (the drop-in over libsalvox_b200.so) with a
doctest-compatible shim (tests/cpp/doctest_shim/doctest.h). The binaries are
built here by __graft_entry__.build() and travel to the GPU box; this file only
runs them.

GPU: every test case of every suite passes (86 cases: volume/IO, entropy and
candidate histograms, seek steps and trajectories, the exhaustive scan, detect,
Hu, reports, the CLI with our salvox-b200 standing in for the reference's
binary). CPU: every case either passes or fails only because there is no CUDA
device (the drop-in has no CPU fallback) -- argument validation, messages and
the host-side formats run without a GPU.
"""
import os
import re
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BUILD = os.path.join(ROOT, "tests", "cpp", "build")
SUITES = ["volume", "entropy", "seek", "pipeline", "cli"]


def _run(suite):
    exe = os.path.join(BUILD, "ref_test_" + suite)
    if not os.path.exists(exe):
        pytest.skip(f"{exe} not built (make -C tests/cpp ref_suite needs /root/reference)")
    env = dict(os.environ, SALVOX_CLI=os.path.join(ROOT, "cpp", "salvox-b200"))
    r = subprocess.run([exe], capture_output=True, text=True, timeout=600, env=env)
    m = re.search(r"test cases: (\d+) \| (\d+) passed \| (\d+) failed", r.stdout)
    assert m, r.stdout[-2000:] + r.stderr[-2000:]
    return r, int(m.group(1)), int(m.group(3))


@pytest.mark.gpu
@pytest.mark.parametrize("suite", SUITES)
def test_reference_suite_passes_on_device(suite):
    r, ran, failed = _run(suite)
    assert ran > 0 and failed == 0 and r.returncode == 0, r.stderr[-4000:]


@pytest.mark.parametrize("suite", ["volume", "entropy", "seek", "pipeline"])
def test_reference_suite_host_side_without_device(suite):
    import torch

    if torch.cuda.is_available():
        pytest.skip("device present: the GPU test covers this suite")
    r, ran, failed = _run(suite)
    assert ran > 0
    lines = r.stderr.splitlines()
    for i, ln in enumerate(lines):  # each failed check's next line says why: the device
        if "is NOT correct!" in ln:
            why = lines[i + 1] if i + 1 < len(lines) else ""
            assert "no CUDA device" in why, ln + "\n" + why
