"""The shift seek has three engines with identical arithmetic (DESIGN.md "Seed
kernels"): the CTA producer/consumer engine (few seeds), and the one-warp-per-
seed kernel in its latency and 80-register occupancy variants (many seeds).
The engine is picked by seed count, so the parity tests exercise whichever the
test size selects; here every shift parity test reruns with each engine forced
(SALVOX_SEEK_ENGINE, read once per process -> a subprocess per engine)."""
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.mark.parametrize("engine", ["cta", "warp", "warp12"])
def test_shift_parity_under_each_engine(engine):
    env = dict(os.environ, SALVOX_SEEK_ENGINE=engine)
    r = subprocess.run([sys.executable, "-m", "pytest", "-q", "-m", "gpu", "-k", "shift or detect or abmsod",
                        "tests/test_gpu_seek.py", "tests/test_gpu_edge.py", "tests/test_golden.py",
                        "tests/test_gpu_abmsod.py"],
                       cwd=ROOT, env=env, capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-2000:]
    assert " passed" in r.stdout


@pytest.mark.parametrize("variant", ["0", "2", "3"])
def test_exhaustive_kernel_variants_parity(variant):
    """The non-default exhaustive kernels (kb_kernel: 512 threads / register
    snapshots; kb_tmem_kernel: 1024 threads / TMEM snapshots; kb_quad_kernel
    without the offset doubles) stay exact: the exhaustive
    parity suites rerun with SALVOX_KB_VARIANT forced."""
    env = dict(os.environ, SALVOX_KB_VARIANT=variant)
    r = subprocess.run([sys.executable, "-m", "pytest", "-q", "-m", "gpu",
                        "tests/test_gpu_exhaustive.py", "tests/test_golden.py", "-k",
                        "exh or square or squares or histograms or slabs or scales or range"],
                       cwd=ROOT, env=env, capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-2000:]
    assert " passed" in r.stdout
