"""Memory-safety net (compute-sanitizer is closed on the pool and
there was no bounds-checked build): the GPU parity tests that exercise every
list builder path (fast, LARGE, exact, fallback, drifted storage, overflowing
padded rows), every force kernel and the MD step graphs are re-run against
liblj_check.so -- the same sources built with -DLJ_CHECK, whose kernels check
every gathered list index against the atom count, every staged candidate slot
and work item against its shared-memory bounds, and that the fill pass of a
compact list accepts exactly the count pass's entries, and trap otherwise (a
trap fails the test with a CUDA error)."""
import os
import subprocess
import sys

import pytest
import torch

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

SUBSET = ("list or force_parity or ordered or half_cells or overflow or deferred or padding or "
          "cutoff_edge or counterexample or graph or nve or rebuild or energy")


def test_parity_suite_under_bounds_checks():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_1806_05713_b200 import build
    build.build()
    build.build(check=True)
    env = dict(os.environ, LJ_LIBRARY="check")
    cmd = [sys.executable, "-m", "pytest", "-q", "-m", "gpu", "-p", "no:cacheprovider", "-k", SUBSET,
           os.path.join(ROOT, "tests", "test_gpu_parity.py"), os.path.join(ROOT, "tests", "test_gpu_cutoff.py"),
           os.path.join(ROOT, "tests", "test_gpu_md.py")]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=2400, env=env, cwd=ROOT)
    assert r.returncode == 0, r.stdout[-4000:] + r.stderr[-2000:]
    assert " passed" in r.stdout
