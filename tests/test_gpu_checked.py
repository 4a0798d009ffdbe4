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

# every builder path, every force kernel family (default lanes, index vectors, the ordered,
# half-cells and variant kernels), energy, and the step graphs -- a few minutes, not the full matrix
SUBSET = ("list or ordered or overflow or deferred or padding or counterexample or step_graph or rebuild or "
          "half_cells or variants_at or energy or interleaved or host_io")
NODES = ([f"tests/test_gpu_parity.py::test_force_parity[{lanes}-{half}-{cfg}]"
          for lanes in (0, 772, 66052) for half in (True, False) for cfg in (1, 3)]
         + [f"tests/test_gpu_cutoff.py::test_force_at_cutoff_edge[{half}-772]" for half in (False, True)])


def test_parity_suite_under_bounds_checks():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_1806_05713_b200 import build
    build.build()
    build.build(check=True)
    env = dict(os.environ, LJ_LIBRARY="check")
    for args in (["-k", SUBSET, "tests/test_gpu_parity.py", "tests/test_gpu_cutoff.py", "tests/test_gpu_md.py"],
                 NODES):
        cmd = [sys.executable, "-m", "pytest", "-q", "-m", "gpu", "-p", "no:cacheprovider", *args]
        r = subprocess.run(cmd, capture_output=True, text=True, timeout=2400, env=env, cwd=ROOT)
        assert r.returncode == 0, r.stdout[-4000:] + r.stderr[-2000:]
        assert " passed" in r.stdout
