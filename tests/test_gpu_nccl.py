"""The NCCL path of the multi-GPU driver on the GPU (VERDICT r01 "no -m gpu test
runs NCCL"): tests/nccl_md_worker.py under torch.distributed.run, one rank per
visible GPU (1 on the test pool, with LJ_FORCE_COLLECTIVES=1 so that every
collective of the P > 1 step is issued)."""
import json
import os
import socket
import subprocess
import sys

import pytest
import torch

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


@pytest.fixture(scope="module")
def result():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_1806_05713_b200 import build
    build.build()
    env = dict(os.environ, LJ_FORCE_COLLECTIVES="1", TORCH_NCCL_ASYNC_ERROR_HANDLING="1")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=1",
           "--master-addr", "127.0.0.1", "--master-port", str(_free_port()),
           os.path.join(ROOT, "tests", "nccl_md_worker.py")]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=900, env=env, cwd=ROOT)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
    line = [x for x in r.stdout.splitlines() if x.startswith("{")][-1]
    return json.loads(line)


def test_nccl_process_group(result):
    assert result["backend"] == "nccl" and result["collective"]


def test_eager_nccl_steps_match_oracle(result):
    assert result["energy_points"]
    assert result["energy_start_rel"] <= 1e-12
    assert result["energy_first10_max_rel"] <= 1e-9
    ours, ref = result["rebuilds"]
    assert abs(ours - ref) <= 3


@pytest.mark.parametrize("tag", ["resort", "fixed"])
def test_captured_multirank_step_equals_eager(result, tag):
    assert result[f"graph_rebuilds_{tag}"] >= 3
    assert result[f"graph_equals_eager_{tag}"]
    assert result[f"graph_interactions_equal_{tag}"]


def test_async_allgather_overlap_equals_blocking(result):
    assert result["overlap_active"]
    assert result["overlap_equals_blocking"]
