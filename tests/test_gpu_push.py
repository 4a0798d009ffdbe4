"""lj_integrate_push (fused drift + NVLink push) on one GPU.

1. Emulated ranks (one process, as B200_PROFILING.md asks for multi-rank device
   logic on fewer GPUs): the replicas of three "peers" are plain buffers on the
   same device; the pushed rows must equal the drifted rows bit for bit, every
   other row is untouched, and q_out / the displacement are bit-identical to
   lj_integrate + lj_max_displacement.
2. The CUDA IPC plumbing with two real processes on the same GPU: process 0
   exports a buffer (lj_ipc_get_handle), process 1 maps it (lj_ipc_open) and
   pushes into it; process 0 reads the rows back after a host barrier.  No
   kernel waits on another process's kernel.
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def lj():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_1806_05713_b200 import build, lj as _lj
    build.build()
    _lj.load()
    return _lj


def _records(lj, rng, n, scale=10.0):
    x = torch.from_numpy(rng.uniform(0, scale, (n, 3))).cuda()
    r = lj.pack_aos4(x)
    r[:, 3] = torch.from_numpy(rng.normal(size=n)).cuda()     # pads must be carried, never used
    return r


@pytest.mark.parametrize("inplace", [False, True])
def test_push_emulated_ranks(lj, inplace):
    rng = np.random.default_rng(11)
    n, dt = 50_000, 0.01
    q = _records(lj, rng, n)
    p = _records(lj, rng, n, 1.0)
    q_ref = q.clone()
    q_ref[:, :3] += torch.from_numpy(rng.normal(0, 0.05, (n, 3))).cuda()
    b, e = 10_000, 30_007                                      # this rank's rows
    peers = [torch.full((n, 4), -7.0, dtype=torch.float64, device="cuda") for _ in range(3)]
    ranges = [(b, b + 1234), (e - 999, e), (b + 5000, b + 5001)]
    targets = [(t.data_ptr(), lo, hi) for t, (lo, hi) in zip(peers, ranges)]
    q_out = q if inplace else torch.zeros_like(q)
    q_in = q if inplace else q.clone()
    out = torch.zeros(1, dtype=torch.float64, device="cuda")
    # reference: the unfused calls
    q_a = q.clone()
    lj.integrate(q_a, p, dt, b, e)
    d_a = torch.zeros(1, dtype=torch.float64, device="cuda")
    lj.max_displacement(q_a, q_ref, b, e, d_a)
    lj.integrate_push(q_in, q_out, p, q_ref, dt, b, e, out, targets)
    torch.cuda.synchronize()
    assert torch.equal(q_out[b:e], q_a[b:e])
    if not inplace:
        assert torch.equal(q_out[:b], torch.zeros_like(q_out[:b])) and torch.equal(q_out[e:], torch.zeros_like(q_out[e:]))
        assert torch.equal(q_in, q)
    assert out.item() == d_a.item()
    for t, (lo, hi) in zip(peers, ranges):
        assert torch.equal(t[lo:hi], q_a[lo:hi])
        assert bool((t[:lo] == -7.0).all()) and bool((t[hi:] == -7.0).all())


def test_push_no_targets_is_integrate_displacement(lj):
    rng = np.random.default_rng(12)
    n = 4096
    q, p = _records(lj, rng, n), _records(lj, rng, n, 1.0)
    q_ref = q.clone()
    a, b = q.clone(), q.clone()
    o1, o2 = (torch.zeros(1, dtype=torch.float64, device="cuda") for _ in range(2))
    lj.integrate_push(a, a, p, q_ref, 0.005, 0, n, o1, [])
    lj.integrate_displacement(b, p, q_ref, 0.005, 0, n, o2)
    assert torch.equal(a, b) and o1.item() == o2.item()


def _ipc_worker(rank, port, outdir):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=2)
    try:
        from paper_1806_05713_b200 import lj
        torch.cuda.set_device(0)
        n, lo, hi = 20_000, 3_000, 7_500
        rng = np.random.default_rng(5)
        if rank == 0:
            buf = torch.full((n, 4), -1.0, dtype=torch.float64, device="cuda")
            torch.cuda.synchronize()
            h = [lj.ipc_handle(buf[100:])]                       # an offset view of the allocation
            dist.broadcast_object_list(h, src=0)
            dist.barrier()                                     # process 1 has pushed and synchronised
            got = buf[100:].cpu().numpy()
            np.save(os.path.join(outdir, "got.npy"), got)
            dist.barrier()
        else:
            h = [None]
            dist.broadcast_object_list(h, src=0)
            ptr = lj.ipc_open(*h[0])
            q = lj.pack_aos4(torch.from_numpy(rng.uniform(0, 10, (n, 3))).cuda())
            p = lj.pack_aos4(torch.from_numpy(rng.normal(0, 1, (n, 3))).cuda())
            out = torch.zeros(1, dtype=torch.float64, device="cuda")
            lj.integrate_push(q, q, p, q.clone(), 0.01, 0, n, out, [(ptr, lo, hi)])
            torch.cuda.synchronize()
            np.save(os.path.join(outdir, "sent.npy"), q.cpu().numpy())
            dist.barrier()
            dist.barrier()                                     # process 0 has read: unmap
            lj.ipc_close(ptr)
    finally:
        dist.destroy_process_group()


def test_push_through_cuda_ipc(lj, tmp_path):
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    mp.start_processes(_ipc_worker, args=(port, str(tmp_path)), nprocs=2, start_method="spawn")
    got, sent = np.load(tmp_path / "got.npy"), np.load(tmp_path / "sent.npy")
    lo, hi = 3_000, 7_500
    assert np.array_equal(got[lo:hi], sent[lo:hi])
    assert (got[:lo] == -1.0).all() and (got[hi:] == -1.0).all()


def test_push_against_the_oracle(lj):
    """the fused drift + push compared with the ORACLE directly (reading
    O6 integrate, C-16 displacement): own rows, every pushed replica row and the
    maximum displacement bit-identical to oracle.integrate / oracle.max_displacement."""
    import oracle
    rng = np.random.default_rng(23)
    n, dt = 20_000, 0.005
    qn = rng.uniform(0, 30, (n, 3))
    pn = rng.normal(0, 1, (n, 3))
    qrefn = qn + rng.normal(0, 0.05, (n, 3))
    b, e = 4_000, 13_333
    q = lj.pack_aos4(torch.from_numpy(qn).cuda())
    p = lj.pack_aos4(torch.from_numpy(pn).cuda())
    q_ref = lj.pack_aos4(torch.from_numpy(qrefn).cuda())
    peers = [torch.zeros((n, 4), dtype=torch.float64, device="cuda") for _ in range(2)]
    ranges = [(b, b + 700), (e - 1500, e)]
    q_out = torch.zeros_like(q)
    out = torch.zeros(1, dtype=torch.float64, device="cuda")
    lj.integrate_push(q, q_out, p, q_ref, dt, b, e, out,
                      [(t.data_ptr(), lo, hi) for t, (lo, hi) in zip(peers, ranges)])
    torch.cuda.synchronize()
    ref = oracle.integrate(qn, pn, dt, b, e)
    got = q_out[:, :3].cpu().numpy()
    assert np.array_equal(got[b:e], ref[b:e])
    for t, (lo, hi) in zip(peers, ranges):
        assert np.array_equal(t[lo:hi, :3].cpu().numpy(), ref[lo:hi])
        assert not t[:lo].any() and not t[hi:].any()
    assert out.item() == oracle.max_displacement(ref, qrefn, b, e)


@pytest.mark.parametrize("P", [1, 3, 4])
def test_resort_with_peer_momenta_emulated_ranks(lj, P):
    """lj_permute_rows_peers (the multi-rank re-sort of graph_collective) with P emulated
    ranks on one GPU: rank k's share buffer holds only its own rows' momenta (the rest is
    junk); for every rank r, perm is the oracle's cell order, q_out = q[perm], and the own
    new rows of p_out are the global momenta of the permuted atoms, read from whichever
    rank owned each atom -- other rows untouched."""
    import lj_inputs
    import oracle
    w = lj_inputs.config(1)
    n = w.n - w.n % P
    qn = np.ascontiguousarray(w.q[:n])
    n_own = n // P
    g = lj.geom(w.L, w.rc, w.rs)
    rng = np.random.default_rng(P)
    pg = rng.normal(0, 1, (n, 3))
    p_glob = lj.pack_aos4(torch.from_numpy(pg).cuda())
    shares = []
    for k in range(P):
        s = torch.full((n, 4), -7.0, dtype=torch.float64, device="cuda")
        s[k * n_own:(k + 1) * n_own] = p_glob[k * n_own:(k + 1) * n_own]
        shares.append(s)
    table = torch.tensor([s.data_ptr() for s in shares], dtype=torch.int64, device="cuda")
    import ctypes
    b = ctypes.c_size_t()
    assert lj.load().lj_build_list_workspace(n, g, ctypes.byref(b)) == 0
    ws = torch.empty(b.value, dtype=torch.uint8, device="cuda")
    ref_perm = oracle.cell_order(qn, w.L, w.rs)
    for r in range(P):
        q = lj.pack_aos4(torch.from_numpy(qn).cuda())
        q_out = torch.zeros_like(q)
        q_ref = torch.zeros_like(q)
        p_out = torch.full((n, 4), 5.0, dtype=torch.float64, device="cuda")
        perm = torch.empty(n, dtype=torch.int64, device="cuda")
        lj.permute_rows_peers(q, q_out, q_ref, p_out, table, n_own, r * n_own, (r + 1) * n_own, perm, g, ws)
        torch.cuda.synchronize()
        pm = perm.cpu().numpy()
        assert np.array_equal(pm, ref_perm)
        assert np.array_equal(q_out[:, :3].cpu().numpy(), oracle.wrap(qn, w.L)[pm])
        assert torch.equal(q_ref, q_out)
        own = slice(r * n_own, (r + 1) * n_own)
        assert np.array_equal(p_out[own, :3].cpu().numpy(), pg[pm[own]])
        rest = torch.ones(n, dtype=torch.bool, device="cuda")
        rest[own] = False
        assert bool((p_out[rest] == 5.0).all())
