"""Multi-rank plumbing of the row-split MD driver on CPU with
gloo, world size 2: the product driver paper_1806_05713_b200.md.LeapfrogMD
with an oracle-backed compute backend (test infrastructure) in place of liblj.

Full-list rows are independent, so P ranks must reproduce the 1-rank run
bit for bit (DESIGN.md Pin-12): momenta of every row, positions, the rebuild
schedule and the cell-order permutation."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import lj_inputs
import oracle
from paper_1806_05713_b200 import lj, md


class OracleBackend:
    """CPU backend over the oracle with the LibBackend interface (tests only)."""

    def __init__(self, n, g, row_begin, row_end, half=False, shm_dir=None):
        self.n, self.g, self.rb, self.re, self.half = n, g, row_begin, row_end, half
        self.shm_dir, self._paths = shm_dir, {}

    def records(self, xyz):
        out = torch.zeros((xyz.shape[0], 4), dtype=torch.float64)
        out[:, :3] = torch.as_tensor(np.ascontiguousarray(xyz))
        return out

    def empty_records(self, n):
        return torch.zeros((n, 4), dtype=torch.float64)

    @staticmethod
    def _xyz(t):
        return np.ascontiguousarray(t[:, :3].numpy())

    def build(self, q):
        return oracle.list_cells(self._xyz(q), self.g.L, self.g.rs, self.half, self.rb, self.re)

    def cell_order(self, q):
        return torch.as_tensor(oracle.cell_order(self._xyz(q), self.g.L, self.g.rs))

    def permute(self, src, perm, dst):
        dst.copy_(src[perm])

    def force(self, q, p, dt, lst, counter=None):
        out = oracle.force_step(self._xyz(q), self._xyz(p), self.g.L, self.g.rc, dt, lst)
        p[:, :3] = torch.as_tensor(out)

    def force_rows(self, q, p, dt, lst, a, b, counter=None):
        o = a - lst.row_begin
        sub = oracle.CSR(lst.number_of_partners[o:o + (b - a)], lst.pointer[o:o + (b - a) + 1], lst.sorted_list,
                         a, b, lst.half)
        self.force(q, p, dt, sub)

    def interior(self, lst):
        """Same definition as lj_list_interior, in numpy."""
        rb, re_ = lst.row_begin, lst.row_end
        mid = (rb + re_) // 2
        a, b = rb, re_
        for r in range(lst.rows):
            j = lst.row(r)
            if len(j) and (j.min() < rb or j.max() >= re_):
                i = rb + r
                if i < mid:
                    a = max(a, i + 1)
                else:
                    b = min(b, i)
        return a, b

    def partner_ranges(self, lst, bounds):
        """Same definition as lj_list_partner_ranges, in numpy."""
        j = lst.sorted_list[:lst.n_entries].astype(np.int64)
        out = []
        for s in range(len(bounds) - 1):
            m = j[(j >= bounds[s]) & (j < bounds[s + 1])]
            out.append((int(m.min()), int(m.max())) if len(m) else None)
        return out

    def integrate(self, q, p, dt, b, e):
        q[:, :3] = torch.as_tensor(oracle.integrate(self._xyz(q), self._xyz(p), dt, b, e))

    def max_disp(self, q, q_ref, b, e, out):
        out[0] = oracle.max_displacement(self._xyz(q), self._xyz(q_ref), b, e)

    def wrap(self, q, q_ref):
        q[:, :3] = torch.as_tensor(oracle.wrap(self._xyz(q), self.g.L))
        if q_ref is not None:
            q_ref.copy_(q)

    # exchange="push": the peers' q replicas are file-backed shared tensors (the CPU
    # stand-in for CUDA IPC mappings); integrate_push stores into them directly
    def shared_records(self, n):
        path = os.path.join(self.shm_dir, f"q_{os.getpid()}_{len(self._paths)}.bin")
        t = torch.from_file(path, shared=True, size=n * 4, dtype=torch.float64).view(n, 4)
        t.zero_()
        self._paths[t.data_ptr()] = path
        return t

    def share(self, t):
        return self._paths[t.data_ptr()], t.shape[0]

    def open_shared(self, handle):
        path, n = handle
        return torch.from_file(path, shared=True, size=n * 4, dtype=torch.float64).view(n, 4)

    def integrate_push(self, q_in, q_out, p, q_ref, dt, b, e, out, targets):
        new = oracle.integrate(self._xyz(q_in), self._xyz(p), dt, b, e)
        q_out[b:e, :3] = torch.as_tensor(new[b:e])
        q_out[b:e, 3] = q_in[b:e, 3]
        out[0] = oracle.max_displacement(self._xyz(q_out), self._xyz(q_ref), b, e)
        for peer, lo, hi in targets:
            peer[lo:hi] = q_out[lo:hi]

    def energy(self, q, p, lst, out):
        ke, pe = oracle.energy(self._xyz(q), self._xyz(p), self.g.L, self.g.rc, lst)
        out[0], out[1] = ke, pe


def make_system(n_drop, cells=8):
    w = lj_inputs.make_system(cells, jitter_seed=1, T=1.0, mom_seed=5, dt=0.01)
    q, p = w.q, w.p
    if n_drop:
        q, p = q[:-n_drop].copy(), p[:-n_drop].copy()
    return w, q, p


def run(rank, world, n_drop, reorder, steps, comm=None, overlap=None, exchange="allgather", shm_dir=None):
    # overlap needs slabs wider than 2 r_s to have interior rows: 12^3 FCC cells (L = 19)
    w, q, p = make_system(n_drop, 12 if (overlap or exchange != "allgather") else 8)
    g = lj.geom(w.L, w.rc, w.rs)
    rb, re_ = md.row_range(q.shape[0], rank, world)
    sim = md.LeapfrogMD(OracleBackend(q.shape[0], g, rb, re_, shm_dir=shm_dir), q, p, g, w.dt, rank, world, comm,
                        count_interactions=False, reorder=reorder, overlap=overlap, exchange=exchange)
    if world > 1 and exchange != "allgather":   # P = 2: two short ranges, not the whole slab
        assert sim.halo and 0 < sim.halo_bytes() < (q.shape[0] - (re_ - rb)) * 32, "a halo, not everything"
    if world > 1 and exchange == "push":
        assert sim.push and not sim.overlap
    if world > 1 and overlap:
        assert sim.overlap
        a, b = sim.interior_rows
        assert rb <= a <= b <= re_
        if world == 2:
            assert rb < a < b < re_, "the slabs must have interior and boundary rows"
    sim.half_kick()
    for _ in range(steps):
        sim.step()
    sim.kdk_step()
    e = sim.energy()
    # gather every rank's own rows of p to rank 0 (q is replicated)
    p_full = sim.p.clone()
    sim._allgather(p_full)
    return sim.q.numpy().copy(), p_full.numpy().copy(), sim.stats.rebuilds, e


def _worker(rank, world, port, n_drop, reorder, steps, outdir, overlap=None, exchange="allgather"):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        q, p, rb, e = run(rank, world, n_drop, reorder, steps, dist.group.WORLD, overlap, exchange, outdir)
        np.savez(os.path.join(outdir, f"r{rank}.npz"), q=q, p=p, rb=rb, e=np.array(e))
    finally:
        dist.destroy_process_group()


def free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


@pytest.mark.parametrize("world,n_drop,reorder,overlap,exchange", [
    (2, 0, True, False, "allgather"), (2, 0, False, False, "allgather"), (2, 3, True, None, "allgather"),
    (2, 0, True, True, "allgather"), (2, 0, False, True, "allgather"),
    (2, 0, True, False, "halo"), (3, 0, True, True, "halo"), (3, 0, False, False, "halo"),
    (2, 0, True, None, "push"), (3, 0, True, None, "push"), (3, 0, False, None, "push"),
    (2, 3, True, None, "push")])
def test_ranks_equal_one_rank(tmp_path, world, n_drop, reorder, overlap, exchange):
    """overlap=True: the position exchange runs asynchronously while the interior
    rows' forces are computed; exchange="halo": only the rows
    each rank's list reads are sent between rebuilds (NEXT-2); exchange="push": the
    drift stores those rows straight into the peers' double-buffered replicas
    (NEXT-2 fused variant, shared files standing in for CUDA IPC) -- all
    bit-identical to one rank."""
    steps = 12        # T = 1, dt = 0.01: the list is rebuilt every ~4-5 steps
    q1, p1, rb1, e1 = run(0, 1, n_drop, reorder, steps, overlap=overlap, exchange=exchange)
    assert rb1 >= 2, "the test must exercise rebuilds"
    mp.start_processes(_worker, args=(world, free_port(), n_drop, reorder, steps, str(tmp_path), overlap, exchange),
                       nprocs=world, start_method="spawn")
    for r in range(world):
        d = np.load(tmp_path / f"r{r}.npz")
        assert np.array_equal(d["q"], q1)
        assert np.array_equal(d["p"], p1)
        assert int(d["rb"]) == rb1
        # energies: per-rank partial sums reduced -> equal up to summation order
        assert np.allclose(d["e"], np.array(e1), rtol=1e-12, atol=0)


def test_reorder_keeps_the_physics():
    """Cell-order re-sorting at rebuilds permutes storage, not the trajectory."""
    qa, pa, rba, _ = run(0, 1, 0, True, 12)
    qb, pb, rbb, _ = run(0, 1, 0, False, 12)
    assert rba == rbb
    ida = pa[:, 3].astype(np.int64)
    idb = pb[:, 3].astype(np.int64)
    assert np.array_equal(np.sort(ida), np.arange(len(ida)))
    A = np.empty_like(qa)
    A[ida] = qa
    B = np.empty_like(qb)
    B[idb] = qb
    # same trajectory up to summation order within rows (list rows are sorted in each index space)
    d = A[:, :3] - B[:, :3]
    L = lj_inputs.box_length(8)
    d -= L * np.round(d / L)
    assert np.abs(d).max() < 1e-12


def test_row_range_partition():
    for n in (1, 7, 4000, 16_384_000):
        for world in (1, 2, 3, 8):
            rr = [md.row_range(n, r, world) for r in range(world)]
            assert rr[0][0] == 0 and rr[-1][1] == n
            assert all(rr[k][1] == rr[k + 1][0] for k in range(world - 1))
            sizes = [b - a for a, b in rr]
            assert max(sizes) - min(sizes) <= 1
