"""MD driver over the C ABI: leapfrog velocity Verlet with the bookkeeping
rebuild (readings O8, C-16), row-split across ranks
 with a per-step exchange of positions.

One rank per GPU.  Rank r owns atoms/rows [r N/P, (r+1) N/P): it keeps the
replicated positions q (N AoS4 records), its own momenta p (global-indexed,
only own rows meaningful), its own bookkeeping reference q_ref and the CSR list
of its own rows.  Per step (SURVEY §3 call stack 4):

    force(dt) on own rows          -- lj_force_step (kernel)
    q += p dt; disp = max|q-q_ref| -- lj_integrate_displacement (one kernel)
    all-reduce MAX disp            -- torch.distributed, P > 1 only
    if 2 disp >= rs - rc:          -- host decision (one 8-byte readback)
        all-gather q; rebuild      -- lj_rebuild (wrap + cell order + list)
    else: exchange q               -- P > 1 only: NCCL all-gather (asynchronous
                                      with overlap: the next force step computes
                                      the interior rows while it is in flight),
                                      halo send/recv, or the drift kernel's own
                                      NVLink push (exchange="push")

On one rank, LeapfrogMD.graph(K) runs K such steps as one CUDA graph with the
rebuild decision on the device (lj_md_graph: no host round trip).

The compute backend is injectable so the multi-rank plumbing can be tested on
CPU with gloo (tests/test_dist_gloo.py); the product backend is LibBackend,
which has no fallback: it raises if liblj.so or the GPU is missing.
"""
from __future__ import annotations

import dataclasses
import os

import torch
import torch.distributed as dist

from . import lj


def row_range(n: int, rank: int, world: int) -> tuple[int, int]:
    """Rows of `rank`: [rank*n//world, (rank+1)*n//world) (contiguous slabs in lattice order)."""
    return n * rank // world, n * (rank + 1) // world


class LibBackend:
    """liblj.so on the current CUDA device."""

    def __init__(self, n, g: lj.Geom, row_begin, row_end, device, half=False, deferred=True, interleaved=None):
        lj.load()
        self.device = torch.device(device)
        self.n, self.g = n, g
        # Deferred builds (no host round trip per rebuild) are switched on after the first,
        # synchronous build, and only if its longest row leaves ROW_MARGIN entries below the
        # padded stride.  A later row over the stride is still safe: the builder stores
        # min(count, stride) and raises the overflow flag, which resolve() / StepGraph.finish()
        # turn into LJ_ERR_UNSUPPORTED.
        self._want_deferred = bool(deferred)
        # The interleaved padded layout (LJ_LIST_INTERLEAVED: the force kernel's index loads are
        # one 128-B line per warp) unless LJ_LIST_INTERLEAVE=0 (A/B measurements).
        if interleaved is None:
            interleaved = os.environ.get("LJ_LIST_INTERLEAVE", "1") != "0"
        self.builder = lj.ListBuilder(n, g, half, row_begin, row_end, device=self.device, padded=True,
                                      deferred=False, interleaved=interleaved)
        self.perm = None   # scratch of the re-sorting rebuild (allocated on first use)

    ROW_MARGIN = 24

    def headroom_ok(self) -> bool:
        """The last build's longest row is at least ROW_MARGIN below the padded stride."""
        return self.builder.padded and \
            self.builder.max_row_length() + self.ROW_MARGIN <= lj.LJ_PADDED_ROW_STRIDE

    def _after_build(self, lst):
        if self._want_deferred and not self.builder.deferred:
            self._want_deferred = False   # decided once, on the first synchronous build
            if self.headroom_ok():
                self.builder.enable_deferred()
        return lst

    def resolve(self, lst):
        """Finish a deferred build (call after a synchronisation)."""
        self.builder.resolve(lst)

    def records(self, xyz):
        t = xyz if isinstance(xyz, torch.Tensor) else torch.from_numpy(xyz)
        return lj.pack_aos4(t.to(self.device, dtype=torch.float64))

    def empty_records(self, n):
        return torch.empty((n, 4), dtype=torch.float64, device=self.device)

    def build(self, q):
        return self._after_build(self.builder.build(q))

    def rebuild(self, q, p, q_out, p_out, q_ref):
        """Fused wrap + cell-order permutation + list build (lj_rebuild, one cell pass)."""
        if self.perm is None:
            self.perm = torch.empty(self.n, dtype=torch.int64, device=self.device)
        return self._after_build(self.builder.rebuild(q, p, q_out, p_out, q_ref, self.perm))

    def cell_order(self, q):
        """perm[new] = old (stable sort by cell id), using the builder's workspace."""
        perm = torch.empty(self.n, dtype=torch.int64, device=self.device)
        ws = self.builder.workspace
        lj._check(lj.load().lj_cell_order(lj._ptr(q), self.n, self.g, lj._ptr(perm), lj._ptr(ws), ws.numel(),
                                          lj._stream()))
        return perm

    def permute(self, src, perm, dst):
        lj._check(lj.load().lj_permute_rows(lj._ptr(src), lj._ptr(dst), lj._ptr(perm), self.n, lj._stream()))

    def force(self, q, p, dt, lst, counter=None):
        lj.force_step(q, p, self.g, dt, lst, n_interactions=counter)

    def force_rows(self, q, p, dt, lst, a, b, counter=None):
        """Force on the rows [a, b) of lst only."""
        lj.force_step(q, p, self.g, dt, lst.rows_view(a, b), n_interactions=counter)

    def interior(self, lst):
        """Rows [A, B) whose partners are all own rows (lj_list_interior)."""
        return lj.list_interior(lst)

    def partner_ranges(self, lst, bounds):
        """Per owner slab, (min, max) partner index of lst's rows (lj_list_partner_ranges)."""
        return lj.list_partner_ranges(lst, bounds)

    def integrate(self, q, p, dt, b, e):
        lj.integrate(q, p, dt, b, e)

    def max_disp(self, q, q_ref, b, e, out):
        lj.max_displacement(q, q_ref, b, e, out)

    def integrate_disp(self, q, p, q_ref, dt, b, e, out):
        """integrate + max_disp in one pass (lj_integrate_displacement)."""
        lj.integrate_displacement(q, p, q_ref, dt, b, e, out)

    # ---- fused drift + NVLink push (exchange="push", one process per GPU) ----
    def shared_records(self, n):
        """A q replica other ranks push into (a plain device allocation, exported by CUDA IPC)."""
        return torch.empty((n, 4), dtype=torch.float64, device=self.device)

    def share(self, t):
        return lj.ipc_handle(t)

    def open_shared(self, handle):
        return lj.ipc_open(*handle)

    def integrate_push(self, q_in, q_out, p, q_ref, dt, b, e, out, targets):
        lj.integrate_push(q_in, q_out, p, q_ref, dt, b, e, out, targets)

    def close_shared(self, ptr):
        lj.ipc_close(ptr)

    def wrap(self, q, q_ref):
        lj.wrap(q, self.g.L, q_ref)

    def energy(self, q, p, lst, out):
        lj.energy(q, p, self.g, lst, out)


class _TorchGraph:
    """A torch.cuda.CUDAGraph with the interface StepGraph expects of lj.MDGraph."""

    def __init__(self, graph, steps, kernels_steps, kernels_rebuild, keep=()):
        self.graph, self.steps = graph, steps
        self._k = (kernels_steps, kernels_rebuild)
        self._keep = keep   # the buffers whose device pointers the graph holds (alive as long as it)

    def launch(self):
        self.graph.replay()

    def kernels(self):
        return self._k

    def force_ms(self):
        return []   # no per-step event nodes in this graph: the bench times the force kernel separately

    def close(self):
        self.graph = None
        self._keep = ()


@dataclasses.dataclass
class StepStats:
    rebuilds: int = 0
    steps: int = 0


class StepGraph:
    """A LeapfrogMD.graph(): the steps run on the device without host round trips."""

    def __init__(self, sim, g, status, energy_every=0, energies=None):
        self.sim, self.g, self.status = sim, g, status
        self.energy_every, self._energies = energy_every, energies
        self._seen = 0
        # the graph holds the device pointers of these buffers: an eager step
        # that swaps sim.q / sim.p (a re-sorting rebuild) invalidates it
        self._q, self._p = sim.q, sim.p

    def energies(self):
        """[(step, KE, PE)] of the last completed launch (energy_every > 0; one rank: no reduction)."""
        if self._energies is None:
            return []
        e = self._energies.view(-1, 2).tolist()
        return [(k * self.energy_every, ke, pe) for k, (ke, pe) in enumerate(e)]

    def launch(self):
        if self.sim.q is not self._q or self.sim.p is not self._p:
            raise RuntimeError("StepGraph: the driver's q/p buffers changed since the graph was captured "
                               "(an eager step re-sorted the atoms); create a new graph with sim.graph()")
        self.g.launch()

    def finish(self):
        """After the launch has completed: rebuild count, list size, overflow check."""
        st = self.status.tolist()
        if st[1]:
            raise lj.LJError(lj.LJ_ERR_UNSUPPORTED, "graph rebuild: a row exceeded the padded stride")
        new = st[0] - self._seen
        self._seen = st[0]
        self.sim.stats.rebuilds += new
        self.sim.stats.steps += self.g.steps
        if new:
            self.sim.lst.n_entries = int(st[2])
        return new

    def close(self):
        self.g.close()


class LeapfrogMD:
    """Row-split leapfrog MD.  `comm` is None for a single rank, else a
    torch.distributed process group (NCCL on GPUs, gloo in CPU tests)."""

    def __init__(self, backend, q_xyz, p_xyz, g: lj.Geom, dt: float, rank: int = 0, world: int = 1, comm=None,
                 count_interactions: bool = True, reorder: bool = True, overlap: bool | None = None,
                 exchange: str = "allgather"):
        self.be, self.g, self.dt = backend, g, float(dt)
        self.n = q_xyz.shape[0]
        self.rank, self.world, self.comm = rank, world, comm
        # collectives run for P > 1; LJ_FORCE_COLLECTIVES=1 also issues them at P = 1 (exercises the
        # NCCL code path on a single GPU under torchrun)
        self.collective = comm is not None and (world > 1 or os.environ.get("LJ_FORCE_COLLECTIVES") == "1")
        self.rb, self.re = row_range(self.n, rank, world)
        self.q = backend.records(q_xyz)
        self.p = backend.records(p_xyz)
        self.q_ref = backend.empty_records(self.n)
        self.disp = torch.zeros(1, dtype=torch.float64, device=self.q.device)
        self.counter = torch.zeros(1, dtype=torch.int64, device=self.q.device) if count_interactions else None
        self.stats = StepStats()
        self.margin = g.rs - g.rc
        # storage slot -> original atom id, carried in the pad lane of p (the driver
        # owns p; every kernel ignores and preserves pads)
        self.reorder = reorder
        self.p[:, 3] = torch.arange(self.n, dtype=torch.float64, device=self.p.device)
        # fused drift + NVLink push (exchange="push"): every rank's
        # integrate kernel stores its updated boundary rows straight into the other
        # ranks' q replicas (lj_integrate_push over CUDA IPC); the replicas are
        # double-buffered (q / q_alt) so that a push of step s never lands in the
        # buffer a slower rank's force of step s is still reading
        if exchange not in ("allgather", "halo", "push"):
            raise ValueError("exchange must be 'allgather', 'halo' or 'push'")
        self.push = (exchange == "push" and self.collective and world > 1
                     and all(hasattr(backend, f) for f in ("integrate_push", "share", "open_shared", "shared_records")))
        if self.push:
            q_sh = backend.shared_records(self.n)
            q_sh.copy_(self.q)
            self.q = q_sh
            self.q_alt = backend.shared_records(self.n)
            self._qbufs = [self.q, self.q_alt]
            self._cur = 0
            self._peers = self._open_peers()
        elif reorder:
            self.q_alt = backend.empty_records(self.n)
        if reorder:
            self.p_alt = backend.empty_records(self.n)
        # comm/compute overlap: the all-gather of the positions
        # runs asynchronously while the next force step computes the interior rows
        # (all partners own); boundary rows wait for it.  Needs equal slabs.
        can = self.collective and self.n % world == 0 and hasattr(backend, "force_rows") and not self.push
        self.overlap = can if overlap is None else (bool(overlap) and can)
        self._pending = None                  # async all-gather of q in flight
        self.interior_rows = (self.rb, self.re)
        # halo exchange: between rebuilds each rank receives only the
        # position rows its list reads from other ranks (lj_list_partner_ranges) instead of
        # all of them; rebuilds, kdk_step and gather_all_positions() use the full all-gather
        self.halo = (exchange in ("halo", "push") and self.collective and world > 1
                     and hasattr(backend, "partner_ranges"))
        self._halo_plan = None                # (sends [(rank, lo, hi)], recvs [(rank, lo, hi)])
        self._stale = False                   # other ranks' rows outside the halo are out of date
        self._rebuild()

    # ---- collectives (no-ops for one rank) ----
    def _allgather(self, x):
        """Replicate the own-row slab of x (n records) on every rank."""
        if self.collective:
            own = x[self.rb:self.re]
            if self.n % self.world == 0:
                # in-place all-gather: rank r's slab is already at its offset
                dist.all_gather_into_tensor(x, own.clone() if self._gloo() else own, group=self.comm)
            else:
                # uneven slabs: gather equal-size padded slabs, then scatter them back
                m = -(-self.n // self.world)
                send = torch.zeros((m, x.shape[1]), dtype=x.dtype, device=x.device)
                send[: self.re - self.rb] = own
                buf = torch.empty((self.world * m, x.shape[1]), dtype=x.dtype, device=x.device)
                dist.all_gather_into_tensor(buf, send, group=self.comm)
                for r in range(self.world):
                    b, e = row_range(self.n, r, self.world)
                    if r != self.rank:
                        x[b:e] = buf[r * m: r * m + (e - b)]

    def _allgather_q(self):
        self.sync_positions()
        self._allgather(self.q)
        self._stale = False

    def _allgather_q_async(self):
        """Start the in-place all-gather of the own position rows (completed by sync_positions)."""
        if self.collective:
            own = self.q[self.rb:self.re]
            self._pending = [dist.all_gather_into_tensor(self.q, own.clone() if self._gloo() else own,
                                                         group=self.comm, async_op=True)]

    def sync_positions(self):
        """Complete a pending exchange: afterwards q holds every position the own rows' forces read
        (all positions after an all-gather; see gather_all_positions for the halo mode)."""
        if self._pending is not None:
            for w in self._pending:
                w.wait()
            self._pending = None

    def gather_all_positions(self):
        """Make every rank's q hold all current positions (a full all-gather in the halo mode)."""
        self.sync_positions()
        if self._stale:
            self._allgather_q()

    # ---- halo exchange (NEXT-2) ----
    def _plan_halo(self):
        """After a build: which own rows every other rank reads, and which rows of theirs we read.
        Each owner slab is queried as two halves, so that a slab read from both of its sides
        (P = 2: the periodic neighbour on the left and on the right is the same rank) gives
        two short ranges instead of one that spans the slab."""
        W = self.world
        bounds = []
        for s in range(W):
            b, e = row_range(self.n, s, W)
            bounds += [b, (b + e) // 2]
        bounds.append(self.n)
        need = self.be.partner_ranges(self.lst, bounds)
        mine = torch.zeros((W, 2, 2), dtype=torch.int64, device=self.q.device)
        for k, r in enumerate(need):
            if k // 2 != self.rank and r is not None:
                mine[k // 2, k % 2, 0], mine[k // 2, k % 2, 1] = r[0], r[1] + 1
        table = torch.empty((W * W, 2, 2), dtype=torch.int64, device=self.q.device)
        dist.all_gather_into_tensor(table.view(W * W * 2, 2), mine.view(W * 2, 2), group=self.comm)
        table = table.view(W, W, 2, 2).tolist()   # table[a][s][h] = rows of half h of slab s that a reads

        def ranges(a, s):
            out = [(lo, hi) for lo, hi in table[a][s] if hi > lo]
            if len(out) == 2 and out[0][1] >= out[1][0]:   # touching halves: one range
                out = [(out[0][0], out[1][1])]
            return out

        sends = [(a, lo, hi) for a in range(W) if a != self.rank for lo, hi in ranges(a, self.rank)]
        recvs = [(s, lo, hi) for s in range(W) if s != self.rank for lo, hi in ranges(self.rank, s)]
        self._halo_plan = (sends, recvs)

    def _halo_exchange(self, async_op: bool):
        sends, recvs = self._halo_plan
        ops = [dist.P2POp(dist.isend, self.q[lo:hi], a, group=self.comm) for a, lo, hi in sends]
        ops += [dist.P2POp(dist.irecv, self.q[lo:hi], s, group=self.comm) for s, lo, hi in recvs]
        reqs = dist.batch_isend_irecv(ops) if ops else []
        self._stale = True
        if async_op:
            self._pending = list(reqs)
        else:
            for r in reqs:
                r.wait()

    def halo_bytes(self) -> int:
        """Position bytes this rank receives per step in the halo mode."""
        if self._halo_plan is None:
            return 0
        return sum(hi - lo for _, lo, hi in self._halo_plan[1]) * 32

    def _gloo(self):
        return dist.get_backend(self.comm) == "gloo"

    def _allreduce_max(self, t):
        if self.collective:
            dist.all_reduce(t, op=dist.ReduceOp.MAX, group=self.comm)

    def _allreduce_sum(self, t):
        if self.collective:
            dist.all_reduce(t, op=dist.ReduceOp.SUM, group=self.comm)

    # ---- MD ----
    def half_kick(self, sign: float = 1.0):
        """p += sign F(q) dt/2."""
        self.sync_positions()
        self.be.force(self.q, self.p, sign * 0.5 * self.dt, self.lst)

    def start_leapfrog(self):
        """Synchronised p_0 -> p_{-1/2} = p_0 - F(q_0) dt/2, the state step() expects."""
        self.half_kick(-1.0)

    def _rebuild(self):
        """Wrap, (optionally) re-sort the atoms into cell order (§8(a) a3), snapshot
        q_ref and rebuild the own-row list (§8(a) a2-a4)."""
        self.gather_all_positions()
        self._rebuild_lists()
        if self.overlap:
            self.interior_rows = self.be.interior(self.lst)
        if self.halo:
            self._plan_halo()

    def _rebuild_lists(self):
        if self.reorder:
            if self.collective:
                self._allgather(self.p)          # momenta of all rows, to follow the permutation
            if hasattr(self.be, "rebuild"):      # one fused library call (lj_rebuild)
                self.lst = self.be.rebuild(self.q, self.p, self.q_alt, self.p_alt, self.q_ref)
                self._swap_q()
                self.p, self.p_alt = self.p_alt, self.p
                return
            self.be.wrap(self.q, None)
            perm = self.be.cell_order(self.q)
            self.be.permute(self.q, perm, self.q_alt)
            self.be.permute(self.p, perm, self.p_alt)
            self._swap_q()
            self.p, self.p_alt = self.p_alt, self.p
        self.be.wrap(self.q, self.q_ref)
        self.lst = self.be.build(self.q)

    def _swap_q(self):
        """q <-> q_alt (the push mode tracks which of the two shared buffers is current:
        every rank swaps at the same steps, so the index is the same on all ranks)."""
        self.q, self.q_alt = self.q_alt, self.q
        if self.push:
            self._cur ^= 1

    def _open_peers(self):
        """Map every other rank's two q buffers: peers[b][a] = rank a's buffer b (None for self)."""
        mine = [self.be.share(t) for t in self._qbufs]
        table = [None] * self.world
        dist.all_gather_object(table, mine, group=self.comm)
        return [[None if a == self.rank else self.be.open_shared(table[a][b]) for a in range(self.world)]
                for b in range(2)]

    def atom_ids(self):
        """Original atom id of every storage slot (int64, device)."""
        return self.p[:, 3].to(torch.int64)

    def _resolve(self):
        if hasattr(self.be, "resolve"):
            self.be.resolve(self.lst)

    def check_rebuild(self) -> bool:
        self.be.max_disp(self.q, self.q_ref, self.rb, self.re, self.disp)
        self._allreduce_max(self.disp)
        rebuild = 2.0 * float(self.disp.item()) >= self.margin
        self._resolve()
        if rebuild:
            self._rebuild()
            self.stats.rebuilds += 1
            return True
        return False

    def kick(self, dt: float, counter=None):
        """p += F(q) dt on own rows.  With an all-gather in flight, the interior
        rows go first (they read own positions only), then the boundary rows
        once the other ranks' positions have arrived."""
        if self._pending is None:
            self.be.force(self.q, self.p, dt, self.lst, counter)
            return
        a, b = self.interior_rows
        if b > a:
            self.be.force_rows(self.q, self.p, dt, self.lst, a, b, counter)
        self.sync_positions()
        if a > self.rb:
            self.be.force_rows(self.q, self.p, dt, self.lst, self.rb, a, counter)
        if self.re > b:
            self.be.force_rows(self.q, self.p, dt, self.lst, b, self.re, counter)

    def drift_and_exchange(self):
        """q += p dt on own rows, the bookkeeping check (displacement all-reduce
        MAX first), then the position exchange: a blocking all-gather + rebuild
        when the list expires, else the all-gather (asynchronous with overlap)."""
        if self.push:
            # the drift writes the other buffer and pushes the rows each peer's list
            # reads into that peer's other buffer; the displacement all-reduce below
            # orders every rank's pushes before any rank's next force step
            nxt = self._cur ^ 1
            targets = [(self._peers[nxt][a], lo, hi) for a, lo, hi in self._halo_plan[0]]
            self.be.integrate_push(self.q, self._qbufs[nxt], self.p, self.q_ref, self.dt, self.rb, self.re,
                                   self.disp, targets)
            self._swap_q()
            self._stale = True
        elif hasattr(self.be, "integrate_disp"):
            self.be.integrate_disp(self.q, self.p, self.q_ref, self.dt, self.rb, self.re, self.disp)
        else:
            self.be.integrate(self.q, self.p, self.dt, self.rb, self.re)
            self.be.max_disp(self.q, self.q_ref, self.rb, self.re, self.disp)
        self._allreduce_max(self.disp)
        rebuild = 2.0 * float(self.disp.item()) >= self.margin
        self._resolve()                            # the stream has passed the last (deferred) build
        if rebuild:
            self._allgather_q()
            self._rebuild()
            self.stats.rebuilds += 1
        elif self.push:
            pass                                   # the positions have already been pushed
        elif self.halo:
            self._halo_exchange(async_op=self.overlap)
        elif self.overlap:
            self._allgather_q_async()
        else:
            self._allgather_q()

    def step(self, sample: bool = False):
        """One leapfrog step: p += F(q) dt; q += p dt; all-gather; bookkeeping.
        With sample=True the kick is split in two halves around an energy
        evaluation at the synchronised momenta p_n = p_{n-1/2} + F(q_n) dt/2
        (reading O8/C-17); returns (KE, PE) then, else None."""
        e = None
        if sample:
            self.sync_positions()
            self.be.force(self.q, self.p, 0.5 * self.dt, self.lst, self.counter)
            e = self.energy()
            self.be.force(self.q, self.p, 0.5 * self.dt, self.lst)
        else:
            self.kick(self.dt, self.counter)
        self.drift_and_exchange()
        self.stats.steps += 1
        return e

    def kdk_step(self):
        """One synchronised velocity-Verlet step (O8): kick dt/2, drift, rebuild check, kick dt/2."""
        self.sync_positions()
        self.be.force(self.q, self.p, 0.5 * self.dt, self.lst)
        self.be.integrate(self.q, self.p, self.dt, self.rb, self.re)
        self._allgather_q()
        self.check_rebuild()
        self.be.force(self.q, self.p, 0.5 * self.dt, self.lst)
        self.stats.steps += 1

    def energy(self):
        """(KE, PE) summed over ranks (p must be synchronised, e.g. after kdk_step)."""
        self.sync_positions()
        out = torch.zeros(2, dtype=torch.float64, device=self.q.device)
        self.be.energy(self.q, self.p, self.lst, out)
        self._allreduce_sum(out)
        return float(out[0]), float(out[1])

    # ---- the step as a CUDA graph (NEXT-1: "capture the whole step"; one rank) ----
    def graph(self, steps: int, energy_every: int = 0) -> "StepGraph":
        """The next `steps` leapfrog steps (as step()) as one CUDA graph with a device-side
        rebuild decision (lj_md_graph): launch with .launch(), then .finish() after a
        synchronisation to fold the rebuilds into the driver's state."""
        if self.collective or not hasattr(self.be, "builder"):
            raise ValueError("graph: one rank with the liblj backend only")
        torch.cuda.current_stream().synchronize()
        self.sync_positions()
        self._resolve()
        if hasattr(self.be, "headroom_ok") and not self.be.headroom_ok():
            # rebuilds inside the graph write the padded layout; rows this close to the stride
            # could overflow it (the graph would then stop with LJ_ERR_UNSUPPORTED at finish())
            raise lj.LJError(lj.LJ_ERR_UNSUPPORTED, "graph: list rows within %d entries of the padded stride; "
                             "use eager steps" % self.be.ROW_MARGIN)
        if getattr(self.be, "perm", None) is None:
            self.be.perm = torch.empty(self.n, dtype=torch.int64, device=self.q.device)
        status = torch.zeros(4, dtype=torch.int64, device=self.q.device)
        ns = -(-steps // energy_every) if energy_every > 0 else 0
        energies = torch.zeros(max(2 * ns, 1), dtype=torch.float64, device=self.q.device)
        g = lj.MDGraph(self.q, self.p, self.q_alt if self.reorder else None, self.p_alt if self.reorder else None,
                       self.q_ref, self.be.perm, self.g, self.dt, self.be.builder, self.disp, self.counter, status,
                       self.reorder, steps, energy_every, energies if ns else None)
        return StepGraph(self, g, status, energy_every, energies if ns else None)

    # ---- the multi-rank step as a CUDA graph (NEXT-1 at P > 1) ----
    def graph_collective(self, steps: int, resort: bool | None = None) -> "StepGraph":
        """The next `steps` leapfrog steps at P > 1 (or P = 1 with LJ_FORCE_COLLECTIVES=1) as ONE
        CUDA graph, NCCL included (torch.cuda.graph capture).  Per step: the kick over the own rows;
        the drift + displacement; the own momenta copied into this step's share buffer (two,
        alternating by step parity); the rank's displacement published into the pad lane of its
        first own q record (lj_publish_scalar); the in-place NCCL all-gather of the positions -- which
        thereby also carries every rank's displacement -- and the device-side bookkeeping decision
        over the P pads with the conditional rebuild (lj_md_capture_rebuild).  With resort (default:
        the driver's reorder), the rebuild re-sorts every atom into cell order as lj_rebuild does and
        reads the own new rows' momenta straight from the owner ranks' share buffers over NVLink
        (CUDA IPC mappings) -- no host round trip per step or per rebuild, no momentum
        collective.  Without resort, atoms keep their storage slots (fixed ownership).  Either way
        the eager steps of this driver follow the same trajectory bit for bit.

        Ordering of the share buffers: rank r writes share[k % 2] in step k before its all-gather k;
        a peer reads it only in the rebuild of step k, after all-gather k has completed there; r next
        writes share[k % 2] in step k + 2, after all-gather k + 1 -- which the peer joins only once
        its rebuild of step k is done (stream order)."""
        if not self.collective or self.push or self.halo or self.n % self.world != 0:
            raise ValueError("graph_collective: NCCL driver with equal slabs and the all-gather exchange only")
        if not hasattr(self.be, "builder"):
            raise ValueError("graph_collective: the liblj backend only")
        resort = self.reorder if resort is None else bool(resort)
        torch.cuda.current_stream().synchronize()
        self.gather_all_positions()
        self._resolve()
        if hasattr(self.be, "headroom_ok") and not self.be.headroom_ok():
            raise lj.LJError(lj.LJ_ERR_UNSUPPORTED, "graph: list rows within %d entries of the padded stride; "
                             "use eager steps" % self.be.ROW_MARGIN)
        self.reorder = resort
        self.overlap = False
        status = torch.zeros(4, dtype=torch.int64, device=self.q.device)
        n_own = self.n // self.world
        pads = self.q.view(-1)[3:]                      # pad lane of record 0; rank r's first record at 4 r n_own
        own_pad = self.q[self.rb, 3:4]
        rs = None
        if resort:
            if getattr(self, "q_alt", None) is None:
                self.q_alt = self.be.empty_records(self.n)
            if getattr(self, "p_alt", None) is None:
                self.p_alt = self.be.empty_records(self.n)
            if getattr(self.be, "perm", None) is None:
                self.be.perm = torch.empty(self.n, dtype=torch.int64, device=self.q.device)
            if self.world > 1:
                self._p_share, self._p_tables = self._open_momentum_shares()
            else:   # one rank: the momenta are read from p itself (no copy, no peers)
                self._p_share = None
                t = torch.tensor([self.p.data_ptr()], dtype=torch.int64, device=self.q.device)
                self._p_tables = [t, t]
            rs = [dict(q_alt=self.q_alt, p=self.p, p_alt=self.p_alt, perm=self.be.perm, p_peers=self._p_tables[b],
                       n_own=n_own) for b in range(2)]
        g = torch.cuda.CUDAGraph()
        cs = torch.cuda.Stream(device=self.q.device)
        cs.wait_stream(torch.cuda.current_stream())
        l0 = lj.launch_count()
        kpr = 0
        with torch.cuda.graph(g, stream=cs, capture_error_mode="relaxed"):
            for k in range(steps):
                self.be.force(self.q, self.p, self.dt, self.lst, self.counter)
                self.be.integrate_disp(self.q, self.p, self.q_ref, self.dt, self.rb, self.re, self.disp)
                if resort and self._p_share is not None:
                    lj.copy_records(self.p[self.rb:self.re], self._p_share[k % 2][self.rb:self.re])
                lj.publish_scalar(self.disp, own_pad)
                dist.all_gather_into_tensor(self.q, self.q[self.rb:self.re], group=self.comm)
                kpr = lj.md_capture_rebuild(self.q, self.q_ref, self.g, self.be.builder, pads, self.world,
                                            4 * n_own, status, rs[k % 2] if resort else None)
        torch.cuda.current_stream().wait_stream(cs)
        per_step_total = lj.launch_count() - l0 - kpr * steps
        keep = (self._p_share, self._p_tables) if resort else ()
        return StepGraph(self, _TorchGraph(g, steps, per_step_total, kpr, keep), status)

    def graph_host_io(self, steps: int, q_host: torch.Tensor, p_host: torch.Tensor, chunks: int = 8,
                      chunk_min_rows: int = 1 << 20, timeline: list | None = None) -> "StepGraph":
        """The next `steps` leapfrog steps as ONE CUDA graph in which the state round-trips
        through the caller's page-locked host arrays q_host / p_host ((n, 3) float64, storage
        order) every step -- the end-to-end measurement of bench.py, one rank.  Per step: the
        H2D copies of p and q in `chunks` row chunks on a copy stream (lj_copy_bytes), packed
        into the records (lj_pack_aos4); the device-side bookkeeping decision on the previous
        drift's displacement with the conditional re-sorting rebuild (lj_md_capture_rebuild);
        the kick per row chunk, each chunk's momenta unpacked and sent back (D2H) at once on a
        second copy stream; the drift + displacement; q unpacked and sent back after them.  The
        rebuild thus runs at the START of the step that needs it (the same decision, on the
        same positions, as the eager driver's end-of-step rebuild), so the momenta are final
        after the kick and leave while the drift runs: a chunk's H2D in step k + 1 waits only
        for the same chunk's D2H in step k, and only q's round trip is on the critical path.
        No host round trip per step or per rebuild; the eager driver's trajectory bit for bit,
        except that a rebuild due after the last step is left to the next launch (the host
        arrays then hold the state as of before it).  The momenta's pad lane (atom ids) is not
        carried through the host arrays.  timeline (instrumentation): a list that receives, per step, a
        dict of CUDA events recorded inside the graph at the phase boundaries (elapsed times
        readable after a launch)."""
        if self.world != 1 or self.push or self.halo or not hasattr(self.be, "builder"):
            raise ValueError("graph_host_io: one rank, liblj backend, all-gather exchange")
        n = self.n
        for t, name in ((q_host, "q_host"), (p_host, "p_host")):
            if t.shape != (n, 3) or t.dtype != torch.float64 or not t.is_contiguous() or not t.is_pinned():
                raise ValueError(f"graph_host_io: {name} must be a pinned contiguous (n, 3) float64 tensor")
        torch.cuda.current_stream().synchronize()
        self._resolve()
        if hasattr(self.be, "headroom_ok") and not self.be.headroom_ok():
            raise lj.LJError(lj.LJ_ERR_UNSUPPORTED, "graph: list rows within %d entries of the padded stride; "
                             "use eager steps" % self.be.ROW_MARGIN)
        dev = self.q.device
        status = torch.zeros(4, dtype=torch.int64, device=dev)
        rs = None
        if self.reorder:
            if getattr(self, "q_alt", None) is None:
                self.q_alt = self.be.empty_records(n)
            if getattr(self, "p_alt", None) is None:
                self.p_alt = self.be.empty_records(n)
            if getattr(self.be, "perm", None) is None:
                self.be.perm = torch.empty(n, dtype=torch.int64, device=dev)
            self._p_table = torch.tensor([self.p.data_ptr()], dtype=torch.int64, device=dev)
            rs = dict(q_alt=self.q_alt, p=self.p, p_alt=self.p_alt, perm=self.be.perm, p_peers=self._p_table,
                      n_own=n)
        K = max(1, min(int(chunks), n)) if n >= chunk_min_rows else 1   # (small systems: one chunk)
        cb = [n * c // K for c in range(K + 1)]
        sl = [slice(cb[c], cb[c + 1]) for c in range(K)]
        q_in, p_in, q_out, p_out = (torch.empty((n, 3), dtype=torch.float64, device=dev) for _ in range(4))
        self._host_io = (q_host, p_host, q_in, p_in, q_out, p_out, status)   # the graph holds their pointers
        g = torch.cuda.CUDAGraph()
        # one H2D and one D2H copy stream: on each, a step's momenta chunks precede its positions
        # (they are final first); q's round trip is the critical path
        cs, ci, co = (torch.cuda.Stream(device=dev) for _ in range(3))
        cs.wait_stream(torch.cuda.current_stream())
        l0 = lj.launch_count()
        kpr = 0
        with torch.cuda.graph(g, stream=cs, capture_error_mode="relaxed"):
            # the first decision reads the current displacement (0 right after a rebuild)
            self.be.max_disp(self.q, self.q_ref, 0, n, self.disp)
            start = cs.record_event()
            for st in (ci, co):
                st.wait_event(start)
            ev_qo, ev_po = [None] * K, [None] * K

            def mark(tl, name, st):
                if tl is not None:
                    e = torch.cuda.Event(enable_timing=True, external=True)
                    e.record(st)
                    tl[name] = e

            for _ in range(steps):
                tl = {} if timeline is not None else None
                if tl is not None:
                    timeline.append(tl)
                mark(tl, "start", cs)
                ev_qi, ev_pi = [], []
                with torch.cuda.stream(ci):   # p first: it left first in the previous step
                    for c in range(K):
                        if ev_po[c] is not None:
                            ci.wait_event(ev_po[c])
                        lj.copy_bytes(p_in[sl[c]], p_host[sl[c]])
                        ev_pi.append(ci.record_event())
                    mark(tl, "p_h2d", ci)
                    for c in range(K):
                        if ev_qo[c] is not None:
                            ci.wait_event(ev_qo[c])
                        lj.copy_bytes(q_in[sl[c]], q_host[sl[c]])
                        ev_qi.append(ci.record_event())
                    mark(tl, "q_h2d", ci)
                for c in range(K):
                    cs.wait_event(ev_pi[c])
                    lj.pack_aos4(p_in[sl[c]], out=self.p[sl[c]])
                for c in range(K):
                    cs.wait_event(ev_qi[c])
                    lj.pack_aos4(q_in[sl[c]], out=self.q[sl[c]])
                mark(tl, "q_in", cs)
                kpr = lj.md_capture_rebuild(self.q, self.q_ref, self.g, self.be.builder, self.disp, 1, 0, status, rs)
                mark(tl, "rebuild", cs)
                for c in range(K):   # the kick per chunk; its momenta leave at once
                    if K == 1:
                        self.be.force(self.q, self.p, self.dt, self.lst, self.counter)
                    else:
                        self.be.force_rows(self.q, self.p, self.dt, self.lst, cb[c], cb[c + 1], self.counter)
                    lj.unpack_aos4(self.p[sl[c]], out=p_out[sl[c]])
                    e_p = cs.record_event()
                    with torch.cuda.stream(co):
                        co.wait_event(e_p)
                        lj.copy_bytes(p_host[sl[c]], p_out[sl[c]])
                        ev_po[c] = co.record_event()
                mark(tl, "kick", cs)
                mark(tl, "p_out", co)
                self.be.integrate_disp(self.q, self.p, self.q_ref, self.dt, 0, n, self.disp)
                lj.unpack_aos4(self.q, out=q_out)
                e_q = cs.record_event()
                mark(tl, "drift", cs)
                with torch.cuda.stream(co):
                    co.wait_event(e_q)
                    for c in range(K):
                        lj.copy_bytes(q_host[sl[c]], q_out[sl[c]])
                        ev_qo[c] = co.record_event()
                    mark(tl, "q_out", co)
            for st in (ci, co):
                cs.wait_event(st.record_event())
        torch.cuda.current_stream().wait_stream(cs)
        per_step_total = lj.launch_count() - l0 - kpr * steps
        return StepGraph(self, _TorchGraph(g, steps, per_step_total, kpr, self._host_io + (rs,)), status)

    def _open_momentum_shares(self):
        """Two share buffers for the own momenta and, per buffer, a device table of every rank's
        buffer pointer (CUDA IPC mappings of the peers' buffers; this rank's own pointer locally)."""
        shares = [self.be.shared_records(self.n) for _ in range(2)] if hasattr(self.be, "shared_records") \
            else [self.be.empty_records(self.n) for _ in range(2)]
        if self.world > 1:
            mine = [self.be.share(t) for t in shares]
            table = [None] * self.world
            dist.all_gather_object(table, mine, group=self.comm)
            self._share_peers = [[None if a == self.rank else self.be.open_shared(table[a][b])
                                  for a in range(self.world)] for b in range(2)]
            ptrs = [[shares[b].data_ptr() if a == self.rank else self._share_peers[b][a] for a in range(self.world)]
                    for b in range(2)]
        else:
            self._share_peers = None
            ptrs = [[shares[b].data_ptr()] for b in range(2)]
        tables = [torch.tensor(ptrs[b], dtype=torch.int64, device=self.q.device) for b in range(2)]
        return shares, tables

    def close(self):
        """Unmap the peers' replicas (exchange="push") and momentum shares (graph_collective);
        the driver is unusable afterwards."""
        shares = getattr(self, "_share_peers", None)
        closer = getattr(self.be, "close_shared", None)
        if shares is not None and closer is not None:
            for row in shares:
                for ptr in row:
                    if ptr is not None:
                        closer(ptr)
            self._share_peers = None
        if self.push and self._peers is not None:
            closer = getattr(self.be, "close_shared", None)
            if closer is not None:
                for row in self._peers:
                    for ptr in row:
                        if ptr is not None:
                            closer(ptr)
            self._peers = None
            self.push = False

    def interactions(self) -> int:
        """List entries inside r_c counted by the force kernels since the last call, summed over ranks."""
        if self.counter is None:
            return 0
        c = self.counter.clone()
        self._allreduce_sum(c)
        self.counter.zero_()
        v = int(c.item())
        self._resolve()
        return v
