"""GPU parity at BASELINE.json's full sizes (configs 4 and 5: 2.048 M and 16.384 M
atoms), in the launch configuration bench.py times: cell-ordered storage, the
padded list layout and the force kernel's default lanes / gathers in flight.

The oracle cannot build or step these systems whole within a test, so it checks
SAMPLED row windows -- the first and last rows (cells on the x = 0 and x = L
faces: minimum-image partners), the middle and a seeded random window -- each
computed by the oracle on its own (oracle.list_cells / force_step with a row
range), plus properties that hold at any size (entry count = sum of row
lengths, rows ascending and inside [0, n), total momentum change of a full-list
step zero up to rounding).  Bars as tests/test_gpu_parity.py: lists bit-exact,
momenta C-12 <= 1e-12.
"""
import numpy as np
import pytest
import torch

import lj_inputs
import oracle

pytestmark = pytest.mark.gpu

TOL = 1e-12
WIN = 2048


@pytest.fixture(scope="module")
def lj():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_1806_05713_b200 import build, lj as _lj
    build.build()
    _lj.load()
    return _lj


def _windows(n, seed):
    a = int(np.random.default_rng(seed).integers(WIN, n - 2 * WIN))
    return [(0, WIN), (n // 2 - WIN // 2, n // 2 + WIN // 2), (a, a + WIN), (n - WIN, n)]


@pytest.mark.parametrize("cfg,interleaved", [(4, False), (4, True), (5, True)])
def test_fullsize_sampled_parity(lj, cfg, interleaved):
    dev = torch.device("cuda:0")
    w = lj_inputs.config(cfg)
    perm = oracle.cell_order(w.q, w.L, w.rs)          # the bench's storage order
    qn = np.ascontiguousarray(w.q[perm])
    pn = np.ascontiguousarray(w.p[perm])
    g = lj.geom(w.L, w.rc, w.rs)
    q = lj.pack_aos4(torch.from_numpy(qn).to(dev))
    p = lj.pack_aos4(torch.from_numpy(pn).to(dev))
    b = lj.ListBuilder(w.n, g, False, device=dev, padded=True, interleaved=interleaved)
    gl = b.build(q)
    assert gl.padded and gl.interleaved == interleaved, "the bench's layout: padded (interleaved) rows"
    prow = gl.padded_rows()
    npart = gl.number_of_partners.cpu().numpy()
    assert int(npart.sum()) == gl.n_entries
    # one force step, default launch configuration (as bench.py)
    p1 = p.clone()
    lj.force_step(q, p1, g, w.dt, gl)
    dp = (p1[:, :3] - p[:, :3]).cpu().numpy()
    # full list: every pair's two impulses are exact negatives -> sum zero up to rounding
    assert np.abs(dp.sum(axis=0)).max() <= 1e-11 * np.abs(dp).sum(axis=0).max()
    p1h = p1[:, :3].cpu().numpy()
    for (a, e) in _windows(w.n, cfg):
        ol = oracle.list_cells(qn, w.L, w.rs, False, a, e)
        assert np.array_equal(npart[a:e], ol.number_of_partners), f"row lengths differ in [{a},{e})"
        rows = prow[a:e].cpu().numpy()
        for r in range(a, e):
            assert np.array_equal(rows[r - a, :npart[r]], ol.row(r - a)), f"row {r}"
        ref = oracle.force_step(qn, pn, w.L, w.rc, w.dt, ol)
        S = oracle.abs_contrib(qn, pn, w.L, w.rc, w.dt, ol)
        err = oracle.parity_error(p1h[a:e], ref[a:e], S[a:e])
        assert err <= TOL, f"C-12 error {err} in rows [{a},{e})"


def test_fullsize_half_list_sampled(lj):
    """Config 4's system with the half list (the paper's Alg. 3 layout), sampled rows bit-exact."""
    dev = torch.device("cuda:0")
    w = lj_inputs.config(4)
    perm = oracle.cell_order(w.q, w.L, w.rs)
    qn = np.ascontiguousarray(w.q[perm])
    g = lj.geom(w.L, w.rc, w.rs)
    q = lj.pack_aos4(torch.from_numpy(qn).to(dev))
    gl = lj.ListBuilder(w.n, g, True, device=dev, padded=True, interleaved=True).build(q)
    prow = gl.padded_rows()
    npart = gl.number_of_partners.cpu().numpy()
    assert int(npart.sum()) == gl.n_entries
    for (a, e) in _windows(w.n, 44):
        ol = oracle.list_cells(qn, w.L, w.rs, True, a, e)
        assert np.array_equal(npart[a:e], ol.number_of_partners)
        rows = prow[a:e].cpu().numpy()
        for r in range(a, e):
            assert np.array_equal(rows[r - a, :npart[r]], ol.row(r - a)), f"row {r}"


def test_fullsize_snapshot_parity_after_md_rebuild(lj):
    """SURVEY Pin-13 on the bench path: config 4 through the product MD driver
    (leapfrog kick + drift + bookkeeping, fused lj_rebuild re-sorting into cell
    order) until the list has been rebuilt on evolved positions; the oracle then
    builds sampled rows from that GPU snapshot of q and the pair sets must be
    identical; the permutation carried in p's pad lane stays a permutation."""
    from paper_1806_05713_b200 import md
    dev = torch.device("cuda:0")
    w = lj_inputs.config(4)
    g = lj.geom(w.L, w.rc, w.rs)
    sim = md.LeapfrogMD(md.LibBackend(w.n, g, 0, w.n, dev), w.q, w.p, g, w.dt, reorder=True)
    for _ in range(12):
        sim.kick(w.dt)
        sim.drift_and_exchange()
        if sim.stats.rebuilds >= 1:
            break
    assert sim.stats.rebuilds >= 1, "no bookkeeping rebuild within 12 steps"
    torch.cuda.synchronize()
    qs = np.ascontiguousarray(sim.q[:, :3].cpu().numpy())
    assert qs.min() >= 0.0 and qs.max() < w.L        # wrapped at the rebuild
    ids = np.sort(sim.atom_ids().cpu().numpy())
    assert np.array_equal(ids, np.arange(w.n))
    lst = sim.lst
    assert lst.interleaved, "the bench's layout"
    prow = lst.padded_rows()
    npart = lst.number_of_partners.cpu().numpy()
    for (a, e) in _windows(w.n, 13):
        ol = oracle.list_cells(qs, w.L, w.rs, False, a, e)
        assert np.array_equal(npart[a:e], ol.number_of_partners)
        rows = prow[a:e].cpu().numpy()
        for r in range(a, e):
            assert np.array_equal(rows[r - a, :npart[r]], ol.row(r - a)), f"row {r}"
