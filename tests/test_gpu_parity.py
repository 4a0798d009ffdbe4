"""GPU parity: the CUDA path (through the C ABI) against the CPU oracle.

Bars: neighbour lists, integrate, wrap, displacement,
cell order -- bit-exact; momenta after a force step -- C-12 metric
max|p_gpu - p_ref| / S <= 1e-12 (BASELINE.json north_star tolerance with the
denominator of reading C-12); the ordered kernel -- bit-exact.
"""
import ctypes

import numpy as np
import pytest
import torch

import lj_inputs
import oracle

pytestmark = pytest.mark.gpu

TOL = 1e-12


@pytest.fixture(scope="module")
def lj():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_1806_05713_b200 import build, lj as _lj
    build.build()
    _lj.load()
    return _lj


@pytest.fixture(scope="module")
def dev():
    return torch.device("cuda:0")


def to_dev(x, dev, pad=None):
    t = torch.from_numpy(np.ascontiguousarray(x)).to(dev)
    from paper_1806_05713_b200 import lj as _lj
    r = _lj.pack_aos4(t)
    if pad is not None:
        r[:, 3] = torch.from_numpy(pad).to(dev)
    return r


def from_dev(x):
    return x[:, :3].cpu().numpy()


def assert_same_list(gl, ol):
    n_e = gl.n_entries
    assert n_e == ol.n_entries
    assert np.array_equal(gl.number_of_partners.cpu().numpy(), ol.number_of_partners)
    assert np.array_equal(gl.pointer.cpu().numpy(), ol.pointer)
    assert np.array_equal(gl.sorted_list[:n_e].cpu().numpy(), ol.sorted_list)


@pytest.fixture(scope="module")
def systems():
    out = {1: lj_inputs.config(1), 2: lj_inputs.config(2)}
    w3 = lj_inputs.config(3)
    perm = oracle.cell_order(w3.q, w3.L, w3.rs)
    w3.q = np.ascontiguousarray(w3.q[perm])
    w3.p = np.ascontiguousarray(w3.p[perm])
    out[3] = w3
    return out


# ---- lists ------------------------------------------------------------------

@pytest.mark.parametrize("cfg", [1, 2, 3])
@pytest.mark.parametrize("half", [True, False])
def test_list_bit_exact(lj, dev, systems, cfg, half):
    w = systems[cfg]
    g = lj.geom(w.L, w.rc, w.rs)
    gl = lj.build_list(to_dev(w.q, dev), g, half)
    assert_same_list(gl, oracle.list_cells(w.q, w.L, w.rs, half))


@pytest.mark.parametrize("rows", [(0, 1), (17, 17), (1000, 2000), (1234, 3999), (3999, 4000), (0, 4000)])
def test_list_row_ranges(lj, dev, systems, rows):
    w = systems[1]
    g = lj.geom(w.L, w.rc, w.rs)
    gl = lj.build_list(to_dev(w.q, dev), g, False, *rows)
    assert_same_list(gl, oracle.list_cells(w.q, w.L, w.rs, False, *rows))


@pytest.mark.parametrize("seed,n,L", [(0, 1000, 10.0), (1, 3000, 14.0), (2, 1, 10.0), (3, 0, 10.0), (4, 5000, 9.9)])
@pytest.mark.parametrize("half", [True, False])
def test_list_random_gas_and_edges(lj, dev, seed, n, L, half):
    """Dense/ragged random systems incl. nc = 3 (smallest grid), n = 1 and n = 0."""
    q = lj_inputs.random_gas(n, L, seed)
    g = lj.geom(L, 3.0, 3.3)
    qd = to_dev(q.reshape(-1, 3), dev) if n else torch.empty((0, 4), dtype=torch.float64, device=dev)
    gl = lj.build_list(qd, g, half)
    if n:
        assert_same_list(gl, oracle.list_cells(q, L, 3.3, half))
    else:
        assert gl.n_entries == 0 and gl.pointer.cpu().tolist() == [0]


def test_list_unwrapped_positions(lj, dev, systems):
    """Positions drifted outside [0,L) (between rebuilds): cells use wrapped coordinates."""
    w = systems[1]
    rng = np.random.default_rng(5)
    q = w.q + rng.uniform(-0.15, 0.15, w.q.shape)
    g = lj.geom(w.L, w.rc, w.rs)
    gl = lj.build_list(to_dev(q, dev), g, False)
    assert_same_list(gl, oracle.list_cells(q, w.L, w.rs, False))


@pytest.mark.parametrize("half", [True, False])
def test_list_pairs_at_the_search_radius(lj, dev, half):
    """Pairs whose distance is within a few ulps (up to 1e-6) of r_s, in every
    direction and across the periodic faces: the fast builder decides these in
    its exact fp64 band (reading C-4: strict r2 < rs*rs) -- the pair set must
    still equal the oracle's."""
    rs, L = 3.3, 40.0
    rng = np.random.default_rng(11)
    offs = [-1e-6, -1e-9, -1e-12, -4e-15, 0.0, 4e-15, 1e-12, 1e-9, 1e-6]
    pts = []
    centres = [(x, y, z) for x in range(5) for y in range(5) for z in range(5)]
    for k, (x, y, z) in enumerate(centres):
        c = (np.array([x, y, z]) + 0.5) * 8.0 + rng.uniform(-0.5, 0.5, 3)
        if k % 7 == 0:   # straddle a box face
            c[k % 3] = 0.3
        u = rng.normal(size=3)
        u /= np.linalg.norm(u)
        d = rs + offs[k % len(offs)]
        a, b = c - 0.5 * d * u, c + 0.5 * d * u
        pts += [np.mod(a, L), np.mod(b, L)]
    q = np.ascontiguousarray(np.array(pts))
    q = np.where(q >= L, q - L, q)
    g = lj.geom(L, 3.0, rs)
    gl = lj.build_list(to_dev(q, dev), g, half)
    ol = oracle.list_cells(q, L, rs, half)
    assert ol.n_entries > 0
    assert_same_list(gl, ol)


def test_list_capacity_protocol(lj, dev, systems):
    w = systems[1]
    g = lj.geom(w.L, w.rc, w.rs)
    q = to_dev(w.q, dev)
    L = lj.load()
    b = ctypes.c_size_t()
    assert L.lj_build_list_workspace(w.n, g, ctypes.byref(b)) == 0
    ws = torch.empty(b.value, dtype=torch.uint8, device=dev)
    npart = torch.empty(w.n, dtype=torch.int32, device=dev)
    ptr = torch.empty(w.n + 1, dtype=torch.int64, device=dev)
    ne = ctypes.c_int64(-1)
    st = L.lj_build_list(lj._ptr(q), w.n, g, 1, 0, w.n, lj._ptr(npart), lj._ptr(ptr), None, 0, ctypes.byref(ne),
                         lj._ptr(ws), ws.numel(), lj._stream())
    assert st == lj.LJ_ERR_CAPACITY
    assert ne.value == oracle.list_cells(w.q, w.L, w.rs, True).n_entries
    # too-small workspace and partial half range are rejected before launching
    st = L.lj_build_list(lj._ptr(q), w.n, g, 1, 0, w.n, lj._ptr(npart), lj._ptr(ptr), None, 0, ctypes.byref(ne),
                         lj._ptr(ws), 16, lj._stream())
    assert st == lj.LJ_ERR_ARG
    st = L.lj_build_list(lj._ptr(q), w.n, g, 1, 0, 10, lj._ptr(npart), lj._ptr(ptr), None, 0, ctypes.byref(ne),
                         lj._ptr(ws), ws.numel(), lj._stream())
    assert st == lj.LJ_ERR_UNSUPPORTED


def test_cell_order_and_permute(lj, dev, systems):
    w = systems[2]
    g = lj.geom(w.L, w.rc, w.rs)
    q = to_dev(w.q, dev)
    perm = lj.cell_order(q, g)
    assert np.array_equal(perm.cpu().numpy(), oracle.cell_order(w.q, w.L, w.rs))
    qp = lj.permute_rows(q, perm)
    assert np.array_equal(from_dev(qp), w.q[perm.cpu().numpy()])


# ---- force --------------------------------------------------------------------

def oracle_force(w, p0, half):
    ol = oracle.list_cells(w.q, w.L, w.rs, half)
    full = ol if not half else oracle.list_cells(w.q, w.L, w.rs, False)
    return oracle.force_step(w.q, p0, w.L, w.rc, w.dt, ol), oracle.abs_contrib(w.q, p0, w.L, w.rc, w.dt, full), full


@pytest.mark.parametrize("cfg", [1, 2, 3])
@pytest.mark.parametrize("half", [True, False])
@pytest.mark.parametrize("lanes", [0, 1, 4, 8, 16, 32, 4 | 768, 4 | 1024, 16 | 1024,
                                   2 | 512 | 65536, 4 | 512 | 65536, 4 | 1024 | 65536, 8 | 1024 | 65536,
                                   1 | 1024 | 65536])
def test_force_parity(lj, dev, systems, cfg, half, lanes):
    w = systems[cfg]
    rng = np.random.default_rng(cfg)
    p0 = rng.normal(0, 1, (w.n, 3))
    ref, S, full = oracle_force(w, p0, half)
    g = lj.geom(w.L, w.rc, w.rs)
    q = to_dev(w.q, dev)
    gl = lj.build_list(q, g, half)
    p = to_dev(p0, dev)
    cnt = torch.zeros(1, dtype=torch.int64, device=dev)
    lj.force_step(q, p, g, w.dt, gl, lanes_per_row=lanes, n_interactions=cnt)
    got = from_dev(p)
    e = oracle.parity_error(got, ref, S)
    assert e <= TOL, f"C-12 error {e}"
    # interactions counted = entries inside r_c (integer, exact)
    n_in = _entries_inside(w, half)
    assert int(cnt.item()) == n_in


def _entries_inside(w, half):
    ol = oracle.list_cells(w.q, w.L, w.rs, half)
    pr = ol.pairs()
    d = w.q[pr[:, 1]] - w.q[pr[:, 0]]
    d = np.where(d > 0.5 * w.L, d - w.L, np.where(d < -0.5 * w.L, d + w.L, d))
    r2 = (d[:, 0] * d[:, 0] + d[:, 1] * d[:, 1]) + d[:, 2] * d[:, 2]
    return int(np.count_nonzero(r2 < w.rc * w.rc))


@pytest.mark.parametrize("cfg", [1, 2])
def test_ordered_kernel_bit_exact(lj, dev, systems, cfg):
    """Pin-11: the ordered full-list kernel reproduces the oracle bit for bit."""
    w = systems[cfg]
    rng = np.random.default_rng(10 + cfg)
    p0 = rng.normal(0, 1, (w.n, 3))
    ref, _, _ = oracle_force(w, p0, False)
    g = lj.geom(w.L, w.rc, w.rs)
    q = to_dev(w.q, dev)
    gl = lj.build_list(q, g, False)
    p = to_dev(p0, dev)
    lj.force_step(q, p, g, w.dt, gl, ordered=True)
    assert np.array_equal(from_dev(p), ref)


def test_force_row_range_partition(lj, dev, systems):
    """Pin-12 on the GPU: per-range results concatenate to the 1-range result bit-exactly."""
    w = systems[1]
    g = lj.geom(w.L, w.rc, w.rs)
    q = to_dev(w.q, dev)
    p0 = np.random.default_rng(3).normal(0, 1, (w.n, 3))
    whole = to_dev(p0, dev)
    lj.force_step(q, whole, g, w.dt, lj.build_list(q, g, False))
    parts = to_dev(p0, dev)
    for b, e in ((0, 1333), (1333, 2667), (2667, 4000)):
        lj.force_step(q, parts, g, w.dt, lj.build_list(q, g, False, b, e))
    assert torch.equal(whole, parts)


def test_padding_ignored_and_preserved(lj, dev, systems):
    w = systems[1]
    g = lj.geom(w.L, w.rc, w.rs)
    rng = np.random.default_rng(4)
    pad_q, pad_p = rng.normal(0, 1e6, w.n), rng.normal(0, 1e6, w.n)
    p0 = rng.normal(0, 1, (w.n, 3))
    outs = []
    for pq, pp in ((None, None), (pad_q, pad_p)):
        q = to_dev(w.q, dev, pq)
        p = to_dev(p0, dev, pp)
        for half in (True, False):
            lj.force_step(q, p, g, w.dt, lj.build_list(q, g, half))
        if pq is not None:
            assert np.array_equal(q[:, 3].cpu().numpy(), pad_q)
            assert np.array_equal(p[:, 3].cpu().numpy(), pad_p)
        outs.append(from_dev(p))
    ref_half, S, _ = oracle_force(w, p0, True)
    ref, _, _ = oracle_force(w, ref_half, False)
    for o in outs:
        assert oracle.parity_error(o, ref, S + np.abs(ref_half)) <= TOL


@pytest.mark.parametrize("line", [(1.0, 24.0, 0.0), (2 ** (1 / 6), 0.0, 1e-13), (2.5, -1.55998e-2, 5e-8)])
def test_spec_two_atom_examples(lj, dev, line):
    """SPEC.md:56-58 through the C ABI (periodic box large enough to be open)."""
    r, df, tol = line
    q = np.array([[5.0, 5.0, 5.0], [5.0 + r, 5.0, 5.0]])
    g = lj.geom(20.0, 3.0, 3.3)
    qd = to_dev(q, dev)
    for half in (True, False):
        p = to_dev(np.zeros((2, 3)), dev)
        lj.force_step(qd, p, g, 1.0, lj.build_list(qd, g, half))
        got = from_dev(p)
        assert abs(-got[0, 0] / r - df) <= tol
        assert np.array_equal(got[1], -got[0])


def test_cutoff_strict_gpu(lj, dev):
    g = lj.geom(20.0, 3.0, 3.3)
    for r, nonzero in ((3.0 + 1e-12, False), (3.0, False), (3.0 - 1e-12, True)):
        q = to_dev(np.array([[5.0, 5.0, 5.0], [5.0 + r, 5.0, 5.0]]), dev)
        for half in (True, False):
            for ordered in ((False, True) if not half else (False,)):
                p = to_dev(np.zeros((2, 3)), dev)
                lj.force_step(q, p, g, 0.01, lj.build_list(q, g, half), ordered=ordered)
                assert (from_dev(p)[0, 0] != 0.0) == nonzero


def test_perfect_lattice_gpu(lj, dev):
    """Pin-4: 140 partners per atom, zero force, PE/atom = lattice sum."""
    C = 8
    q = lj_inputs.fcc_positions(C)
    L = lj_inputs.box_length(C)
    g = lj.geom(L, 3.0, 3.3)
    qd = to_dev(q, dev)
    full = lj.build_list(qd, g, False)
    assert torch.all(full.number_of_partners == 140)
    p = to_dev(np.zeros_like(q), dev)
    lj.force_step(qd, p, g, 1.0, full)
    S = oracle.abs_contrib(q, None, L, 3.0, 1.0, oracle.list_cells(q, L, 3.3, False))
    assert np.all(np.abs(from_dev(p)) <= 1e-13 * S)
    e = lj.energy(qd, p, g, full).cpu().numpy()
    assert e[1] / q.shape[0] == pytest.approx(-7.762386540408147023, rel=1e-12)


# ---- integrate / bookkeeping / energy ---------------------------------------------

def test_integrate_wrap_displacement_bit_exact(lj, dev, systems):
    w = systems[1]
    rng = np.random.default_rng(8)
    p0 = rng.normal(0, 1, (w.n, 3))
    q = to_dev(w.q, dev)
    p = to_dev(p0, dev)
    qref = q.clone()
    lj.integrate(q, p, 0.37, 100, 3900)
    ref = oracle.integrate(w.q, p0, 0.37, 100, 3900)
    assert np.array_equal(from_dev(q), ref)
    d = lj.max_displacement(q, qref, 50, 3950).item()
    assert d == oracle.max_displacement(ref, w.q, 50, 3950)
    q2 = q.clone()
    lj.wrap(q2, w.L, qref)
    assert np.array_equal(from_dev(q2), oracle.wrap(ref, w.L))
    assert torch.equal(q2, qref)


@pytest.mark.parametrize("half", [True, False])
def test_energy(lj, dev, systems, half):
    w = systems[1]
    p0 = np.random.default_rng(9).normal(0, 1, (w.n, 3))
    g = lj.geom(w.L, w.rc, w.rs)
    q = to_dev(w.q, dev)
    gl = lj.build_list(q, g, half)
    e = lj.energy(q, to_dev(p0, dev), g, gl).cpu().numpy()
    ke, pe = oracle.energy(w.q, p0, w.L, w.rc, oracle.list_cells(w.q, w.L, w.rs, half))
    assert e[0] == pytest.approx(ke, rel=1e-12)
    assert e[1] == pytest.approx(pe, rel=1e-12)


def test_argument_errors(lj, dev, systems):
    w = systems[1]
    q = to_dev(w.q, dev)
    L = lj.load()
    bad = lj.geom(w.L, 3.3, 3.0)   # rc > rs
    st = L.lj_force_step(lj._ptr(q), lj._ptr(q), w.n, bad, 0.01, 0, 0, w.n, None, None, None, lj._stream())
    assert st == lj.LJ_ERR_ARG and b"rc" in L.lj_last_error()
    g = lj.geom(w.L, w.rc, w.rs)
    flat = torch.empty(4 * w.n + 1, dtype=torch.float64, device=dev)
    mis = ctypes.c_void_p(flat.data_ptr() + 8)   # 8-byte aligned, not 32
    st = L.lj_integrate(mis, lj._ptr(q), 0, 10, 0.1, lj._stream())
    assert st == lj.LJ_ERR_ARG
    st = L.lj_force_step(lj._ptr(q), lj._ptr(q), w.n, g, 0.01, 1, 0, 10, None, None, None, lj._stream())
    assert st == lj.LJ_ERR_UNSUPPORTED
    with pytest.raises(TypeError):
        lj.integrate(q.float(), q.float(), 0.1)


def test_kdk_step_matches_oracle(lj, dev):
    """One velocity-Verlet (KDK) step through the ABI vs the oracle's md_run (O8)."""
    w = lj_inputs.make_system(10, jitter_seed=1, T=1.0, mom_seed=5, dt=0.005)
    q1, p1, _, _ = oracle.md_run(w.q, w.p, w.L, w.rc, w.rs, w.dt, 1)
    g = lj.geom(w.L, w.rc, w.rs)
    q = to_dev(w.q, dev)
    p = to_dev(w.p, dev)
    gl = lj.build_list(q, g, False)
    lj.force_step(q, p, g, 0.5 * w.dt, gl)
    lj.integrate(q, p, w.dt)
    lj.force_step(q, p, g, 0.5 * w.dt, gl)
    full = oracle.list_cells(w.q, w.L, w.rs, False)
    S = oracle.abs_contrib(q1, w.p, w.L, w.rc, w.dt, full)
    assert oracle.parity_error(from_dev(p), p1, S) <= TOL
    # positions differ only through p_{1/2} rounding: tiny absolute error
    assert np.abs(from_dev(q) - q1).max() < 1e-14


@pytest.mark.parametrize("cfg", [1, 3])
@pytest.mark.parametrize("half", [True, False])
def test_padded_layout_same_rows(lj, dev, systems, cfg, half):
    """LJ_LIST_PADDED: pointer[r] = r * stride, rows identical to the oracle's."""
    w = systems[cfg]
    g = lj.geom(w.L, w.rc, w.rs)
    q = to_dev(w.q, dev)
    b = lj.ListBuilder(w.n, g, half, device=dev, padded=True)
    gl = b.build(q)
    assert b.padded
    ol = oracle.list_cells(w.q, w.L, w.rs, half)
    assert gl.n_entries == ol.n_entries
    ptr = gl.pointer.cpu().numpy()
    assert np.array_equal(ptr, np.arange(w.n + 1) * lj.LJ_PADDED_ROW_STRIDE)
    npart = gl.number_of_partners.cpu().numpy()
    assert np.array_equal(npart, ol.number_of_partners)
    sl = gl.sorted_list.cpu().numpy()
    for r in range(0, w.n, 97):
        assert np.array_equal(sl[ptr[r]:ptr[r] + npart[r]], ol.row(r))
    # force over the padded list = force over the compact list (same summation order per row)
    p0 = np.random.default_rng(1).normal(0, 1, (w.n, 3))
    pa, pb = to_dev(p0, dev), to_dev(p0, dev)
    lj.force_step(q, pa, g, w.dt, gl)
    lj.force_step(q, pb, g, w.dt, lj.build_list(q, g, half))
    if half:
        ref, S, _ = oracle_force(w, p0, True)
        assert oracle.parity_error(from_dev(pa), ref, S) <= TOL
    else:
        assert torch.equal(pa, pb)


IL_LANES = [0, 1 | 512, 2 | 768, 4 | 512, 4 | 768, 4 | 1024, 8 | 512, 8 | 768, 16 | 512, 32 | 768,
            4 | 512 | (1 << 16), 4 | 1024 | (1 << 16), 8 | 512 | (1 << 16), 2 | 1024 | (1 << 16)]


@pytest.mark.parametrize("cfg", [1, 3])
@pytest.mark.parametrize("half,rows", [(False, None), (True, None), (False, (123, 3001)), (False, (8, 4000))])
def test_interleaved_layout(lj, dev, systems, cfg, half, rows):
    """LJ_LIST_INTERLEAVED (include/liblj.h): pointer[r] = bit 62 | (r//8)*8*S + (r%8)*4,
    entry e of row r at pointer + e + 28*(e//4), pointer[rows] = the padded extent; the rows
    are the oracle's (read from that definition on the host); and every consumer -- the force
    kernel for every lanes / unroll / index-vector variant, the ordered kernel, energy,
    interior rows, partner ranges, the half-cell kernel -- gives the same result on the
    interleaved list as on the plain padded one (bit-identical where deterministic)."""
    w = systems[cfg]
    rb, re_ = rows or (0, w.n)
    g = lj.geom(w.L, w.rc, w.rs)
    q = to_dev(w.q, dev)
    plain = lj.ListBuilder(w.n, g, half, rb, re_, device=dev, padded=True).build(q)
    bil = lj.ListBuilder(w.n, g, half, rb, re_, device=dev, padded=True, interleaved=True)
    il = bil.build(q)
    assert il.interleaved and not plain.interleaved and il.n_entries == plain.n_entries
    R, S = re_ - rb, lj.LJ_PADDED_ROW_STRIDE
    r = np.arange(R, dtype=np.int64)
    ptr = il.pointer.cpu().numpy()
    assert np.array_equal(ptr[:R], (1 << 62) | ((r // 8) * 8 * S + (r % 8) * 4))
    assert ptr[R] == (R + 7) // 8 * 8 * S
    sl = il.sorted_list.cpu().numpy()
    npart = il.number_of_partners.cpu().numpy()
    ol = oracle.list_cells(w.q, w.L, w.rs, half, rb, re_)
    assert np.array_equal(npart, ol.number_of_partners)
    for rr in list(range(0, R, 37)) + [R - 1]:
        e = np.arange(npart[rr])
        assert np.array_equal(sl[(int(ptr[rr]) & ((1 << 62) - 1)) + e + 28 * (e // 4)], ol.row(rr)), rr
    v = torch.arange(S, device=dev)[None, :] < il.number_of_partners[:, None]
    assert torch.equal(il.padded_rows()[v], plain.padded_rows()[v])
    p0 = np.random.default_rng(3).normal(0, 1, (w.n, 3))
    ref, Sab, _ = oracle_force(w, p0, half) if rows is None else (None, None, None)
    for lanes in IL_LANES:
        pa, pb = to_dev(p0, dev), to_dev(p0, dev)
        ca, cb = (torch.zeros(1, dtype=torch.int64, device=dev) for _ in range(2))
        lj.force_step(q, pa, g, w.dt, plain, lanes_per_row=lanes, n_interactions=ca)
        lj.force_step(q, pb, g, w.dt, il, lanes_per_row=lanes, n_interactions=cb)
        assert int(ca.item()) == int(cb.item()), lanes
        if half:   # fp64 REDs: the order of the partner contributions is not deterministic
            assert oracle.parity_error(from_dev(pb), ref, Sab) <= TOL, lanes
        else:
            assert torch.equal(pa, pb), lanes
    if not half:
        pa, pb = to_dev(p0, dev), to_dev(p0, dev)
        lj.force_step(q, pa, g, w.dt, plain, ordered=True)
        lj.force_step(q, pb, g, w.dt, il, ordered=True)
        assert torch.equal(pa, pb)
        assert lj.list_interior(plain) == lj.list_interior(il)
        bounds = [w.n * s // 4 for s in range(4)] + [w.n]
        assert lj.list_partner_ranges(plain, bounds) == lj.list_partner_ranges(il, bounds)
        sink = torch.zeros(4, dtype=torch.float64, device=dev)
        lj.gather_probe(q, il, 0, sink)
    pt = to_dev(p0, dev)
    ea = lj.energy(q, pt, g, plain).cpu().numpy()
    eb = lj.energy(q, pt, g, il).cpu().numpy()
    assert np.allclose(ea, eb, rtol=1e-13, atol=0.0)
    if half and rows is None:   # the per-cell shared-memory kernel reads the same rows
        pc = to_dev(p0, dev)
        lj.force_step_half_cells(q, pc, g, w.dt, il, bil.cell_starts())
        assert oracle.parity_error(from_dev(pc), ref, Sab) <= TOL


def test_padded_layout_falls_back_on_long_rows(lj, dev):
    """Rows longer than the stride (dense gas) -> UNSUPPORTED -> the builder switches to compact."""
    q = lj_inputs.random_gas(5000, 9.9, 4)
    g = lj.geom(9.9, 3.0, 3.3)
    b = lj.ListBuilder(5000, g, False, device=dev, padded=True)
    gl = b.build(to_dev(q, dev))
    assert not b.padded
    assert_same_list(gl, oracle.list_cells(q, 9.9, 3.3, False))


@pytest.mark.parametrize("padded,rows", [(True, (0, 4000)), (False, (0, 4000)), (True, (1000, 3000)),
                                         (False, (123, 456)), ("il", (0, 4000)), ("il", (123, 3001))])
def test_rebuild_fused_equals_steps(lj, dev, systems, padded, rows):
    """lj_rebuild == lj_wrap + lj_cell_order + lj_permute_rows (q, p, q_ref) +
    lj_build_list_ex on the permuted system, bit for bit, for drifted (unwrapped)
    positions; and its cell order equals the oracle's."""
    w = systems[1]
    g = lj.geom(w.L, w.rc, w.rs)
    rng = np.random.default_rng(41)
    q_np = w.q + rng.uniform(-0.15, 0.15, w.q.shape)   # some atoms outside [0, L)
    p_np = rng.normal(0, 1, (w.n, 3))
    pad = np.arange(w.n, dtype=np.float64)
    rb, re_ = rows
    # step by step
    qa = to_dev(q_np, dev, pad)
    pa = to_dev(p_np, dev, pad)
    lj.wrap(qa, w.L)
    perm_a = lj.cell_order(qa, g)
    qa2, pa2 = lj.permute_rows(qa, perm_a), lj.permute_rows(pa, perm_a)
    il = padded == "il"
    padded = bool(padded)
    la = lj.ListBuilder(w.n, g, False, rb, re_, device=dev, padded=padded, interleaved=il).build(qa2)
    # fused
    qb = to_dev(q_np, dev, pad)
    pb = to_dev(p_np, dev, pad)
    qb2, pb2, qref = torch.empty_like(qb), torch.empty_like(pb), torch.empty_like(qb)
    perm_b = torch.empty(w.n, dtype=torch.int64, device=dev)
    lb = lj.ListBuilder(w.n, g, False, rb, re_, device=dev, padded=padded,
                        interleaved=il).rebuild(qb, pb, qb2, pb2, qref, perm_b)
    assert torch.equal(qa, qb)          # wrapped in place
    assert torch.equal(perm_a, perm_b)
    assert torch.equal(qa2, qb2) and torch.equal(pa2, pb2) and torch.equal(qa2, qref)
    assert la.n_entries == lb.n_entries
    assert torch.equal(la.number_of_partners, lb.number_of_partners) and torch.equal(la.pointer, lb.pointer)
    nrow = re_ - rb
    if padded:
        assert la.interleaved == lb.interleaved == il
        v = torch.arange(lj.LJ_PADDED_ROW_STRIDE, device=dev)[None, :] < la.number_of_partners[:, None]
        assert torch.equal(la.padded_rows()[v], lb.padded_rows()[v])
    for r in range(0, nrow, max(1, nrow // 50)):   # valid entries of sampled rows (compact)
        if padded:
            break
        b0, n0 = int(la.pointer[r]), int(la.number_of_partners[r])
        assert torch.equal(la.sorted_list[b0:b0 + n0], lb.sorted_list[b0:b0 + n0])
    # the permutation is the oracle's cell order of the wrapped positions
    assert np.array_equal(perm_b.cpu().numpy(), oracle.cell_order(oracle.wrap(q_np, w.L), w.L, w.rs))
    # and the list is the oracle's list of the permuted system
    ol = oracle.list_cells(from_dev(qb2), w.L, w.rs, False, rb, re_)
    assert int(lb.n_entries) == ol.n_entries


@pytest.mark.parametrize("rows", [(0, 4000), (1000, 3000), (1500, 1800)])
def test_list_interior_and_row_views(lj, dev, systems, rows):
    """lj_list_interior against its definition (numpy over the oracle's list), and
    the force over row views [rb,A) + [A,B) + [B,re) == the force over [rb,re),
    bit for bit (full-list rows are independent)."""
    w = systems[3]   # cell order: the slab's boundary rows sit at its ends
    g = lj.geom(w.L, w.rc, w.rs)
    rb, re_ = rows
    q = to_dev(w.q, dev)
    gl = lj.ListBuilder(w.n, g, False, rb, re_, device=dev, padded=True).build(q)
    A, B = lj.list_interior(gl)
    ol = oracle.list_cells(w.q, w.L, w.rs, False, rb, re_)
    mid = (rb + re_) // 2
    a, b = rb, re_
    for r in range(ol.rows):
        j = ol.row(r)
        if len(j) and (j.min() < rb or j.max() >= re_):
            i = rb + r
            if i < mid:
                a = max(a, i + 1)
            else:
                b = min(b, i)
    assert (A, B) == (a, b)
    p0 = np.random.default_rng(51).normal(0, 1, (w.n, 3))
    pa, pb = to_dev(p0, dev), to_dev(p0, dev)
    lj.force_step(q, pa, g, w.dt, gl)
    for x, y in ((A, B), (rb, A), (B, re_)):
        if y > x:
            lj.force_step(q, pb, g, w.dt, gl.rows_view(x, y))
    assert torch.equal(pa, pb)


@pytest.mark.parametrize("layout", ["aos4", "soa", "aos3", "aos8"])
@pytest.mark.parametrize("lanes", [4, 8])
def test_layout_variants_bit_identical(lj, dev, systems, layout, lanes):
    """NEXT-4 ablation: the paper's layouts change only the gathers and the
    momentum commit -- momenta bit-identical to the AoS4 (library) layout, and
    within C-12 of the oracle."""
    import sys
    sys.path.insert(0, str(__import__("pathlib").Path(__file__).resolve().parents[1] / "tools"))
    from ablation import from_layout, to_layout
    w = systems[1]
    g = lj.geom(w.L, w.rc, w.rs)
    q = to_dev(w.q, dev)
    p0 = np.random.default_rng(61).normal(0, 1, (w.n, 3))
    p = to_dev(p0, dev)
    gl = lj.build_list(q, g, False)
    ql = to_layout(q, layout, p)
    pl = None if layout == "aos8" else to_layout(p, layout)
    cnt = torch.zeros(1, dtype=torch.int64, device=dev)
    lj.force_step_variant(layout, "newton3", ql, pl, w.n, g, w.dt, gl, lanes, n_interactions=cnt)
    got = from_layout(ql if layout == "aos8" else pl, layout, w.n).cpu().numpy()
    pa = to_dev(p0, dev)
    lj.force_step(q, pa, g, w.dt, gl, lanes_per_row=lanes | (2 << 8))
    assert np.array_equal(got, from_dev(pa))
    ref, S, _ = oracle_force(w, p0, False)
    assert oracle.parity_error(got, ref, S) <= TOL
    assert int(cnt.item()) == _entries_inside(w, False)


@pytest.mark.parametrize("rcp,ok", [("newton3", True), ("ieee", True), ("approx", False)])
def test_reciprocal_variants(lj, dev, systems, rcp, ok):
    """NEXT-4: 1/r^2 by MUFU.RCP64H alone misses the 1e-12 bar (why the library
    adds a Newton step); the cubic step and the IEEE reciprocal meet it."""
    import sys
    sys.path.insert(0, str(__import__("pathlib").Path(__file__).resolve().parents[1] / "tools"))
    from ablation import from_layout, to_layout
    w = systems[1]
    g = lj.geom(w.L, w.rc, w.rs)
    q = to_dev(w.q, dev)
    p0 = np.random.default_rng(62).normal(0, 1, (w.n, 3))
    p = to_dev(p0, dev)
    gl = lj.build_list(q, g, False)
    pl = to_layout(p, "aos4")
    lj.force_step_variant("aos4", rcp, to_layout(q, "aos4"), pl, w.n, g, w.dt, gl, 4)
    ref, S, _ = oracle_force(w, p0, False)
    e = oracle.parity_error(from_layout(pl, "aos4", w.n).cpu().numpy(), ref, S)
    assert (e <= TOL) == ok, e


@pytest.mark.parametrize("P,r", [(1, 0), (4, 1), (8, 0), (8, 7), (3, 2)])
def test_list_partner_ranges(lj, dev, systems, P, r):
    """lj_list_partner_ranges against its definition (numpy over the oracle's list)."""
    w = systems[3]
    g = lj.geom(w.L, w.rc, w.rs)
    bounds = [w.n * s // P for s in range(P)] + [w.n]
    rb, re_ = bounds[r], bounds[r + 1]
    gl = lj.ListBuilder(w.n, g, False, rb, re_, device=dev, padded=True).build(to_dev(w.q, dev))
    got = lj.list_partner_ranges(gl, bounds)
    j = oracle.list_cells(w.q, w.L, w.rs, False, rb, re_).sorted_list.astype(np.int64)
    for s in range(P):
        m = j[(j >= bounds[s]) & (j < bounds[s + 1])]
        assert got[s] == ((int(m.min()), int(m.max())) if len(m) else None)


@pytest.mark.parametrize("rows", [(0, 4000), (123, 3456)])
def test_integrate_displacement_fused(lj, dev, systems, rows):
    """lj_integrate_displacement == lj_integrate + lj_max_displacement, bit for bit."""
    w = systems[1]
    rb, re_ = rows
    rng = np.random.default_rng(81)
    q0 = to_dev(w.q, dev)
    p = to_dev(rng.normal(0, 1, (w.n, 3)), dev)
    qref = to_dev(w.q + rng.uniform(-0.05, 0.05, w.q.shape), dev)
    qa, qb = q0.clone(), q0.clone()
    lj.integrate(qa, p, 0.01, rb, re_)
    da = lj.max_displacement(qa, qref, rb, re_)
    db = torch.full((1,), 5.0, dtype=torch.float64, device=dev)
    lj.integrate_displacement(qb, p, qref, 0.01, rb, re_, db)
    assert torch.equal(qa, qb) and float(da.item()) == float(db.item())


# ---- half list without per-entry global atomics ----------

@pytest.mark.parametrize("cfg", [1, 2, 3])
@pytest.mark.parametrize("lanes", [0, 8 | 512, 4 | 768])
@pytest.mark.parametrize("padded", [True, False])
def test_force_half_cells(lj, dev, systems, cfg, lanes, padded):
    """Config 3 (cell order) is the fast path; configs 1 (lattice order) and 2
    (shuffled) put partners outside the cell windows -- the global-RED path."""
    w = systems[cfg]
    p0 = np.random.default_rng(30 + cfg).normal(0, 1, (w.n, 3))
    ref, S, _ = oracle_force(w, p0, True)
    g = lj.geom(w.L, w.rc, w.rs)
    q = to_dev(w.q, dev)
    b = lj.ListBuilder(w.n, g, True, device=dev, padded=padded)
    gl = b.build(q)
    cst = b.cell_starts()
    assert int(cst[-1].item()) == w.n and bool((cst[1:] >= cst[:-1]).all())
    p = to_dev(p0, dev, pad=np.arange(w.n, dtype=np.float64))
    cnt = torch.zeros(1, dtype=torch.int64, device=dev)
    lj.force_step_half_cells(q, p, g, w.dt, gl, cst, lanes_per_row=lanes, n_interactions=cnt)
    e = oracle.parity_error(from_dev(p), ref, S)
    assert e <= TOL, f"C-12 error {e}"
    assert int(cnt.item()) == _entries_inside(w, True)
    assert np.array_equal(p[:, 3].cpu().numpy(), np.arange(w.n, dtype=np.float64))   # pads preserved


def test_force_half_cells_after_rebuild_and_dense_windows(lj, dev, systems):
    """lj_rebuild output (cell order by construction) and a dense gas whose cell
    windows exceed the shared-memory window (all partners take global REDs)."""
    w = systems[1]
    g = lj.geom(w.L, w.rc, w.rs)
    q = to_dev(w.q, dev)
    p0 = to_dev(np.random.default_rng(3).normal(0, 1, (w.n, 3)), dev)
    b = lj.ListBuilder(w.n, g, True, device=dev, padded=True)
    qo, po = torch.empty_like(q), torch.empty_like(p0)
    perm = torch.empty(w.n, dtype=torch.int64, device=dev)
    gl = b.rebuild(q, p0, qo, po, None, perm)
    cst = b.cell_starts()
    qn, pn = from_dev(qo), from_dev(po)
    ol = oracle.list_cells(qn, w.L, w.rs, True)
    full = oracle.list_cells(qn, w.L, w.rs, False)
    ref = oracle.force_step(qn, pn, w.L, w.rc, w.dt, ol)
    S = oracle.abs_contrib(qn, pn, w.L, w.rc, w.dt, full)
    lj.force_step_half_cells(qo, po, g, w.dt, gl, cst)
    assert oracle.parity_error(from_dev(po), ref, S) <= TOL
    # dense gas: 27 cells x ~190 atoms > the window
    qg = lj_inputs.random_gas(5000, 9.9, 4, min_dist_hint=0.7)
    g2 = lj.geom(9.9, 3.0, 3.3)
    b2 = lj.ListBuilder(5000, g2, True, device=dev)
    qd = to_dev(qg, dev)
    gl2 = b2.build(qd)
    pd0 = np.zeros((5000, 3))
    ol2 = oracle.list_cells(qg, 9.9, 3.3, True)
    ref2 = oracle.force_step(qg, pd0, 9.9, 3.0, 0.001, ol2)
    S2 = oracle.abs_contrib(qg, pd0, 9.9, 3.0, 0.001, oracle.list_cells(qg, 9.9, 3.3, False))
    pd = to_dev(pd0, dev)
    lj.force_step_half_cells(qd, pd, g2, 0.001, gl2, b2.cell_starts())
    assert oracle.parity_error(from_dev(pd), ref2, S2) <= TOL


@pytest.mark.parametrize("n", [0, 1, 2])
def test_degenerate_systems_step(lj, dev, n):
    """n = 0, 1, 2 through every step entry point: no partners -> momenta unchanged
    (n = 2: one pair at r = 1.2, C-12 against the oracle)."""
    L = 10.0
    g = lj.geom(L, 3.0, 3.3)
    xyz = np.array([[1.0, 1.0, 1.0], [2.2, 1.0, 1.0]])[:n]
    q = to_dev(xyz.reshape(-1, 3), dev) if n else torch.empty((0, 4), dtype=torch.float64, device=dev)
    p0 = np.random.default_rng(n).normal(0, 1, (n, 3))
    p = to_dev(p0.reshape(-1, 3), dev) if n else torch.empty((0, 4), dtype=torch.float64, device=dev)
    for half in (False, True):
        b = lj.ListBuilder(n, g, half, device=dev, padded=True)
        gl = b.build(q)
        pa = p.clone()
        lj.force_step(q, pa, g, 0.01, gl)
        pb = p.clone()
        if half:
            lj.force_step_half_cells(q, pb, g, 0.01, gl, b.cell_starts())
        else:
            lj.force_step(q, pb, g, 0.01, gl, ordered=True)
        if n:
            ol = oracle.list_cells(xyz, L, 3.3, half)
            ref = oracle.force_step(xyz, p0, L, 3.0, 0.01, ol)
            S = oracle.abs_contrib(xyz, p0, L, 3.0, 0.01, oracle.list_cells(xyz, L, 3.3, False))
            assert oracle.parity_error(from_dev(pa), ref, S) <= TOL
            assert oracle.parity_error(from_dev(pb), ref, S) <= TOL
            if n == 1:
                assert torch.equal(pa, p)
        else:
            assert pa.numel() == 0 and pb.numel() == 0
    out = torch.zeros(1, dtype=torch.float64, device=dev)
    q2 = q.clone()
    lj.integrate_push(q, q2, p, q.clone(), 0.01, 0, n, out, [])
    lj.integrate(q, p, 0.01, 0, n)
    assert torch.equal(q, q2)


@pytest.mark.parametrize("il", [False, True])
def test_deferred_padded_build(lj, dev, systems, il):
    """LJ_LIST_DEFERRED: the same list as the synchronous padded build, n_entries
    resolved after a synchronisation; a row over the stride is reported by resolve()."""
    w = systems[3]
    g = lj.geom(w.L, w.rc, w.rs)
    q = to_dev(w.q, dev)
    ref = lj.ListBuilder(w.n, g, False, device=dev, padded=True, interleaved=il).build(q)
    b = lj.ListBuilder(w.n, g, False, device=dev, padded=True, deferred=True, interleaved=il)
    gl = b.build(q)
    assert gl.n_entries == -1
    torch.cuda.synchronize()
    b.resolve()
    assert gl.n_entries == ref.n_entries
    assert torch.equal(gl.number_of_partners, ref.number_of_partners)
    assert torch.equal(gl.pointer, ref.pointer)
    assert gl.interleaved == ref.interleaved == il
    v = torch.arange(lj.LJ_PADDED_ROW_STRIDE, device=dev)[None, :] < gl.number_of_partners[:, None]
    assert torch.equal(gl.padded_rows()[v], ref.padded_rows()[v])
    # a second deferred build before resolving: the builder synchronises and resolves the first
    gl2 = b.build(q)
    assert gl.n_entries == ref.n_entries
    torch.cuda.synchronize()
    b.resolve(gl2)
    assert gl2.n_entries == ref.n_entries
    # dense gas: rows longer than the stride -> resolve raises
    qg = to_dev(lj_inputs.random_gas(5000, 9.9, 4), dev)
    bd = lj.ListBuilder(5000, lj.geom(9.9, 3.0, 3.3), False, device=dev, padded=True, deferred=True)
    bd.build(qg)
    torch.cuda.synchronize()
    with pytest.raises(lj.LJError):
        bd.resolve()


@pytest.mark.parametrize("il", [False, True])
def test_overflowed_padded_list_stays_in_bounds(lj, dev, il):
    """a padded row over the stride stores min(count, stride) in
    number_of_partners, so a force step that runs before the overflow is
    noticed (deferred build, graph rebuild) reads inside the list; the overflow
    is still reported (resolve() / the graph status)."""
    S = lj.LJ_PADDED_ROW_STRIDE
    qg = to_dev(lj_inputs.random_gas(5000, 9.9, 4), dev)
    g = lj.geom(9.9, 3.0, 3.3)
    bd = lj.ListBuilder(5000, g, False, device=dev, padded=True, deferred=True, interleaved=il)
    lst = bd.build(qg)
    p = to_dev(np.zeros((5000, 3)), dev)
    lj.force_step(qg, p, g, 0.0, lst)             # before resolve(): must not fault
    torch.cuda.synchronize()
    assert int(lst.number_of_partners.max().item()) == S
    with pytest.raises(lj.LJError):
        bd.resolve()
    # graph rebuild: a rho = 1 gas whose first build fits, then a dense cluster appears
    n, L = 8000, 20.0
    q0 = lj_inputs.random_gas(n, L, 9)
    gg = lj.geom(L, 3.0, 3.3)
    q = to_dev(q0, dev)
    pm = to_dev(np.zeros((n, 3)), dev)
    b = lj.ListBuilder(n, gg, False, device=dev, padded=True, interleaved=il)
    b.build(q)
    assert b.padded and b.interleaved == il
    q2 = q0.copy()
    q2[:400] = 10.0 + np.random.default_rng(1).uniform(-1.5, 1.5, (400, 3))   # ~28 atoms per unit volume
    q.copy_(to_dev(q2, dev))
    q_ref = q.clone()
    q_ref[:, 0] += 1.0                            # displacement 1 > margin/2: the graph rebuilds at once
    disp = torch.zeros(1, dtype=torch.float64, device=dev)
    status = torch.zeros(4, dtype=torch.int64, device=dev)
    perm = torch.empty(n, dtype=torch.int64, device=dev)
    gr = lj.MDGraph(q, pm, None, None, q_ref, perm, gg, 0.0, b, disp, None, status, False, 3)
    gr.launch()
    torch.cuda.synchronize()                      # no fault: the steps after the rebuild stay in bounds
    st = status.tolist()
    assert st[0] >= 1 and st[1] == 1              # rebuilt, overflow flagged
    assert int(b.npart.max().item()) == S
    gr.close()


@pytest.mark.parametrize("drift", [0.05, 0.15, 0.4, 1.5])
@pytest.mark.parametrize("half", [False, True])
def test_list_storage_drifted_from_cell_order(lj, dev, systems, drift, half):
    """Storage sorted into cell order once, then atoms moved (fixed row ownership, as
    the multi-rank graph keeps it): cells hold a few atoms whose indices lie in other
    cells' ranges.  The builder ranks the candidates by run intervals (few overlaps) or
    sorts their keys (many) -- the pair set and the ascending rows stay the oracle's."""
    w = systems[3]
    rng = np.random.default_rng(int(drift * 100) + half)
    q = lj_inputs.wrap_into_box(w.q + rng.uniform(-drift, drift, w.q.shape), w.L)
    g = lj.geom(w.L, w.rc, w.rs)
    for padded, il in ((False, False), (True, False), (True, True)):
        b = lj.ListBuilder(w.n, g, half, device=dev, padded=padded, interleaved=il)
        gl = b.build(to_dev(q, dev))
        ol = oracle.list_cells(q, w.L, w.rs, half)
        if padded:
            n_e = ol.n_entries
            assert gl.n_entries == n_e and gl.interleaved == il
            assert np.array_equal(gl.number_of_partners.cpu().numpy(), ol.number_of_partners)
            rows = gl.padded_rows().cpu().numpy()
            for i in range(0, w.n, 97):   # sampled rows: identical, ascending
                k = ol.number_of_partners[i]
                assert np.array_equal(rows[i, :k], ol.sorted_list[ol.pointer[i]:ol.pointer[i] + k])
        else:
            assert_same_list(gl, ol)
