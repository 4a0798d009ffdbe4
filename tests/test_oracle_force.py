"""Pins of the oracle's force step (Alg. 3) and energy.

Pin-4 (perfect lattice: zero force, closed-form PE/atom from an independent
lattice sum), Pin-6 (sorted-list result == O(N^2) definition, half == full),
Pin-7 (Newton 3), Pin-12 (row ranges partition the full-list result).
"""
import itertools

import mpmath
import numpy as np
import pytest

import lj_inputs
import oracle

RS, RC = lj_inputs.RS, lj_inputs.RC
TOL = 1e-12   # C-12 tolerance, BASELINE.json north_star "max relative error of 1e-12"


@pytest.fixture(scope="module")
def cfg1():
    w = lj_inputs.config(1)
    half = oracle.list_cells(w.q, w.L, w.rs, True)
    full = oracle.list_cells(w.q, w.L, w.rs, False)
    rng = np.random.default_rng(99)
    p0 = rng.normal(0, 1, (w.n, 3))      # non-zero start momenta exercise "p += impulse"
    S = oracle.abs_contrib(w.q, p0, w.L, w.rc, w.dt, full)
    return w, half, full, p0, S


def test_sorted_list_equals_definition(cfg1):
    w, half, full, p0, S = cfg1
    ref = oracle.force_brute(w.q, p0, w.L, w.rc, w.dt)
    for csr in (half, full):
        p = oracle.force_step(w.q, p0, w.L, w.rc, w.dt, csr)
        assert oracle.parity_error(p, ref, S) <= TOL
        # and the change is not trivially zero
        assert np.abs(p - p0).max() > 1e-3


def test_half_vs_full_and_metric_headroom(cfg1):
    w, half, full, p0, S = cfg1
    ph = oracle.force_step(w.q, p0, w.L, w.rc, w.dt, half)
    pf = oracle.force_step(w.q, p0, w.L, w.rc, w.dt, full)
    e = oracle.parity_error(ph, pf, S)
    assert e <= 1e-14   # reordering alone gives ~1e-15 in this metric


def test_newton3_momentum_conserved(cfg1):
    """Pin-7 (C-13): |sum_i dp_i| <= 1e-12 * sum_i S_i for half and full lists."""
    w, half, full, p0, S = cfg1
    Sd = oracle.abs_contrib(w.q, None, w.L, w.rc, w.dt, full)
    for csr in (half, full):
        dp = oracle.force_step(w.q, np.zeros_like(p0), w.L, w.rc, w.dt, csr)
        tot = np.abs(dp.sum(axis=0))
        assert np.all(tot <= TOL * Sd.sum(axis=0))


def test_full_list_impulses_are_exactly_antisymmetric():
    """Minimum image is sign-symmetric (O2): a two-row full list gives exactly opposite dp."""
    w = lj_inputs.config(1)
    full = oracle.list_cells(w.q, w.L, w.rs, False)
    i = 123
    j = int(full.row(i)[5])
    sub_rows = {i: [j], j: [i]}
    for a, b in sub_rows.items():
        pass
    npart = np.array([1], dtype=np.int32)
    ptr = np.array([0, 1], dtype=np.int64)
    ci = oracle.CSR(npart, ptr, np.array([j], dtype=np.int32), i, i + 1, False)
    cj = oracle.CSR(npart, ptr, np.array([i], dtype=np.int32), j, j + 1, False)
    z = np.zeros((w.n, 3))
    pi = oracle.force_step(w.q, z, w.L, w.rc, w.dt, ci)[i]
    pj = oracle.force_step(w.q, z, w.L, w.rc, w.dt, cj)[j]
    assert np.array_equal(pi, -pj)


@pytest.mark.parametrize("nparts", [2, 3, 8])
def test_row_ranges_partition_full_list(cfg1, nparts):
    """Pin-12: rows are independent -> per-range results concatenate bit-exactly."""
    w, half, full, p0, S = cfg1
    ref = oracle.force_step(w.q, p0, w.L, w.rc, w.dt, full)
    out = p0.copy()
    bounds = [w.n * k // nparts for k in range(nparts + 1)]
    for b, e in zip(bounds[:-1], bounds[1:]):
        part = oracle.list_cells(w.q, w.L, w.rs, False, b, e)
        pr = oracle.force_step(w.q, p0, w.L, w.rc, w.dt, part)
        assert np.array_equal(pr[:b], p0[:b]) and np.array_equal(pr[e:], p0[e:])
        out[b:e] = pr[b:e]
    assert np.array_equal(out, ref)


def test_storage_permutation_invariance(cfg1):
    """Same physics in a permuted index space (config 2/3 semantics, C-11)."""
    w, half, full, p0, S = cfg1
    ref = oracle.force_step(w.q, p0, w.L, w.rc, w.dt, half)
    perm = oracle.cell_order(w.q[::-1].copy(), w.L, w.rs)   # some non-trivial permutation
    qp, pp = w.q[perm], p0[perm]
    lp = oracle.list_cells(qp, w.L, w.rs, True)
    out = oracle.force_step(qp, pp, w.L, w.rc, w.dt, lp)
    back = np.empty_like(out)
    back[perm] = out
    assert oracle.parity_error(back, ref, S) <= TOL


def lattice_pe_per_atom():
    """Independent closed form: 1/2 sum over FCC lattice vectors r < rc of V(r) - V(rc), 50 digits."""
    mpmath.mp.dps = 50
    a = mpmath.mpf(4) ** (mpmath.mpf(1) / 3)
    V = lambda r: 4 * (r ** -12 - r ** -6)
    tot = mpmath.mpf(0)
    m = 6
    for h, k, l in itertools.product(range(-m, m + 1), repeat=3):
        if (h + k + l) % 2 or (h, k, l) == (0, 0, 0):
            continue
        r = a / 2 * mpmath.sqrt(h * h + k * k + l * l)
        if r < 3:
            tot += V(r) - V(mpmath.mpf(3))
    return float(tot / 2)


def test_perfect_lattice_zero_force_and_energy():
    """Pin-4: perfect FCC, inversion symmetry -> zero force; PE/atom = lattice sum."""
    pe_exact = lattice_pe_per_atom()
    assert pe_exact == pytest.approx(-7.762386540408147023, rel=1e-15)
    C = 7
    q = lj_inputs.fcc_positions(C)
    L = lj_inputs.box_length(C)
    n = q.shape[0]
    for half in (True, False):
        csr = oracle.list_cells(q, L, RS, half)
        dp = oracle.force_step(q, np.zeros((n, 3)), L, RC, 1.0, csr)
        S = oracle.abs_contrib(q, None, L, RC, 1.0, csr)
        assert np.all(np.abs(dp) <= 1e-13 * S)
        ke, pe = oracle.energy(q, np.zeros((n, 3)), L, RC, csr)
        assert ke == 0.0
        assert pe / n == pytest.approx(pe_exact, rel=1e-12)
    assert oracle.energy_brute(q, L, RC) / n == pytest.approx(pe_exact, rel=1e-12)


def test_energy_list_equals_brute(cfg1):
    w, half, full, p0, S = cfg1
    ke_h, pe_h = oracle.energy(w.q, p0, w.L, w.rc, half)
    ke_f, pe_f = oracle.energy(w.q, p0, w.L, w.rc, full)
    pe_b = oracle.energy_brute(w.q, w.L, w.rc)
    assert pe_h == pytest.approx(pe_b, rel=1e-12)
    assert pe_f == pytest.approx(pe_b, rel=1e-12)
    assert ke_h == ke_f == pytest.approx(0.5 * np.sum(p0 * p0), rel=1e-12)


def test_impulse_is_minus_energy_gradient(cfg1):
    """dp_i = -dt dE/dq_i for one atom of the jittered lattice, by central differences
    of the (independently pinned) brute-force energy."""
    w, half, full, p0, S = cfg1
    i = 777
    dp = oracle.force_step(w.q, np.zeros((w.n, 3)), w.L, w.rc, 1.0, full)[i]
    h = 1e-6
    for k in range(3):
        qp = w.q.copy()
        qm = w.q.copy()
        qp[i, k] += h
        qm[i, k] -= h
        # energy restricted to atom i's pairs is enough and cheaper: use the full-list
        # energy of the single row (1/2 factor), doubled
        ci = oracle.list_cells(qp, w.L, w.rs, False, i, i + 1)
        cm = oracle.list_cells(qm, w.L, w.rs, False, i, i + 1)
        ep = 2 * oracle.energy(qp, np.zeros((w.n, 3)), w.L, w.rc, ci)[1]
        em = 2 * oracle.energy(qm, np.zeros((w.n, 3)), w.L, w.rc, cm)[1]
        assert dp[k] == pytest.approx(-(ep - em) / (2 * h), rel=1e-6, abs=1e-7)


def test_integrate_and_displacement():
    q = np.array([[0.0, 1.0, 2.0], [3.0, 4.0, 5.0], [1.0, 1.0, 1.0]])
    p = np.array([[1.0, 0.0, 0.0], [0.0, 2.0, 0.0], [3.0, 4.0, 0.0]])
    q1 = oracle.integrate(q, p, 0.5, 1, 3)
    assert np.array_equal(q1[0], q[0])
    assert np.array_equal(q1[1], [3.0, 5.0, 5.0])
    assert np.array_equal(q1[2], [2.5, 3.0, 1.0])
    assert oracle.max_displacement(q1, q) == 2.5          # |(1.5, 2, 0)| = 2.5
    assert oracle.max_displacement(q1, q, 0, 2) == 1.0
    w = oracle.wrap(np.array([[-0.5, 10.0, 10.5]]), 10.0)
    assert np.array_equal(w, [[9.5, 0.0, 0.5]])
    # tiny negative rounds to L in x - L*floor(x/L): guarded back to 0 (C-3)
    w = oracle.wrap(np.array([[-1e-18, 0.0, 0.0]]), 10.0)
    assert 0.0 <= w[0, 0] < 10.0


def test_all_core_timing_build_is_bit_identical(cfg1):
    """The OpenMP timing leg (liblj_oracle_omp.so, bench.py cpu_baseline all-core run)
    splits full-list rows over threads; each row's arithmetic is unchanged."""
    w, half, full, p0, S = cfg1
    ref = oracle.force_step(w.q, p0, w.L, w.rc, w.dt, full)
    p = np.ascontiguousarray(p0.copy())
    q = np.ascontiguousarray(w.q)
    oracle.force_step_full_rows_parallel(q, p, w.L, w.rc, w.dt, full, threads=4)
    assert np.array_equal(p, ref)
