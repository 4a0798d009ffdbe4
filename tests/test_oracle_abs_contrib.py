"""Pins of the C-12 denominator S = lj_oracle_abs_contrib (reading C-12).

S_ik = |p0_ik| + sum over the pairs (i, j) of atom i with r < r_c of
dt (48 + 24 r^6) / r^14 |d_k|: the sum of the absolute values of the terms
that make up p_ik after one force step (Alg. 1, with the
cancelling "48 - 24 r^6" replaced by its absolute bound 48 + 24 r^6).  Every
parity bar of the GPU suite divides by S, so a slip in S (a dropped dt, r^2
used for |d_k|, a half list counted twice, a missing p0 term) would loosen or
tighten every bar silently.  These pins fix S against values that do not come
from lj_oracle.c:

  * a two-atom closed form, term by term, in exact rational arithmetic;
  * an independent numpy recomputation on config 1 from a brute-force pair
    enumeration (scipy cKDTree, not the oracle's lists) with the coefficient
    written as dt (48 r^-14 + 24 r^-8), for full and half lists;
  * the half list gives the same S as the full list (each pair contributes
    to both of its atoms exactly once either way).
"""
from fractions import Fraction

import numpy as np
import pytest
from scipy.spatial import cKDTree

import lj_inputs
import oracle


@pytest.mark.parametrize("r,dt", [(1.0, 1.0), (1.3, 0.01), (2.2, 0.005), (2.9999, 0.37)])
def test_two_atom_closed_form(r, dt):
    rng = np.random.default_rng(int(r * 1000))
    u = rng.normal(size=3)
    u /= np.linalg.norm(u)
    q = np.array([[5.0, 6.0, 7.0], [5.0, 6.0, 7.0] + r * u])
    d = q[1] - q[0]
    p0 = rng.normal(0, 1, (2, 3))
    # exact rational evaluation of |p0| + dt (48 + 24 r^6)/r^14 |d_k| with r^2 = |d|^2 of the stored doubles
    r2 = sum(Fraction(x) * Fraction(x) for x in d)
    a = Fraction(dt) * (48 + 24 * r2 ** 3) / r2 ** 7
    want = np.array([[float(abs(Fraction(p0[i, k])) + a * abs(Fraction(d[k]))) for k in range(3)] for i in range(2)])
    full = oracle.CSR(np.array([1, 1], dtype=np.int32), np.array([0, 1, 2], dtype=np.int64),
                      np.array([1, 0], dtype=np.int32), 0, 2, False)
    S = oracle.abs_contrib(q, p0, 20.0, 3.0, dt, full)
    assert np.allclose(S, want, rtol=2e-15, atol=0)
    # without p0: the pair terms alone, equal for both atoms
    S0 = oracle.abs_contrib(q, None, 20.0, 3.0, dt, full)
    assert np.allclose(S0[0], [float(a * abs(Fraction(x))) for x in d], rtol=2e-15, atol=0)
    assert np.array_equal(S0[0], S0[1])
    # a half list (row 0 holds j = 1) adds the same term to both atoms
    half = oracle.CSR(np.array([1, 0], dtype=np.int32), np.array([0, 1, 1], dtype=np.int64),
                      np.array([1], dtype=np.int32), 0, 2, True)
    assert np.array_equal(oracle.abs_contrib(q, None, 20.0, 3.0, dt, half), S0)


def test_two_atom_outside_cutoff_contributes_nothing():
    q = np.array([[5.0, 5.0, 5.0], [8.0 + 1e-12, 5.0, 5.0]])
    p0 = np.array([[0.5, -0.25, 1.0], [0.0, 2.0, -3.0]])
    full = oracle.CSR(np.array([1, 1], dtype=np.int32), np.array([0, 1, 2], dtype=np.int64),
                      np.array([1, 0], dtype=np.int32), 0, 2, False)
    assert np.array_equal(oracle.abs_contrib(q, p0, 20.0, 3.0, 0.01, full), np.abs(p0))


def _numpy_S(q, p0, L, rc, dt, rs):
    """Independent S: cKDTree pair enumeration (r < r_s), numpy minimum image and
    coefficient dt (48 r^-14 + 24 r^-8), accumulated with np.add.at."""
    pairs = cKDTree(q, boxsize=L).query_pairs(rs, output_type="ndarray")
    i, j = pairs[:, 0], pairs[:, 1]
    d = q[j] - q[i]
    d = np.where(d > 0.5 * L, d - L, np.where(d < -0.5 * L, d + L, d))
    r2 = np.einsum("ij,ij->i", d, d)
    keep = r2 < rc * rc
    i, j, d, r2 = i[keep], j[keep], d[keep], r2[keep]
    coef = dt * (48.0 * r2 ** -7 + 24.0 * r2 ** -4)
    S = np.abs(p0).copy()
    np.add.at(S, i, coef[:, None] * np.abs(d))
    np.add.at(S, j, coef[:, None] * np.abs(d))
    return S, len(i)


@pytest.mark.parametrize("half", [False, True])
def test_config1_independent_recomputation(half):
    w = lj_inputs.config(1)
    q = lj_inputs.wrap_into_box(w.q.copy(), w.L)
    p0 = np.random.default_rng(5).normal(0, 1, (w.n, 3))
    want, npairs = _numpy_S(q, p0, w.L, w.rc, w.dt, w.rs)
    assert npairs > 200_000   # config 1: ~244.9 k unique pairs inside r_c
    got = oracle.abs_contrib(q, p0, w.L, w.rc, w.dt, oracle.list_cells(q, w.L, w.rs, half))
    # only the summation order and the coefficient's rounding differ
    assert np.max(np.abs(got - want) / want) <= 1e-13
    # the pair terms are a large part of S (a dropped dt or term would show)
    assert np.median((want - np.abs(p0)) / want) > 0.5


def test_slips_are_detected():
    """The plausible slips change S by far more than the 1e-13 agreement above."""
    w = lj_inputs.config(1)
    q = lj_inputs.wrap_into_box(w.q.copy(), w.L)
    p0 = np.zeros((w.n, 3))
    full = oracle.list_cells(q, w.L, w.rs, False)
    S = oracle.abs_contrib(q, p0, w.L, w.rc, w.dt, full)
    S_dt1 = oracle.abs_contrib(q, p0, w.L, w.rc, 1.0, full)           # dt scales S linearly
    assert np.allclose(S_dt1 * w.dt, S, rtol=1e-14)
    S_half_as_full = oracle.abs_contrib(q, p0, w.L, w.rc, w.dt,
                                        oracle.CSR(full.number_of_partners, full.pointer, full.sorted_list,
                                                   0, w.n, True))   # a full list flagged half counts twice
    assert np.allclose(S_half_as_full, 2 * S, rtol=1e-14)
