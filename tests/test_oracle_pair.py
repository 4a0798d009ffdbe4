"""Pins of the oracle's pair arithmetic (DESIGN.md Pin-1, Pin-2, Pin-3).

The impulse coefficient is pinned to (a) the SPEC worked examples (golden),
and (b) the force obtained by differentiating Eq. 1 numerically
in 50-digit arithmetic -- an independent route that fails on a dropped term, a
wrong power or a wrong sign of the momentum update.
"""
import math

import mpmath
import numpy as np
import pytest

import oracle
from lj_testutil import golden_kv, golden_lines

mpmath.mp.dps = 50


def two_atom_dp(r, dt=1.0, L=0.0, axis=0, rc=3.0):
    q = np.zeros((2, 3))
    q[1, axis] = r
    p = oracle.force_brute(q, np.zeros((2, 3)), L, rc, dt)
    return p


def eq1_force_on_i(qi, qj):
    """F_i = -grad_{q_i} V(|q_j - q_i|), V = 4(r^-12 - r^-6) (Eq. 1),
    by 50-digit central differences (independent of the oracle's df formula)."""
    qi = [mpmath.mpf(x) for x in qi]
    qj = [mpmath.mpf(x) for x in qj]

    def V(a):
        r = mpmath.sqrt(sum((qj[k] - a[k]) ** 2 for k in range(3)))
        return 4 * (r ** -12 - r ** -6)

    h = mpmath.mpf("1e-20")
    F = []
    for k in range(3):
        ap = list(qi)
        am = list(qi)
        ap[k] += h
        am[k] -= h
        F.append(-(V(ap) - V(am)) / (2 * h))
    return [float(f) for f in F]


@pytest.mark.parametrize("line", golden_lines("pair_impulse.txt"))
def test_spec_pair_impulse_examples(line):
    # Delta p_i = -df * r_vec with r_vec = (r,0,0), so df = -Delta p_ix / r
    toks = line.split()
    r, df_exp, tol = float(toks[0]), float(toks[1]), float(toks[2])
    p = two_atom_dp(r)
    assert abs(-p[0, 0] / r - df_exp) <= tol
    assert p[0, 1] == 0.0 and p[0, 2] == 0.0
    # Newton 3 exactly (same rounded product added and subtracted)
    assert np.array_equal(p[1], -p[0])


@pytest.mark.parametrize("r", [0.9, 1.0, 1.05, 1.5, 2.0, 2.5, 2.99])
@pytest.mark.parametrize("direction", [(1, 0, 0), (0.3, -0.5, 0.8), (-0.2, -0.1, -0.9)])
def test_impulse_equals_minus_grad_eq1(r, direction):
    """Delta p_i = dt * F_i with F_i = -grad V (Eq. 1) in 3D, dt = 0.01."""
    d = np.asarray(direction, dtype=np.float64)
    d = d / np.linalg.norm(d) * r
    q = np.array([[0.3, 0.4, 0.5], [0.3, 0.4, 0.5]]) + np.vstack([np.zeros(3), d])
    dt = 0.01
    p = oracle.force_brute(q, np.zeros((2, 3)), 0.0, 3.0, dt)
    F = eq1_force_on_i(q[0], q[1])
    for k in range(3):
        assert p[0, k] == pytest.approx(dt * F[k], rel=1e-12, abs=1e-15)
        assert p[1, k] == -p[0, k]


def test_impulse_high_precision_values():
    # closed form -dV/dr * r at 40 digits, evaluated here from Eq. 1 by mpmath
    # i at the origin, j at (r,0,0): F_i,x = -d/dx_i V(x_j - x_i) = +V'(r), dt = 1
    for r in ["0.9", "1.5", "2.5", "2.9"]:
        rr = mpmath.mpf(r)
        dVdr = mpmath.diff(lambda x: 4 * (x ** -12 - x ** -6), rr)
        p = two_atom_dp(float(r))
        assert p[0, 0] == pytest.approx(float(dVdr), rel=1e-14)


def test_single_root_at_2_pow_one_sixth():
    """df has exactly one root for r > 0, at 2^(1/6)."""
    rs = np.linspace(0.9, 2.99, 400)
    signs = np.sign([-two_atom_dp(r)[0, 0] for r in rs])
    changes = np.nonzero(np.diff(signs))[0]
    assert len(changes) == 1
    r0 = rs[changes[0]]
    assert abs(r0 - 2 ** (1 / 6)) < rs[1] - rs[0]


def test_cutoff_strict():
    """Pin-2: r = 3 + 1e-12 -> no interaction; r = 3 - 1e-12 -> interaction."""
    assert np.all(two_atom_dp(3.0 + 1e-12, dt=0.01) == 0.0)
    p = two_atom_dp(3.0 - 1e-12, dt=0.01)
    assert p[0, 0] != 0.0
    # and exactly at r_c (r2 == rc2): excluded (reading C-4: interact iff r2 < rc2)
    assert np.all(two_atom_dp(3.0, dt=0.01) == 0.0)


def test_periodic_minimum_image_pair():
    """Two atoms across the periodic boundary interact through the short image."""
    L = 10.0
    q = np.array([[0.2, 5.0, 5.0], [9.2, 5.0, 5.0]])  # image distance 1.0
    p = oracle.force_brute(q, np.zeros((2, 3)), L, 3.0, 1.0)
    # j's image sits at x = -0.8, i.e. on the -x side of i: repulsion pushes i to +x
    assert p[0, 0] == pytest.approx(24.0, rel=1e-14)
    assert p[1, 0] == pytest.approx(-24.0, rel=1e-14)


def test_spec_oracle_examples():
    g = golden_kv("oracle_sweep.txt")
    p = two_atom_dp(g["two_atom_distance"][0])
    assert np.array_equal(p[0], np.array(g["two_atom_dp0"]))
    assert np.array_equal(p[1], np.array(g["two_atom_dp1"]))
    # equilateral triangle (Pin-3): |dp| = 24 sqrt 3 along the bisectors, total 0
    s = g["triangle_side"][0]
    q = np.array([[0.0, 0.0, 0.0], [s, 0.0, 0.0], [0.5 * s, math.sqrt(3) / 2 * s, 0.0]]) + 5.0
    p = oracle.force_brute(q, np.zeros((3, 3)), 0.0, 3.0, 1.0)
    centroid = q.mean(axis=0)
    for a in range(3):
        assert np.linalg.norm(p[a]) == pytest.approx(g["triangle_dp_magnitude"][0], rel=1e-14)
        out = (q[a] - centroid) / np.linalg.norm(q[a] - centroid)   # repulsive at r=1 < 2^(1/6)
        assert np.dot(p[a], out) == pytest.approx(np.linalg.norm(p[a]), rel=1e-14)
    assert np.all(np.abs(p.sum(axis=0)) <= 1e-13)


@pytest.mark.parametrize("line", golden_lines("shifted_potential.txt"))
def test_spec_potential_examples(line):
    toks = line.split()
    r2, v, tol = float(toks[0]), float(toks[1]), float(toks[2])
    assert abs(oracle.pair_energy(r2, 3.0) - v) <= tol


def test_potential_matches_eq1_and_shift():
    # V(r) - V(rc) from Eq. 1 at 50 digits
    for r in ["0.95", "1.3", "2.2", "2.999"]:
        rr = mpmath.mpf(r)
        V = lambda x: 4 * (x ** -12 - x ** -6)
        exact = float(V(rr) - V(mpmath.mpf(3)))
        assert oracle.pair_energy(float(rr) ** 2, 3.0) == pytest.approx(exact, rel=1e-13, abs=1e-16)
    # the shift constant: V(3) = -5.4794417442387772114e-3
    assert -oracle.pair_energy(1e300, 3.0) == 0.0
    assert float(4 * (mpmath.mpf(3) ** -12 - mpmath.mpf(3) ** -6)) == pytest.approx(-5.4794417442387772114e-3, rel=1e-15)
