"""Test inputs with pairs at the cutoff distance r_c, to within a few ulps.

Reading C-4 (PAPER.md:152-156 simple truncation, "r_c +- 1e-12"):
a pair interacts iff r2 < r_c^2 with r2 = (dx*dx + dy*dy) + dz*dz evaluated
without FMA (reading O3).  A kernel that forms r2 with FMAs, as the fast GPU
kernels do for speed, rounds differently in the last bits; for pairs whose
exact squared distance lies within about one ulp of 9.0 the two roundings can
fall on different sides of r_c^2, which adds or drops the truncation jump
(|F(r_c)| dt ~ 1.1e-2 dt per component) and breaks the 1e-12 bar.

`star_system` builds a periodic box of "stars": a centre atom with up to six
partners at distance r_c along a randomly rotated octahedron (so the partners
stay >= r_c sqrt(2) apart), on a grid offset so that stars straddle every box
face.  Each partner's coordinates are then nudged by +-1 ulp per axis (27
candidates) and the candidate is kept whose oracle-style r2 and FMA-style r2
disagree about r2 < r_c^2, where one exists; otherwise a random one.

This is test-input construction (it lives in tests/, not in lj_inputs), so it
may evaluate squared distances: the FMA emulation below is exact rational
arithmetic, not the oracle's or the kernels' code.
"""
from __future__ import annotations

from fractions import Fraction

import numpy as np

RC = 3.0
RC2 = RC * RC


def fma_exact(a: float, b: float, c: float) -> float:
    """fma(a, b, c) = round(a*b + c) (IEEE round-to-nearest-even), by exact rationals."""
    return float(Fraction(a) * Fraction(b) + Fraction(c))


def r2_fma(d) -> float:
    """The fast kernels' form: fma(dz, dz, fma(dy, dy, dx*dx))."""
    dx, dy, dz = (float(x) for x in d)
    return fma_exact(dz, dz, fma_exact(dy, dy, dx * dx))


def r2_plain(d) -> float:
    """Reading O3: (dx*dx + dy*dy) + dz*dz, each operation rounded."""
    dx, dy, dz = (float(x) for x in d)
    return (dx * dx + dy * dy) + dz * dz


def min_image(d: np.ndarray, L: float) -> np.ndarray:
    return np.where(d > 0.5 * L, d - L, np.where(d < -0.5 * L, d + L, d))


def wrap(x: np.ndarray, L: float) -> np.ndarray:
    x = x - L * np.floor(x / L)
    return np.where(x >= L, x - L, x)


def _rotation(rng):
    a = rng.normal(size=(3, 3))
    qm, r = np.linalg.qr(a)
    return qm * np.sign(np.diag(r))


def star_system(seed: int = 0, L: float = 60.0, spacing: float = 7.5, arms: int = 6):
    """(q (n,3) in [0, L), n_disagree): stars of a centre + `arms` partners at r_c."""
    rng = np.random.default_rng(seed)
    m = int(L // spacing)
    off = rng.uniform(-0.3, 0.3, 3)
    pts = []
    n_dis = 0
    octa = np.array([[1, 0, 0], [-1, 0, 0], [0, 1, 0], [0, -1, 0], [0, 0, 1], [0, 0, -1]], dtype=np.float64)
    steps = np.array([(a, b, c) for a in (-1, 0, 1) for b in (-1, 0, 1) for c in (-1, 0, 1)])
    for ix in range(m):
        for iy in range(m):
            for iz in range(m):
                c = wrap(np.array([ix, iy, iz]) * spacing + off + rng.uniform(-0.2, 0.2, 3), L)
                pts.append(c)
                R = _rotation(rng)
                for a in range(arms):
                    base = wrap(c + RC * (R @ octa[a]), L)
                    best, found = None, False
                    for s in rng.permutation(len(steps)):
                        cand = base.copy()
                        for k in range(3):
                            for _ in range(abs(steps[s][k])):
                                cand[k] = np.nextafter(cand[k], np.inf if steps[s][k] > 0 else -np.inf)
                        cand = wrap(cand, L)
                        d = min_image(cand - c, L)
                        if (r2_plain(d) < RC2) != (r2_fma(d) < RC2):
                            best, found = cand, True
                            break
                        if best is None:
                            best = cand
                    n_dis += found
                    pts.append(best)
    q = np.ascontiguousarray(np.array(pts, dtype=np.float64))
    return q, n_dis


def disagreements(q: np.ndarray, L: float, i: np.ndarray, j: np.ndarray) -> int:
    """Pairs (i, j) whose FMA-form and oracle-form r2 fall on different sides of r_c^2."""
    n = 0
    for a, b in zip(i, j):
        d = min_image(q[b] - q[a], L)
        n += (r2_plain(d) < RC2) != (r2_fma(d) < RC2)
    return n


# DESIGN.md / VERDICT r01 counterexample: oracle r2 = 8.999999999999998 (interacts),
# fma(dz, dz, fma(dy, dy, dx*dx)) = 9.0 (does not).
COUNTEREXAMPLE_D = (-2.4350224239778626, -0.7106506006664154, 1.6017620043244367)


def counterexample_pair(L: float = 20.0):
    """Two atoms whose stored difference is exactly COUNTEREXAMPLE_D."""
    qi = np.array([2.5, 1.0, 0.25])   # chosen so that qi + d and (qi + d) - qi are exact
    qj = qi + np.array(COUNTEREXAMPLE_D)
    assert np.array_equal(qj - qi, np.array(COUNTEREXAMPLE_D))
    return np.ascontiguousarray(np.array([qi, qj]))
