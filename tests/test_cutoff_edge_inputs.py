"""CPU pins of the r_c-edge test inputs (tests/cutoff_edge.py) and of the
oracle's cutoff decision on them (reading C-4).

The GPU cutoff tests (tests/test_gpu_cutoff.py) are only as strong as their
inputs: these checks make sure the star system really contains many pairs
whose FMA-form and plain-form r^2 straddle r_c^2, and that the oracle decides
them on the plain form (O3) -- the reading the GPU kernels must reproduce.
"""
import numpy as np

import cutoff_edge as ce
import oracle


def test_fma_emulation_is_exact():
    # fma differs from a rounded product + rounded sum exactly where it should
    a = 1.0 + 2.0 ** -30
    assert ce.fma_exact(a, a, -1.0) == 2.0 ** -29 + 2.0 ** -60
    assert (a * a) - 1.0 == 2.0 ** -29          # the plain form loses the 2^-60 term
    assert ce.fma_exact(3.0, 3.0, 0.0) == 9.0


def test_star_system_has_many_straddling_pairs():
    q, n_dis = ce.star_system(0)
    L = 60.0
    assert q.shape == (8 ** 3 * 7, 3)
    assert np.all((q >= 0) & (q < L))
    assert n_dis >= 150, n_dis
    # the disagreements are real pairs of the oracle's list (all r_c pairs are within r_s)
    full = oracle.list_cells(q, L, 3.3, False)
    pr = full.pairs()
    got = ce.disagreements(q, L, pr[:, 0], pr[:, 1])
    # each straddling pair appears twice in a full list (both rows); other pairs rarely straddle
    assert got >= 2 * n_dis
    # stars straddle the box faces (some partner pairs need a periodic image)
    d = q[pr[:, 1]] - q[pr[:, 0]]
    assert np.any(np.abs(d) > 0.5 * L)


def test_oracle_decides_on_the_plain_form():
    """The counterexample: plain r2 = 9 - 2 ulp interacts, FMA r2 = 9.0 would not."""
    q = ce.counterexample_pair()
    d = q[1] - q[0]
    assert ce.r2_plain(d) < 9.0 <= ce.r2_fma(d)
    L = 20.0
    full = oracle.list_cells(q, L, 3.3, False)
    assert full.n_entries == 2
    p = oracle.force_step(q, np.zeros((2, 3)), L, 3.0, 0.01, full)
    # interacting: |dp| = dt |F(r_c)| ~ 1.1e-4 per unit direction, opposite for the two atoms
    assert np.all(np.abs(p[0]) > 1e-5)
    assert np.array_equal(p[0], -p[1])


def test_oracle_force_on_star_system_counts_plain_form():
    q, _ = ce.star_system(0)
    L = 60.0
    full = oracle.list_cells(q, L, 3.3, False)
    pr = full.pairs()
    d = ce.min_image(q[pr[:, 1]] - q[pr[:, 0]], L)
    inside_plain = np.count_nonzero((d[:, 0] * d[:, 0] + d[:, 1] * d[:, 1]) + d[:, 2] * d[:, 2] < 9.0)
    inside_fma = sum(ce.r2_fma(x) < 9.0 for x in d)
    assert inside_plain != inside_fma   # the two readings count different pair sets here
