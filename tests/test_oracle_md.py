"""Pins of the oracle's NVE loop (reading O8; DESIGN.md Pin-10).

Velocity Verlet is second order: the energy fluctuation scales as dt^2 and the
trajectory is time-reversible.  A wrong kick/drift order, a wrong sign or a
stale list breaks one of these.
"""
import numpy as np
import pytest

import lj_inputs
import oracle


@pytest.fixture(scope="module")
def nve_runs():
    w = lj_inputs.make_system(10, jitter_seed=1, T=1.0, mom_seed=5, dt=0.005)
    out = {}
    for dt, steps in ((0.005, 1000), (0.0025, 1000)):
        q, p, e, rb = oracle.md_run(w.q, w.p, w.L, w.rc, w.rs, dt, steps, sample_every=int(0.05 / dt))
        out[dt] = (q, p, e, rb)
    return w, out


def test_nve_energy_fluctuation_and_dt2_scaling(nve_runs):
    w, out = nve_runs
    q, p, e, rb = out[0.005]
    E = e[:, 2]
    fl = np.abs(E - E[0]).max() / w.n
    # max|E-E0|/N ~ 1.4e-3 at dt = 0.005 over 1000 steps (order of magnitude)
    assert 2e-4 < fl < 5e-3
    # first half (2.5 time units) at dt/2 over the same physical time: ~4x smaller
    E2 = out[0.0025][2][:, 2]
    fl_a = np.abs(E[:51] - E[0]).max()
    fl_b = np.abs(E2[:51] - E2[0]).max()
    assert 2.5 < fl_a / fl_b < 6.5
    # bookkeeping rebuilds roughly every 9 steps at T=1, dt=0.005
    assert 60 < rb < 200
    # momentum stays zero (Newton 3 through every step)
    assert np.all(np.abs(p.sum(axis=0)) < 1e-9)
    # temperature stays near the target (equipartition with T ~ 1 initially, then
    # relaxes toward ~half: potential and kinetic share energy); sanity bounds only
    T = 2 * e[-1, 0] / (3 * (w.n - 1))
    assert 0.2 < T < 1.5


def test_time_reversibility():
    w = lj_inputs.make_system(10, jitter_seed=1, T=1.0, mom_seed=5, dt=0.005)
    q1, p1, _, _ = oracle.md_run(w.q, w.p, w.L, w.rc, w.rs, 0.005, 40)
    q2, p2, _, _ = oracle.md_run(q1, -p1, w.L, w.rc, w.rs, 0.005, 40)
    d = q2 - w.q
    d -= w.L * np.round(d / w.L)       # positions are wrapped at rebuilds
    assert np.abs(d).max() < 1e-9
    assert np.abs(p2 + w.p).max() < 1e-9


def test_single_step_matches_kdk_from_pinned_parts():
    """One KDK step (O8) = half kick (pinned force) + drift (pinned integrate) + half kick."""
    w = lj_inputs.make_system(10, jitter_seed=1, T=1.0, mom_seed=5, dt=0.005)
    dt = 0.005
    q1, p1, _, rb = oracle.md_run(w.q, w.p, w.L, w.rc, w.rs, dt, 1)
    full = oracle.list_cells(w.q, w.L, w.rs, False)
    kick0 = oracle.force_step(w.q, np.zeros_like(w.p), w.L, w.rc, 0.5 * dt, full)
    ph = w.p + kick0
    qq = oracle.integrate(w.q, ph, dt)
    assert rb == 0
    kick1 = oracle.force_step(qq, np.zeros_like(w.p), w.L, w.rc, 0.5 * dt, full)
    assert np.array_equal(q1, qq)
    assert np.array_equal(p1, ph + kick1)
