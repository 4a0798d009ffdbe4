"""GPU parity at the cutoff edge (reading C-4: interact iff r2 < r_c^2 on the
oracle's r2 = (dx*dx + dy*dy) + dz*dz).

The star system (tests/cutoff_edge.py) holds ~3000 pairs within a few ulps of
r_c, ~300 of them placed where an FMA-formed r2 and the oracle's r2 fall on
different sides of r_c^2, in random directions and across the periodic faces.
Every force kernel must reproduce the oracle's interacting set: the momenta
within the C-12 bar (a wrongly classified pair costs ~1e-4 of S, far above
1e-12), and the interaction counter equal, as an integer, to the oracle's count.
"""
import numpy as np
import pytest
import torch

import cutoff_edge as ce
import oracle

pytestmark = pytest.mark.gpu

TOL = 1e-12
L_STAR = 60.0
DT = 0.01


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


def to_dev(x, dev):
    from paper_1806_05713_b200 import lj as _lj
    return _lj.pack_aos4(torch.from_numpy(np.ascontiguousarray(x)).to(dev))


def from_dev(x):
    return x[:, :3].cpu().numpy()


@pytest.fixture(scope="module")
def star():
    q, n_dis = ce.star_system(0, L=L_STAR)
    assert n_dis >= 150
    p0 = np.random.default_rng(17).normal(0, 1, q.shape)
    full = oracle.list_cells(q, L_STAR, 3.3, False)
    half = oracle.list_cells(q, L_STAR, 3.3, True)
    S = oracle.abs_contrib(q, p0, L_STAR, 3.0, DT, full)
    ref = {False: oracle.force_step(q, p0, L_STAR, 3.0, DT, full),
           True: oracle.force_step(q, p0, L_STAR, 3.0, DT, half)}
    pr = full.pairs()
    d = ce.min_image(q[pr[:, 1]] - q[pr[:, 0]], L_STAR)
    inside_full = int(np.count_nonzero((d[:, 0] * d[:, 0] + d[:, 1] * d[:, 1]) + d[:, 2] * d[:, 2] < 9.0))
    return dict(q=q, p0=p0, S=S, ref=ref, inside={False: inside_full, True: inside_full // 2})


IDXV = 1 << 16   # LJ_LANES_IDXV
LANES = ([g | (u << 8) for g in (1, 2, 4, 8, 16, 32) for u in (2, 3, 4)] + [0]
         + [g | (v << 8) | IDXV for g in (1, 2, 4, 8, 16) for v in (2, 4)])


@pytest.mark.parametrize("half,lanes", [(h, x) for h in (False, True) for x in LANES])
def test_force_at_cutoff_edge(lj, dev, star, half, lanes):
    g = lj.geom(L_STAR, 3.0, 3.3)
    q = to_dev(star["q"], dev)
    gl = lj.build_list(q, g, half)
    p = to_dev(star["p0"], dev)
    cnt = torch.zeros(1, dtype=torch.int64, device=dev)
    lj.force_step(q, p, g, DT, gl, lanes_per_row=lanes, n_interactions=cnt)
    assert int(cnt.item()) == star["inside"][half]
    e = oracle.parity_error(from_dev(p), star["ref"][half], star["S"])
    assert e <= TOL, f"C-12 error {e}"


def test_ordered_kernel_at_cutoff_edge(lj, dev, star):
    g = lj.geom(L_STAR, 3.0, 3.3)
    q = to_dev(star["q"], dev)
    p = to_dev(star["p0"], dev)
    lj.force_step(q, p, g, DT, lj.build_list(q, g, False), ordered=True)
    assert np.array_equal(from_dev(p), star["ref"][False])


@pytest.mark.parametrize("lanes", [0, 8 | 512, 4 | 768, 4 | 512, 2 | 512])
def test_half_cells_at_cutoff_edge(lj, dev, star, lanes):
    g = lj.geom(L_STAR, 3.0, 3.3)
    q = to_dev(star["q"], dev)
    b = lj.ListBuilder(q.shape[0], g, True, device=dev)
    gl = b.build(q)
    p = to_dev(star["p0"], dev)
    cnt = torch.zeros(1, dtype=torch.int64, device=dev)
    lj.force_step_half_cells(q, p, g, DT, gl, b.cell_starts(), lanes_per_row=lanes, n_interactions=cnt)
    assert int(cnt.item()) == star["inside"][True]
    assert oracle.parity_error(from_dev(p), star["ref"][True], star["S"]) <= TOL


@pytest.mark.parametrize("layout", ["aos4", "soa", "aos3", "aos8"])
@pytest.mark.parametrize("rcp", ["newton3", "ieee"])
def test_variants_at_cutoff_edge(lj, dev, star, layout, rcp):
    import sys
    sys.path.insert(0, str(__import__("pathlib").Path(__file__).resolve().parents[1] / "tools"))
    from ablation import from_layout, to_layout
    g = lj.geom(L_STAR, 3.0, 3.3)
    q = to_dev(star["q"], dev)
    p = to_dev(star["p0"], dev)
    n = q.shape[0]
    gl = lj.build_list(q, g, False)
    ql = to_layout(q, layout, p)
    pl = None if layout == "aos8" else to_layout(p, layout)
    cnt = torch.zeros(1, dtype=torch.int64, device=dev)
    lj.force_step_variant(layout, rcp, ql, pl, n, g, DT, gl, 4, n_interactions=cnt)
    got = from_layout(ql if layout == "aos8" else pl, layout, n).cpu().numpy()
    assert int(cnt.item()) == star["inside"][False]
    assert oracle.parity_error(got, star["ref"][False], star["S"]) <= TOL


@pytest.mark.parametrize("half", [False, True])
def test_energy_at_cutoff_edge(lj, dev, star, half):
    g = lj.geom(L_STAR, 3.0, 3.3)
    q = to_dev(star["q"], dev)
    p = to_dev(star["p0"], dev)
    e = lj.energy(q, p, g, lj.build_list(q, g, half)).cpu().numpy()
    ke, pe = oracle.energy(star["q"], star["p0"], L_STAR, 3.0, oracle.list_cells(star["q"], L_STAR, 3.3, half))
    assert e[0] == pytest.approx(ke, rel=1e-13)
    assert e[1] == pytest.approx(pe, rel=1e-12, abs=1e-12 * abs(ke))


def test_counterexample_every_kernel(lj, dev):
    """d = (-2.4350224239778626, -0.7106506006664154, 1.6017620043244367)
    has oracle r2 = 8.999999999999998 (interacts) but FMA r2 = 9.0."""
    qn = ce.counterexample_pair()
    L = 20.0
    g = lj.geom(L, 3.0, 3.3)
    q = to_dev(qn, dev)
    for half in (False, True):
        ol = oracle.list_cells(qn, L, 3.3, half)
        ref = oracle.force_step(qn, np.zeros((2, 3)), L, 3.0, DT, ol)
        assert np.all(np.abs(ref[0]) > 1e-5)
        for lanes in LANES:
            p = to_dev(np.zeros((2, 3)), dev)
            cnt = torch.zeros(1, dtype=torch.int64, device=dev)
            lj.force_step(q, p, g, DT, lj.build_list(q, g, half), lanes_per_row=lanes, n_interactions=cnt)
            assert int(cnt.item()) == (1 if half else 2)
            S = oracle.abs_contrib(qn, None, L, 3.0, DT, oracle.list_cells(qn, L, 3.3, False))
            assert oracle.parity_error(from_dev(p), ref, S) <= TOL, (half, lanes)
