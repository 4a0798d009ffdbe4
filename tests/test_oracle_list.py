"""Pins of the oracle's neighbour-list code (DESIGN.md Pin-4, Pin-5, Pin-8, Pin-9).

The Verlet list is pinned to its definition (all pairs with r2 < rs2)
evaluated independently with numpy, to the SPEC worked examples, and to the
closed-form FCC shell counts.
"""
import itertools

import numpy as np
import pytest

import lj_inputs
import oracle
from lj_testutil import golden_kv, golden_lines

RS = lj_inputs.RS
RC = lj_inputs.RC


def numpy_pairs(q, L, rs):
    """Independent definition: set of (i,j), i<j, with minimum-image r2 < rs2."""
    n = q.shape[0]
    out = set()
    rs2 = rs * rs
    for i in range(n - 1):
        d = q[i + 1:] - q[i]
        if L > 0:
            d = np.where(d > 0.5 * L, d - L, np.where(d < -0.5 * L, d + L, d))
        r2 = (d[:, 0] * d[:, 0] + d[:, 1] * d[:, 1]) + d[:, 2] * d[:, 2]
        for j in np.nonzero(r2 < rs2)[0]:
            out.add((i, i + 1 + int(j)))
    return out


def csr_pairs_canonical(csr):
    pr = csr.pairs()
    return set(map(tuple, np.sort(pr, axis=1).tolist()))


def check_csr_shape(csr, half):
    assert csr.pointer[0] == 0
    assert np.all(np.diff(csr.pointer) == csr.number_of_partners)
    for r in range(csr.rows):
        row = csr.row(r)
        i = csr.row_begin + r
        assert np.all(np.diff(row) > 0), "rows ascending and distinct (C-10, CDE property P:487)"
        assert i not in row
        if half:
            assert np.all(row > i)


@pytest.mark.parametrize("line", golden_lines("counting_sort.txt"))
def test_spec_counting_sort(line):
    n, pairs, offs, js = [t.strip() for t in line.split("|")]
    pr = [tuple(map(int, s.split(","))) for s in pairs.split(";")] if pairs else []
    off, j = oracle.sort_pair_list(pr, int(n))
    assert off.tolist() == [int(x) for x in offs.split(",")]
    assert j.tolist() == ([int(x) for x in js.split(",")] if js else [])


def test_counting_sort_stable_random():
    rng = np.random.default_rng(0)
    pr = rng.integers(0, 50, (3000, 2))
    off, j = oracle.sort_pair_list(pr, 50)
    for i in range(50):
        assert j[off[i]:off[i + 1]].tolist() == pr[pr[:, 0] == i, 1].tolist()


@pytest.mark.parametrize("line", golden_lines("two_atom_list.txt"))
@pytest.mark.parametrize("builder", [oracle.list_brute, oracle.list_cells])
def test_spec_two_atom_list(line, builder):
    toks = line.split()
    dist = float(toks[0])
    expected = set() if toks[1] == "-" else {tuple(map(int, toks[1].split("-")))}
    q = np.array([[5.0, 5.0, 5.0], [5.0 + dist, 5.0, 5.0]])
    csr = builder(q, 20.0, RS, half=True)
    assert csr_pairs_canonical(csr) == expected


def test_spec_cells_per_side():
    # box 100, r_s 3.3 -> 30 cells per edge
    assert oracle.cells_per_side(100.0, 3.3) == 30


@pytest.mark.parametrize("seed,n,L", [(0, 300, 10.0), (1, 1000, 10.0), (2, 700, 11.7), (3, 1000, 13.2)])
@pytest.mark.parametrize("half", [True, False])
def test_brute_equals_definition_equals_cells(seed, n, L, half):
    """Pin-5: brute-force list == numpy definition == linked-cell list (set and rows)."""
    q = lj_inputs.random_gas(n, L, seed)
    ref = numpy_pairs(q, L, RS)
    b = oracle.list_brute(q, L, RS, half)
    c = oracle.list_cells(q, L, RS, half)
    check_csr_shape(b, half)
    check_csr_shape(c, half)
    assert csr_pairs_canonical(b) == ref
    assert np.array_equal(b.pointer, c.pointer)
    assert np.array_equal(b.sorted_list, c.sorted_list)
    assert b.n_entries == (len(ref) if half else 2 * len(ref))


def test_config1_lists_brute_equals_cells():
    w = lj_inputs.config(1)
    for half in (True, False):
        b = oracle.list_brute(w.q, w.L, w.rs, half)
        c = oracle.list_cells(w.q, w.L, w.rs, half)
        assert np.array_equal(b.number_of_partners, c.number_of_partners)
        assert np.array_equal(b.sorted_list, c.sorted_list)
    # SURVEY D2 (seed-dependent, loose): ~283.6k unique pairs inside r_s
    assert 280_000 < b.n_entries // 2 < 287_000


@pytest.mark.parametrize("rows", [(0, 1000), (1000, 2000), (1234, 3999), (3999, 4000), (17, 17)])
@pytest.mark.parametrize("half", [True, False])
def test_row_range_is_slice(rows, half):
    w = lj_inputs.config(1)
    full = oracle.list_cells(w.q, w.L, w.rs, half)
    part = oracle.list_cells(w.q, w.L, w.rs, half, rows[0], rows[1])
    for r in range(part.rows):
        assert np.array_equal(part.row(r), full.row(rows[0] + r))


def fcc_shells(rcut):
    """Independent FCC enumeration: lattice vectors (a/2)(h,k,l), h+k+l even."""
    a = lj_inputs.lattice_constant()
    counts = {}
    m = int(np.ceil(2 * rcut / a)) + 1
    for h, k, l in itertools.product(range(-m, m + 1), repeat=3):
        if (h + k + l) % 2 or (h, k, l) == (0, 0, 0):
            continue
        s = h * h + k * k + l * l
        if s * (a / 2) ** 2 < rcut * rcut:
            counts[s] = counts.get(s, 0) + 1
    return counts


def test_perfect_lattice_partner_counts():
    """Pin-4: perfect FCC at rho=1 (C=8): every row has exactly the closed-form count
    of lattice vectors inside r_s (140) -- and inside r_c (134)."""
    n_rs = sum(fcc_shells(RS).values())
    n_rc = sum(fcc_shells(RC).values())
    assert (n_rs, n_rc) == (140, 134)
    C = 8
    q = lj_inputs.fcc_positions(C)
    L = lj_inputs.box_length(C)
    full = oracle.list_cells(q, L, RS, half=False)
    assert np.all(full.number_of_partners == n_rs)
    half = oracle.list_cells(q, L, RS, half=True)
    assert half.n_entries == n_rs * q.shape[0] // 2


def test_paper_benchmark_size_and_group_sizes():
    """PAPER.md:70 N = 119164; PAPER.md:496 half-list groups 'approximately 55 to 80'."""
    g = golden_kv("paper_benchmark.txt")
    w = lj_inputs.config(2)
    assert w.n == int(g["n_atoms"][0])
    assert w.n / w.L ** 3 == pytest.approx(g["number_density"][0], rel=1e-12)
    half = oracle.list_cells(w.q, w.L, w.rs, half=True)
    mean = half.number_of_partners.mean()
    assert g["half_partners_min"][0] <= mean <= g["half_partners_max"][0]
    full = oracle.list_cells(w.q, w.L, w.rs, half=False)
    # Pin-9 (loose): full-list mean 141.8 +- 0.3, min 140, max <= 150
    m = full.number_of_partners
    assert abs(m.mean() - 141.8) < 0.3 and m.min() >= 139 and m.max() <= 151
    assert full.n_entries == 2 * half.n_entries


def test_cell_order_matches_numpy_definition():
    """Cell order = stable sort of the atoms by cell id (z fastest)."""
    w = lj_inputs.config(2)
    perm = oracle.cell_order(w.q, w.L, w.rs)
    nc = int(np.floor(w.L / w.rs))
    inv_w = nc / w.L
    c = np.minimum(np.floor(w.q * inv_w).astype(np.int64), nc - 1)  # q already wrapped
    key = (c[:, 0] * nc + c[:, 1]) * nc + c[:, 2]
    assert np.array_equal(perm, np.argsort(key, kind="stable"))
    assert np.array_equal(np.sort(perm), np.arange(w.n))
    for i in range(0, w.n, 997):
        assert oracle.lib().lj_oracle_cell_id(*w.q[i], w.L, w.rs) == key[i]


def test_list_under_reordering_is_same_pair_set():
    """C-11: lists built in the shuffled and the cell-ordered index spaces are the same
    pair set once mapped back through the permutation."""
    w = lj_inputs.config(1)
    rng = np.random.default_rng(11)
    perm = rng.permutation(w.n)
    a = oracle.list_cells(w.q, w.L, w.rs, half=True)
    b = oracle.list_cells(w.q[perm], w.L, w.rs, half=True)
    pb = perm[b.pairs()]
    assert csr_pairs_canonical(a) == set(map(tuple, np.sort(pb, axis=1).tolist()))
