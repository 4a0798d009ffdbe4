"""Seeded synthetic inputs shared by the CUDA path and the CPU oracle.

This module holds NO arithmetic of the method (no distances, no forces, no
lists): it only produces the positions and momenta the paper's benchmark
starts from, so that both sides consume identical arrays.

Workload recipe:
  * FCC lattice, number density rho = 1.0 ("Atoms are placed at
    the face-centered-cubic lattice ... number density is 1.0"), lattice constant
    a = (4/rho)^(1/3), basis {(0,0,0),(0,1/2,1/2),(1/2,0,1/2),(1/2,1/2,0)} a,
    atom index 4*((ix*C+iy)*C+iz)+b  (SURVEY C-19).
  * periodic cube L = C*a = (N/rho)^(1/3)  (BASELINE.json configs[0]; SURVEY C-2).
  * jitter: independent U[-0.05, 0.05) per coordinate in atom order, then wrap
    into [0, L)  (BASELINE.json configs; SURVEY C-14, C-3).
  * momenta: zero (configs 1-3) or Gaussian T=1 with zero net momentum,
    rescaled so sum |p|^2 = 3(N-1)T  (BASELINE.json configs 4-5; SURVEY C-15).
  * storage order: lattice, or a seeded shuffle (config 2), or cell order
    (config 3; the reorder itself is a step of the method and runs in the
    library / oracle, not here).

The paper benchmarks N=119164 ("The number of atoms is 119164");
there is no dataset: every input is this synthetic lattice.
"""
from __future__ import annotations

import dataclasses
import numpy as np

RC = 3.0          # cutoff, "The cutoff length is 3.0"
RS = 3.3          # search length r_s (BASELINE.json north_star / configs; SURVEY C-7)
RHO = 1.0         # number density
JITTER = 0.05     # BASELINE.json configs: "uniform jitter +-0.05"


def lattice_constant(rho: float = RHO) -> float:
    return (4.0 / rho) ** (1.0 / 3.0)


def box_length(cells: int, rho: float = RHO) -> float:
    return cells * lattice_constant(rho)


def fcc_positions(cells: int, rho: float = RHO) -> np.ndarray:
    """(4*C^3, 3) float64 FCC positions, index 4*((ix*C+iy)*C+iz)+b."""
    a = lattice_constant(rho)
    basis = np.array([[0.0, 0.0, 0.0], [0.0, 0.5, 0.5], [0.5, 0.0, 0.5], [0.5, 0.5, 0.0]])
    ix, iy, iz = np.meshgrid(np.arange(cells), np.arange(cells), np.arange(cells), indexing="ij")
    cell = np.stack([ix, iy, iz], axis=-1).reshape(-1, 1, 3).astype(np.float64)
    q = (cell + basis[None, :, :]) * a
    return np.ascontiguousarray(q.reshape(-1, 3))


def wrap_into_box(q: np.ndarray, L: float) -> np.ndarray:
    """x -= L*floor(x/L); guard x == L after rounding (SURVEY C-3)."""
    q = q - L * np.floor(q / L)
    q[q >= L] -= L
    return q


def jittered(q: np.ndarray, L: float, seed: int, amp: float = JITTER) -> np.ndarray:
    rng = np.random.default_rng(seed)
    return wrap_into_box(q + rng.uniform(-amp, amp, q.shape), L)


def gaussian_momenta(n: int, T: float, seed: int) -> np.ndarray:
    """p ~ N(0, sqrt T) per component, mean removed, sum|p|^2 = 3(N-1)T (m = k_B = 1)."""
    rng = np.random.default_rng(seed)
    p = rng.normal(0.0, np.sqrt(T), (n, 3))
    p -= p.mean(axis=0, keepdims=True)
    p *= np.sqrt(3.0 * (n - 1) * T / np.sum(p * p))
    return np.ascontiguousarray(p)


def shuffle_permutation(n: int, seed: int) -> np.ndarray:
    """perm[k] = lattice index of the atom stored at slot k (config 2)."""
    return np.random.default_rng(seed).permutation(n).astype(np.int64)


@dataclasses.dataclass
class Workload:
    name: str
    cells: int
    n: int
    L: float
    rc: float
    rs: float
    dt: float
    q: np.ndarray            # (n, 3) float64, storage order
    p: np.ndarray            # (n, 3) float64, storage order
    order: str               # "lattice" | "shuffled" (cell order is produced by the method)
    lists: tuple             # ("half",) / ("half", "full") / ("full",)
    steps: int
    storage_perm: np.ndarray | None = None   # storage slot -> lattice index, if shuffled


# BASELINE.json configs, seeds per SURVEY.md §8(d).
CONFIGS = {
    1: dict(cells=10, dt=0.01, T=0.0, jitter_seed=1, mom_seed=None, perm_seed=None, lists=("half", "full"), steps=1),
    2: dict(cells=31, dt=0.01, T=0.0, jitter_seed=2, mom_seed=None, perm_seed=3, lists=("half", "full"), steps=100),
    3: dict(cells=31, dt=0.01, T=0.0, jitter_seed=2, mom_seed=None, perm_seed=3, lists=("half", "full"), steps=100),
    4: dict(cells=80, dt=0.01, T=1.0, jitter_seed=4, mom_seed=5, perm_seed=None, lists=("full",), steps=100),
    5: dict(cells=160, dt=0.005, T=1.0, jitter_seed=6, mom_seed=7, perm_seed=None, lists=("full",), steps=1000),
}


def make_system(cells: int, *, jitter_seed: int | None, T: float = 0.0, mom_seed: int | None = None,
                perm_seed: int | None = None, dt: float = 0.01, name: str = "custom",
                lists=("half", "full"), steps: int = 1, rho: float = RHO) -> Workload:
    L = box_length(cells, rho)
    q = fcc_positions(cells, rho)
    if jitter_seed is not None:
        q = jittered(q, L, jitter_seed)
    n = q.shape[0]
    p = gaussian_momenta(n, T, mom_seed) if (T > 0 and mom_seed is not None) else np.zeros((n, 3))
    perm = None
    order = "lattice"
    if perm_seed is not None:
        perm = shuffle_permutation(n, perm_seed)
        q = np.ascontiguousarray(q[perm])
        p = np.ascontiguousarray(p[perm])
        order = "shuffled"
    return Workload(name=name, cells=cells, n=n, L=L, rc=RC, rs=RS, dt=dt, q=q, p=p,
                    order=order, lists=tuple(lists), steps=steps, storage_perm=perm)


def config(k: int) -> Workload:
    c = CONFIGS[k]
    return make_system(c["cells"], jitter_seed=c["jitter_seed"], T=c["T"], mom_seed=c["mom_seed"],
                       perm_seed=c["perm_seed"], dt=c["dt"], name=f"config{k}", lists=c["lists"],
                       steps=c["steps"])


def random_gas(n: int, L: float, seed: int, min_dist_hint: float = 0.0) -> np.ndarray:
    """Uniform random positions in [0,L)^3 (for list/brute-force property tests)."""
    rng = np.random.default_rng(seed)
    return np.ascontiguousarray(rng.uniform(0.0, L, (n, 3)))


def to_aos4(x: np.ndarray, pad: float = 0.0) -> np.ndarray:
    """(n,3) -> (n,4) with a pad column (layout helper for tests; the product path packs on device)."""
    out = np.empty((x.shape[0], 4), dtype=np.float64)
    out[:, :3] = x
    out[:, 3] = pad
    return out
