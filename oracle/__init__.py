"""ctypes wrapper of the plain-C oracle (oracle/lj_oracle.c).

TEST INFRASTRUCTURE ONLY: imported by tests/, __graft_entry__.smoke() and the
cpu_baseline / --impl reference legs of bench.py -- never by the product
package paper_1806_05713_b200, which must fail loudly without its CUDA library.

Arrays are numpy float64 (n,3) / int32 / int64, C-contiguous.  Every function
cites the passage it follows in lj_oracle.c.
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "lj_oracle.c")
_LIB = os.path.join(_HERE, "liblj_oracle.so")
CFLAGS = ["-O2", "-std=c99", "-ffp-contract=off", "-fno-fast-math", "-shared", "-fPIC"]

_lib = None


def build(force: bool = False) -> str:
    """Compile liblj_oracle.so with gcc (no FMA contraction)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        tmp = _LIB + f".tmp{os.getpid()}"
        subprocess.check_call(["gcc", *CFLAGS, "-o", tmp, _SRC, "-lm"])
        os.replace(tmp, _LIB)
    return _LIB


_LIB_OMP = os.path.join(_HERE, "liblj_oracle_omp.so")
_lib_omp = None


def build_omp(force: bool = False) -> str:
    """liblj_oracle_omp.so: the same source with -fopenmp, for the all-core timing leg only."""
    if force or not os.path.exists(_LIB_OMP) or os.path.getmtime(_LIB_OMP) < os.path.getmtime(_SRC):
        tmp = _LIB_OMP + f".tmp{os.getpid()}"
        subprocess.check_call(["gcc", *CFLAGS, "-fopenmp", "-o", tmp, _SRC, "-lm"])
        os.replace(tmp, _LIB_OMP)
    return _LIB_OMP


def force_step_full_rows_parallel(q, p, L, rc, dt, csr: "CSR", threads: int | None = None):
    """All-core timing of the full-list force step (bit-identical to force_step; never
    used for parity).  p is updated in place (float64, C-contiguous); returns the
    number of OpenMP threads used."""
    global _lib_omp
    if _lib_omp is None:
        build_omp()
        L_ = ctypes.CDLL(_LIB_OMP)
        d, i64, vp = ctypes.c_double, ctypes.c_int64, ctypes.c_void_p
        L_.lj_oracle_force_step_full_rows_parallel.restype = None
        L_.lj_oracle_force_step_full_rows_parallel.argtypes = [vp, vp, i64, d, d, d, i64, i64, vp, vp, vp]
        L_.omp_set_num_threads.argtypes = [ctypes.c_int]
        L_.omp_get_max_threads.restype = ctypes.c_int
        _lib_omp = L_
    if csr.half:
        raise ValueError("force_step_full_rows_parallel: full lists only")
    assert q.dtype == np.float64 and q.flags.c_contiguous and p.dtype == np.float64 and p.flags.c_contiguous
    if threads is not None:
        _lib_omp.omp_set_num_threads(int(threads))
    _lib_omp.lj_oracle_force_step_full_rows_parallel(_p(q), _p(p), q.shape[0], L, rc, dt, csr.row_begin,
                                                     csr.row_end, _p(csr.number_of_partners), _p(csr.pointer),
                                                     _p(csr.sorted_list))
    return int(_lib_omp.omp_get_max_threads())


def lib():
    global _lib
    if _lib is None:
        build()
        L = ctypes.CDLL(_LIB)
        d, i64, i32, vp = ctypes.c_double, ctypes.c_int64, ctypes.c_int, ctypes.c_void_p
        sig = {
            "lj_oracle_sort_pair_list": (i64, [vp, vp, i64, i64, vp, vp]),
            "lj_oracle_list_brute": (i64, [vp, i64, d, d, i32, i64, i64, vp, vp, vp, i64]),
            "lj_oracle_list_cells": (i64, [vp, i64, d, d, i32, i64, i64, vp, vp, vp, i64]),
            "lj_oracle_cells_per_side": (i64, [d, d]),
            "lj_oracle_cell_id": (i64, [d, d, d, d, d]),
            "lj_oracle_cell_order": (i64, [vp, i64, d, d, vp]),
            "lj_oracle_force_step": (None, [vp, vp, i64, d, d, d, i32, i64, i64, vp, vp, vp]),
            "lj_oracle_force_brute": (None, [vp, vp, i64, d, d, d]),
            "lj_oracle_abs_contrib": (None, [vp, vp, i64, d, d, d, i32, i64, i64, vp, vp, vp, vp]),
            "lj_oracle_integrate": (None, [vp, vp, i64, i64, d]),
            "lj_oracle_wrap": (None, [vp, i64, d]),
            "lj_oracle_max_displacement": (d, [vp, vp, i64, i64]),
            "lj_oracle_pair_energy": (d, [d, d]),
            "lj_oracle_energy": (None, [vp, vp, i64, d, d, i32, i64, i64, vp, vp, vp, vp]),
            "lj_oracle_energy_brute": (d, [vp, i64, d, d]),
            "lj_oracle_md_run": (i64, [vp, vp, i64, d, d, d, d, i64, i64, vp]),
        }
        for name, (res, args) in sig.items():
            f = getattr(L, name)
            f.restype = res
            f.argtypes = args
        _lib = L
    return _lib


def _p(a):
    return None if a is None else a.ctypes.data_as(ctypes.c_void_p)


def _f64(a):
    return np.ascontiguousarray(a, dtype=np.float64)


class CSR:
    """Row-local CSR list: number_of_partners[rows], pointer[rows+1] (int64),
    sorted_list[E] (int32, global atom indices); rows [row_begin, row_end)."""

    def __init__(self, number_of_partners, pointer, sorted_list, row_begin, row_end, half):
        self.number_of_partners = number_of_partners
        self.pointer = pointer
        self.sorted_list = sorted_list
        self.row_begin = int(row_begin)
        self.row_end = int(row_end)
        self.half = bool(half)

    @property
    def rows(self):
        return self.row_end - self.row_begin

    @property
    def n_entries(self):
        return int(self.pointer[-1])

    def row(self, r):
        b = self.pointer[r]
        return self.sorted_list[b:b + self.number_of_partners[r]]

    def pairs(self):
        """(E,2) int64 array of (i, j) in global indices, row order."""
        i = np.repeat(np.arange(self.row_begin, self.row_end, dtype=np.int64),
                      self.number_of_partners.astype(np.int64))
        return np.stack([i, self.sorted_list.astype(np.int64)], axis=1)


def _build(fn, q, L, rs, half, row_begin, row_end):
    q = _f64(q)
    n = q.shape[0]
    if row_end is None:
        row_end = n
    rows = row_end - row_begin
    npart = np.zeros(rows, dtype=np.int32)
    ptr = np.zeros(rows + 1, dtype=np.int64)
    need = fn(_p(q), n, L, rs, int(half), row_begin, row_end, _p(npart), _p(ptr), None, 0)
    if need < 0:
        raise ValueError("oracle: unsupported geometry (need L > 0 and floor(L/rs) >= 3)")
    lst = np.zeros(max(need, 1), dtype=np.int32)
    got = fn(_p(q), n, L, rs, int(half), row_begin, row_end, _p(npart), _p(ptr), _p(lst), need)
    assert got == need
    return CSR(npart, ptr, lst[:need], row_begin, row_end, half)


def list_brute(q, L, rs, half, row_begin=0, row_end=None) -> CSR:
    """O(N^2) Verlet list + counting sort."""
    return _build(lib().lj_oracle_list_brute, q, L, rs, half, row_begin, row_end)


def list_cells(q, L, rs, half, row_begin=0, row_end=None) -> CSR:
    """Linked-cell Verlet list, rows ascending."""
    return _build(lib().lj_oracle_list_cells, q, L, rs, half, row_begin, row_end)


def sort_pair_list(pairs, n):
    """Counting sort of a pair list."""
    pairs = np.asarray(pairs, dtype=np.int32).reshape(-1, 2)
    pi = np.ascontiguousarray(pairs[:, 0])
    pj = np.ascontiguousarray(pairs[:, 1])
    off = np.zeros(n + 1, dtype=np.int64)
    j = np.zeros(max(len(pairs), 1), dtype=np.int32)
    lib().lj_oracle_sort_pair_list(_p(pi), _p(pj), len(pairs), n, _p(off), _p(j))
    return off, j[:len(pairs)]


def cells_per_side(L, rs):
    return int(lib().lj_oracle_cells_per_side(L, rs))


def cell_order(q, L, rs):
    q = _f64(q)
    perm = np.zeros(q.shape[0], dtype=np.int64)
    if lib().lj_oracle_cell_order(_p(q), q.shape[0], L, rs, _p(perm)) != 0:
        raise ValueError("oracle: unsupported geometry")
    return perm


def force_step(q, p, L, rc, dt, csr: CSR, inplace=False):
    """Alg. 3 with Alg. 1 arithmetic; returns a new p (or updates p in place)."""
    q = _f64(q)
    if inplace:
        assert p.dtype == np.float64 and p.flags.c_contiguous
    else:
        p = _f64(p).copy()
    lib().lj_oracle_force_step(_p(q), _p(p), q.shape[0], L, rc, dt, int(csr.half), csr.row_begin,
                               csr.row_end, _p(csr.number_of_partners), _p(csr.pointer),
                               _p(csr.sorted_list))
    return p


def force_brute(q, p, L, rc, dt):
    """O(N^2) definition (all pairs i<j, r2 < rc2)."""
    q = _f64(q)
    p = _f64(p).copy()
    lib().lj_oracle_force_brute(_p(q), _p(p), q.shape[0], L, rc, dt)
    return p


def abs_contrib(q, p0, L, rc, dt, csr: CSR):
    """C-12 denominators S (n,3)."""
    q = _f64(q)
    S = np.zeros_like(q)
    lib().lj_oracle_abs_contrib(_p(q), _p(None if p0 is None else _f64(p0)), q.shape[0], L, rc, dt,
                                int(csr.half), csr.row_begin, csr.row_end,
                                _p(csr.number_of_partners), _p(csr.pointer), _p(csr.sorted_list), _p(S))
    return S


def integrate(q, p, dt, begin=0, end=None, inplace=False):
    if inplace:
        assert q.dtype == np.float64 and q.flags.c_contiguous
    else:
        q = _f64(q).copy()
    p = _f64(p)
    lib().lj_oracle_integrate(_p(q), _p(p), begin, q.shape[0] if end is None else end, dt)
    return q


def wrap(q, L):
    q = _f64(q).copy()
    lib().lj_oracle_wrap(_p(q), q.shape[0], L)
    return q


def max_displacement(q, q_ref, begin=0, end=None):
    q = _f64(q)
    return float(lib().lj_oracle_max_displacement(_p(q), _p(_f64(q_ref)), begin,
                                                  q.shape[0] if end is None else end))


def pair_energy(r2, rc):
    return float(lib().lj_oracle_pair_energy(r2, rc))


def energy(q, p, L, rc, csr: CSR):
    """(KE, PE) over the list rows (O7)."""
    q = _f64(q)
    out = np.zeros(2)
    lib().lj_oracle_energy(_p(q), _p(_f64(p)), q.shape[0], L, rc, int(csr.half), csr.row_begin,
                           csr.row_end, _p(csr.number_of_partners), _p(csr.pointer),
                           _p(csr.sorted_list), _p(out))
    return float(out[0]), float(out[1])


def energy_brute(q, L, rc):
    q = _f64(q)
    return float(lib().lj_oracle_energy_brute(_p(q), q.shape[0], L, rc))


def md_run(q, p, L, rc, rs, dt, steps, sample_every=0):
    """KDK velocity Verlet with bookkeeping rebuilds (O8).  Returns
    (q, p, energies[(steps//s+1),3] or None, rebuilds)."""
    q = _f64(q).copy()
    p = _f64(p).copy()
    ns = steps // sample_every + 1 if sample_every > 0 else 0
    e = np.zeros((max(ns, 1), 3))
    rb = lib().lj_oracle_md_run(_p(q), _p(p), q.shape[0], L, rc, rs, dt, steps, sample_every, _p(e))
    if rb < 0:
        raise ValueError("oracle: unsupported geometry")
    return q, p, (e[:ns] if ns else None), int(rb)


def parity_error(p_test, p_ref, S):
    """C-12 primary metric: max |p_test - p_ref| / S (S from abs_contrib)."""
    d = np.abs(np.asarray(p_test, dtype=np.float64) - np.asarray(p_ref, dtype=np.float64))
    with np.errstate(divide="ignore", invalid="ignore"):
        e = np.where(S > 0, d / S, np.where(d > 0, np.inf, 0.0))
    return float(e.max()) if e.size else 0.0
