"""Thin Python binding of liblj.so (include/liblj.h): argument marshalling only.

Every step of the hot path runs in the library's CUDA kernels; this module
checks tensor dtype/device/shape/contiguity, passes raw device pointers and
torch's current CUDA stream, and raises LJError on a non-OK status.  There is
no CPU fallback: if liblj.so is missing or no GPU is present, calls fail.
"""
from __future__ import annotations

import ctypes
import math
import dataclasses
import os

import torch

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "liblj.so")

LJ_OK, LJ_ERR_ARG, LJ_ERR_CAPACITY, LJ_ERR_CUDA, LJ_ERR_UNSUPPORTED = 0, 1, 2, 3, 4
LJ_LIST_PADDED, LJ_LIST_DEFERRED, LJ_LIST_INTERLEAVED, LJ_PADDED_ROW_STRIDE = 1, 2, 4, 196   # include/liblj.h
LJ_LANES_IDXV = 1 << 16   # include/liblj.h: index vector loads (lanes_per_row = G | V << 8 | LJ_LANES_IDXV)
LAYOUTS = {"aos4": 0, "soa": 1, "aos3": 2, "aos8": 3}                    # LJ_LAYOUT_*
RECIPROCALS = {"newton3": 0, "newton2": 1, "approx": 2, "ieee": 3}       # LJ_RCP_*

# every symbol include/liblj.h declares
EXPORTS = (
    "lj_pack_aos4", "lj_unpack_aos4", "lj_build_list_workspace", "lj_build_list", "lj_build_list_ex", "lj_rebuild",
    "lj_cell_order",
    "lj_permute_rows", "lj_force_step", "lj_default_lanes", "lj_force_step_ex", "lj_force_step_variant",
    "lj_gather_probe",
    "lj_list_cell_starts", "lj_force_step_half_cells",
    "lj_md_graph_create", "lj_md_graph_launch", "lj_md_graph_force_ms", "lj_md_graph_kernels", "lj_md_graph_destroy",
    "lj_md_capture_rebuild", "lj_copy_records", "lj_copy_bytes", "lj_permute_rows_peers", "lj_publish_scalar",
    "lj_list_interior", "lj_list_partner_ranges", "lj_integrate", "lj_integrate_displacement",
    "lj_integrate_push", "lj_ipc_get_handle", "lj_ipc_open", "lj_ipc_close",
    "lj_wrap",
    "lj_max_displacement", "lj_energy", "lj_status_string", "lj_last_error", "lj_launch_count",
    "lj_version",
)


class LJError(RuntimeError):
    def __init__(self, status, detail):
        super().__init__(f"{_STATUS.get(status, status)}: {detail}")
        self.status = status


_STATUS = {0: "LJ_OK", 1: "LJ_ERR_ARG", 2: "LJ_ERR_CAPACITY", 3: "LJ_ERR_CUDA", 4: "LJ_ERR_UNSUPPORTED"}


class Geom(ctypes.Structure):
    """lj_geom: L (0 = open), rc (cutoff), rs (search length)."""
    _fields_ = [("L", ctypes.c_double), ("rc", ctypes.c_double), ("rs", ctypes.c_double)]


class PushTarget(ctypes.Structure):
    """lj_push_target: rows [lo, hi) also stored to dst (a peer's q replica)."""
    _fields_ = [("dst", ctypes.c_void_p), ("lo", ctypes.c_int64), ("hi", ctypes.c_int64)]


LJ_MAX_PUSH_TARGETS = 63   # include/liblj.h


class MDGraphDesc(ctypes.Structure):
    """lj_md_graph_desc (include/liblj.h)."""
    _fields_ = [("q", ctypes.c_void_p), ("p", ctypes.c_void_p), ("q_alt", ctypes.c_void_p), ("p_alt", ctypes.c_void_p),
                ("q_ref", ctypes.c_void_p), ("perm", ctypes.c_void_p), ("n", ctypes.c_int64), ("g", Geom),
                ("dt", ctypes.c_double), ("number_of_partners", ctypes.c_void_p), ("pointer", ctypes.c_void_p),
                ("sorted_list", ctypes.c_void_p), ("capacity", ctypes.c_int64), ("workspace", ctypes.c_void_p),
                ("workspace_bytes", ctypes.c_size_t), ("disp", ctypes.c_void_p), ("n_interactions", ctypes.c_void_p),
                ("status", ctypes.c_void_p), ("reorder", ctypes.c_int), ("steps", ctypes.c_int),
                ("energy_every", ctypes.c_int), ("energies", ctypes.c_void_p), ("interleaved", ctypes.c_int)]


class MDRebuildDesc(ctypes.Structure):
    """lj_md_rebuild_desc (include/liblj.h)."""
    _fields_ = [("q", ctypes.c_void_p), ("q_ref", ctypes.c_void_p), ("n", ctypes.c_int64), ("g", Geom),
                ("row_begin", ctypes.c_int64), ("row_end", ctypes.c_int64),
                ("number_of_partners", ctypes.c_void_p), ("pointer", ctypes.c_void_p),
                ("sorted_list", ctypes.c_void_p), ("capacity", ctypes.c_int64), ("workspace", ctypes.c_void_p),
                ("workspace_bytes", ctypes.c_size_t), ("disp", ctypes.c_void_p), ("disp_count", ctypes.c_int),
                ("disp_stride", ctypes.c_int64), ("status", ctypes.c_void_p), ("reorder", ctypes.c_int),
                ("q_alt", ctypes.c_void_p), ("p", ctypes.c_void_p), ("p_alt", ctypes.c_void_p),
                ("perm", ctypes.c_void_p), ("p_peers", ctypes.c_void_p), ("n_own", ctypes.c_int64),
                ("interleaved", ctypes.c_int)]


_lib = None


def load() -> ctypes.CDLL:
    """Load liblj.so (built in-tree by paper_1806_05713_b200/build.py).  Fails loudly."""
    global _lib
    if _lib is not None:
        return _lib
    path = LIB_PATH
    if os.environ.get("LJ_LIBRARY") == "check":   # the memory-safety build (bounds checks that trap)
        path = os.path.join(os.path.dirname(LIB_PATH), "liblj_check.so")
    if not os.path.exists(path):
        raise ImportError(f"{os.path.basename(path)} not built ({path}); run python -c "
                          "'import __graft_entry__ as g; g.build()'")
    L = ctypes.CDLL(path)
    vp, i64, i32, d, sz = ctypes.c_void_p, ctypes.c_int64, ctypes.c_int, ctypes.c_double, ctypes.c_size_t
    st = ctypes.c_int
    sig = {
        "lj_pack_aos4": (st, [vp, vp, i64, vp]),
        "lj_unpack_aos4": (st, [vp, vp, i64, vp]),
        "lj_build_list_workspace": (st, [i64, Geom, ctypes.POINTER(sz)]),
        "lj_build_list": (st, [vp, i64, Geom, i32, i64, i64, vp, vp, vp, i64, ctypes.POINTER(i64), vp, sz, vp]),
        "lj_build_list_ex": (st, [vp, i64, Geom, i32, i64, i64, i32, vp, vp, vp, i64, ctypes.POINTER(i64), vp, sz,
                                  vp]),
        "lj_rebuild": (st, [vp, vp, vp, vp, vp, vp, i64, Geom, i32, i64, i64, i32, vp, vp, vp, i64,
                            ctypes.POINTER(i64), vp, sz, vp]),
        "lj_cell_order": (st, [vp, i64, Geom, vp, vp, sz, vp]),
        "lj_permute_rows": (st, [vp, vp, vp, i64, vp]),
        "lj_force_step": (st, [vp, vp, i64, Geom, d, i32, i64, i64, vp, vp, vp, vp]),
        "lj_default_lanes": (i32, [i64, i32]),
        "lj_force_step_ex": (st, [vp, vp, i64, Geom, d, i32, i64, i64, vp, vp, vp, i32, i32, vp, vp]),
        "lj_force_step_variant": (st, [i32, i32, vp, vp, i64, Geom, d, i64, i64, vp, vp, vp, i32, vp, vp]),
        "lj_gather_probe": (st, [vp, i64, i64, i64, vp, vp, vp, i32, vp, vp]),
        "lj_list_cell_starts": (st, [vp, sz, i64, Geom, vp, vp]),
        "lj_md_graph_create": (st, [ctypes.POINTER(MDGraphDesc), ctypes.POINTER(vp)]),
        "lj_md_graph_launch": (st, [vp, vp]),
        "lj_md_capture_rebuild": (st, [ctypes.POINTER(MDRebuildDesc), vp, ctypes.POINTER(ctypes.c_longlong)]),
        "lj_publish_scalar": (st, [vp, vp, vp]),
        "lj_copy_records": (st, [vp, vp, i64, vp]),
        "lj_copy_bytes": (st, [vp, vp, sz, vp]),
        "lj_permute_rows_peers": (st, [vp, vp, vp, vp, vp, i64, i64, i64, vp, i64, Geom, vp, sz, vp]),
        "lj_md_graph_force_ms": (st, [vp, ctypes.POINTER(ctypes.c_float), i32]),
        "lj_md_graph_kernels": (st, [vp, ctypes.POINTER(ctypes.c_longlong), ctypes.POINTER(ctypes.c_longlong)]),
        "lj_md_graph_destroy": (st, [vp]),
        "lj_force_step_half_cells": (st, [vp, vp, i64, Geom, d, vp, vp, vp, vp, i32, vp, vp]),
        "lj_list_interior": (st, [i64, i64, vp, vp, vp, vp, vp]),
        "lj_list_partner_ranges": (st, [i64, i64, vp, vp, vp, vp, i32, vp, vp]),
        "lj_integrate": (st, [vp, vp, i64, i64, d, vp]),
        "lj_integrate_displacement": (st, [vp, vp, vp, i64, i64, d, vp, vp]),
        "lj_integrate_push": (st, [vp, vp, vp, vp, i64, i64, d, vp, ctypes.POINTER(PushTarget), i32, vp]),
        "lj_ipc_get_handle": (st, [vp, ctypes.c_char_p, ctypes.POINTER(i64)]),
        "lj_ipc_open": (st, [ctypes.c_char_p, i64, ctypes.POINTER(vp)]),
        "lj_ipc_close": (st, [vp]),
        "lj_wrap": (st, [vp, vp, i64, d, vp]),
        "lj_max_displacement": (st, [vp, vp, i64, i64, vp, vp]),
        "lj_energy": (st, [vp, vp, i64, Geom, i64, i64, vp, vp, vp, i32, vp, vp]),
        "lj_status_string": (ctypes.c_char_p, [st]),
        "lj_last_error": (ctypes.c_char_p, []),
        "lj_launch_count": (ctypes.c_longlong, []),
        "lj_version": (ctypes.c_char_p, []),
    }
    for name, (res, args) in sig.items():
        f = getattr(L, name)
        f.restype = res
        f.argtypes = args
    _lib = L
    return L


def _check(status):
    if status != LJ_OK:
        raise LJError(status, load().lj_last_error().decode())


def _stream():
    return ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)


def _ptr(t):
    return None if t is None else ctypes.c_void_p(t.data_ptr())


def _addr(t):
    return None if t is None else t.data_ptr()


def _rec(t, name):
    if not (isinstance(t, torch.Tensor) and t.is_cuda and t.dtype == torch.float64 and t.dim() == 2
            and t.shape[1] == 4 and t.is_contiguous()):
        raise TypeError(f"{name}: need a contiguous CUDA float64 (n,4) tensor (AoS4 records)")
    return t


def geom(L, rc, rs) -> Geom:
    return Geom(float(L), float(rc), float(rs))


def launch_count() -> int:
    return int(load().lj_launch_count())


def version() -> str:
    return load().lj_version().decode()


# ---- layout ---------------------------------------------------------------

def pack_aos4(xyz: torch.Tensor, out: torch.Tensor | None = None) -> torch.Tensor:
    """(n,3) float64 CUDA -> (n,4) AoS4 records, pad 0."""
    if not (xyz.is_cuda and xyz.dtype == torch.float64 and xyz.dim() == 2 and xyz.shape[1] == 3):
        raise TypeError("pack_aos4: need a CUDA float64 (n,3) tensor")
    xyz = xyz.contiguous()
    n = xyz.shape[0]
    if out is None:
        out = torch.empty((n, 4), dtype=torch.float64, device=xyz.device)
    _check(load().lj_pack_aos4(_ptr(xyz), _ptr(_rec(out, "out")), n, _stream()))
    return out


def unpack_aos4(q: torch.Tensor, out: torch.Tensor | None = None) -> torch.Tensor:
    """(n,4) AoS4 records -> (n,3) float64 (into `out` if given: contiguous, same device)."""
    _rec(q, "q")
    if out is None:
        out = torch.empty((q.shape[0], 3), dtype=torch.float64, device=q.device)
    elif not (out.is_cuda and out.dtype == torch.float64 and out.is_contiguous() and out.shape == (q.shape[0], 3)):
        raise TypeError("unpack_aos4: out must be a contiguous CUDA float64 (n,3) tensor")
    _check(load().lj_unpack_aos4(_ptr(q), _ptr(out), q.shape[0], _stream()))
    return out


# ---- lists ------------------------------------------------------------------

@dataclasses.dataclass
class CSRList:
    """Row-local sorted list (PAPER.md Fig. sorted_list) on the device."""
    number_of_partners: torch.Tensor   # int32 [rows]
    pointer: torch.Tensor              # int64 [rows+1]
    sorted_list: torch.Tensor          # int32 [capacity] (first n_entries valid)
    n_entries: int                     # -1 while a deferred build is unresolved (ListBuilder.resolve)
    row_begin: int
    row_end: int
    half: bool
    padded: bool = False        # LJ_LIST_PADDED layout (rows at a fixed stride)
    interleaved: bool = False   # LJ_LIST_INTERLEAVED (padded rows in blocks of 8, entries interleaved by 4)

    @property
    def rows(self):
        return self.row_end - self.row_begin

    def rows_view(self, a: int, b: int) -> "CSRList":
        """The rows [a, b) (global indices, within this list's range) as a list of
        their own: offset views of number_of_partners and pointer, same entries."""
        if not (self.row_begin <= a <= b <= self.row_end):
            raise ValueError(f"rows_view: [{a},{b}) not within [{self.row_begin},{self.row_end})")
        o = a - self.row_begin
        return CSRList(self.number_of_partners[o:o + (b - a)], self.pointer[o:], self.sorted_list, self.n_entries,
                       a, b, self.half, self.padded, self.interleaved)

    def padded_rows(self) -> torch.Tensor:
        """The rows of a padded list (either layout) as a [rows, LJ_PADDED_ROW_STRIDE] int32
        tensor in row-major order (entries past number_of_partners undefined).  For tests and
        tools; a view for the plain padded layout, a copy for the interleaved one."""
        if not self.padded:
            raise ValueError("padded_rows: not a padded list")
        base = int(self.pointer[0].item()) & ((1 << 62) - 1)
        R, S = self.rows, LJ_PADDED_ROW_STRIDE
        if not self.interleaved:
            return self.sorted_list[base:base + R * S].view(R, S)
        if base % (8 * S) != 0:
            raise ValueError("padded_rows: an interleaved list view must start at a block of 8 rows")
        nb = (R + 7) // 8
        blk = self.sorted_list[base:base + nb * 8 * S].view(nb, S // 4, 8, 4)
        return blk.permute(0, 2, 1, 3).reshape(nb * 8, S)[:R]


class ListBuilder:
    """Holds the build workspace and a growing list buffer for repeated rebuilds."""

    def __init__(self, n: int, g: Geom, half: bool, row_begin: int = 0, row_end: int | None = None,
                 device=None, headroom: float = 1.15, initial_per_row: int = 0, padded: bool = False,
                 deferred: bool = False, interleaved: bool = False):
        self.n, self.g, self.half = int(n), g, bool(half)
        self.row_begin = int(row_begin)
        self.row_end = int(n if row_end is None else row_end)
        self.device = torch.device("cuda") if device is None else torch.device(device)
        self.headroom = headroom
        b = ctypes.c_size_t(0)
        _check(load().lj_build_list_workspace(self.n, g, ctypes.byref(b)))
        self.workspace = torch.empty(max(int(b.value), 1), dtype=torch.uint8, device=self.device)
        rows = self.row_end - self.row_begin
        self.npart = torch.empty(max(rows, 1), dtype=torch.int32, device=self.device)
        self.pointer = torch.empty(rows + 1, dtype=torch.int64, device=self.device)
        self.padded = padded
        self.interleaved = bool(interleaved) and padded   # LJ_LIST_INTERLEAVED (padded layouts only)
        alloc_rows = rows
        if padded:
            initial_per_row = LJ_PADDED_ROW_STRIDE
            if self.interleaved:
                alloc_rows = (rows + 7) // 8 * 8
        self.sorted_list = torch.empty(max(int(alloc_rows * initial_per_row), 1), dtype=torch.int32,
                                       device=self.device)
        self.rebuilds = 0
        # LJ_LIST_DEFERRED (padded layout only): the build does not synchronise; its status
        # lands in pinned memory and is checked by resolve() after a later synchronisation
        self.deferred = bool(deferred) and padded
        self.status = torch.zeros(2, dtype=torch.int64, pin_memory=True) if self.deferred else None
        self._unresolved = None

    def enable_deferred(self) -> None:
        """Switch a padded builder to LJ_LIST_DEFERRED builds (no host round trip per build)."""
        if self.padded and not self.deferred:
            self.deferred = True
            self.status = torch.zeros(2, dtype=torch.int64, pin_memory=True)

    def max_row_length(self) -> int:
        """Longest row of the last (resolved) build -- a host synchronisation."""
        rows = self.row_end - self.row_begin
        return int(self.npart[:rows].max().item()) if rows > 0 else 0

    def _flags(self):
        return ((LJ_LIST_PADDED if self.padded else 0) | (LJ_LIST_DEFERRED if self.deferred and self.padded else 0)
                | (LJ_LIST_INTERLEAVED if self.interleaved and self.padded else 0))

    def build(self, q: torch.Tensor) -> CSRList:
        _rec(q, "q")
        return self._build(lambda ne: load().lj_build_list_ex(
            _ptr(q), self.n, self.g, int(self.half), self.row_begin, self.row_end,
            self._flags(), _ptr(self.npart), _ptr(self.pointer), _ptr(self.sorted_list),
            self.sorted_list.numel(), ne, _ptr(self.workspace), self.workspace.numel(), _stream()))

    def cell_starts(self, out: torch.Tensor | None = None) -> torch.Tensor:
        """lj_list_cell_starts: the last build's cell starts (int64, ncell + 1) -- the cell
        structure lj_force_step_half_cells works on."""
        nc = int(math.floor(self.g.L / self.g.rs))
        if out is None:
            out = torch.empty(nc ** 3 + 1, dtype=torch.int64, device=self.device)
        _check(load().lj_list_cell_starts(_ptr(self.workspace), self.workspace.numel(), self.n, self.g, _ptr(out),
                                          _stream()))
        return out

    def rebuild(self, q: torch.Tensor, p: torch.Tensor | None, q_out: torch.Tensor, p_out: torch.Tensor | None,
                q_ref: torch.Tensor | None, perm: torch.Tensor) -> CSRList:
        """lj_rebuild: wrap q in place, permute (q, p) into cell order (q_out, p_out, q_ref = q_out,
        perm[new] = old) and build the list of the permuted system, from one cell pass."""
        for t, name in ((q, "q"), (q_out, "q_out"), (p, "p"), (p_out, "p_out"), (q_ref, "q_ref")):
            if t is not None:
                _rec(t, name)
        if not (perm.is_cuda and perm.dtype == torch.int64 and perm.numel() == self.n):
            raise TypeError("rebuild: perm must be a CUDA int64 tensor of length n")
        return self._build(lambda ne: load().lj_rebuild(
            _ptr(q), _ptr(p), _ptr(q_out), _ptr(p_out), _ptr(q_ref), _ptr(perm), self.n, self.g, int(self.half),
            self.row_begin, self.row_end, self._flags(), _ptr(self.npart),
            _ptr(self.pointer), _ptr(self.sorted_list), self.sorted_list.numel(), ne,
            _ptr(self.workspace), self.workspace.numel(), _stream()))

    def resolve(self, lst: CSRList | None = None) -> None:
        """Finish a deferred build once the stream has passed it (after any synchronisation):
        fills lst.n_entries, or raises if a row overflowed the padded stride."""
        if self._unresolved is None:
            return
        lst = self._unresolved if lst is None else lst
        self._unresolved = None
        if int(self.status[1]) != 0:
            raise LJError(LJ_ERR_UNSUPPORTED, "deferred build: a row has more than %d partners "
                          "(build with deferred=False: the builder then switches to the compact layout)"
                          % LJ_PADDED_ROW_STRIDE)
        lst.n_entries = int(self.status[0])

    def _build(self, call) -> CSRList:
        if self.deferred and self.padded:
            if self._unresolved is not None:   # the previous deferred status is still in flight
                torch.cuda.current_stream().synchronize()
                self.resolve()
            self.status.zero_()
            _check(call(ctypes.cast(self.status.data_ptr(), ctypes.POINTER(ctypes.c_int64))))
            self.rebuilds += 1
            rows = self.row_end - self.row_begin
            lst = CSRList(self.npart[:rows], self.pointer, self.sorted_list, -1, self.row_begin, self.row_end,
                          self.half, True, self.interleaved)
            self._unresolved = lst
            return lst
        ne = ctypes.c_int64(0)
        for _ in range(3):
            st = call(ctypes.byref(ne))
            if st == LJ_ERR_UNSUPPORTED and self.padded:   # a row longer than the stride: compact from now on
                self.padded = False
                self.interleaved = False
                continue
            if st == LJ_ERR_CAPACITY:
                cap = int(ne.value * self.headroom) + 1024
                self.sorted_list = torch.empty(cap, dtype=torch.int32, device=self.device)
                continue
            _check(st)
            break
        else:
            raise LJError(LJ_ERR_CAPACITY, "list capacity did not converge")
        self.rebuilds += 1
        rows = self.row_end - self.row_begin
        return CSRList(self.npart[:rows], self.pointer, self.sorted_list, int(ne.value), self.row_begin,
                       self.row_end, self.half, self.padded, self.interleaved)


def build_list(q: torch.Tensor, g: Geom, half: bool, row_begin: int = 0, row_end: int | None = None) -> CSRList:
    """One-shot lj_build_list (allocates its own workspace and exact-size list)."""
    b = ListBuilder(q.shape[0], g, half, row_begin, row_end, device=q.device, headroom=1.0)
    return b.build(q)


def cell_order(q: torch.Tensor, g: Geom) -> torch.Tensor:
    """perm[new] = old: stable sort by cell id (BASELINE.json config 3)."""
    _rec(q, "q")
    n = q.shape[0]
    b = ctypes.c_size_t(0)
    _check(load().lj_build_list_workspace(n, g, ctypes.byref(b)))
    ws = torch.empty(max(int(b.value), 1), dtype=torch.uint8, device=q.device)
    perm = torch.empty(n, dtype=torch.int64, device=q.device)
    _check(load().lj_cell_order(_ptr(q), n, g, _ptr(perm), _ptr(ws), ws.numel(), _stream()))
    return perm


def permute_rows(x: torch.Tensor, perm: torch.Tensor) -> torch.Tensor:
    _rec(x, "x")
    if not (perm.is_cuda and perm.dtype == torch.int64 and perm.numel() == x.shape[0]):
        raise TypeError("permute_rows: perm must be a CUDA int64 tensor of length n")
    out = torch.empty_like(x)
    _check(load().lj_permute_rows(_ptr(x), _ptr(out), _ptr(perm.contiguous()), x.shape[0], _stream()))
    return out


# ---- force / integrate / bookkeeping / energy ---------------------------------

def _list_args(lst: CSRList):
    return (lst.row_begin, lst.row_end, _ptr(lst.number_of_partners), _ptr(lst.pointer), _ptr(lst.sorted_list))


def default_lanes(rows: int, half: bool) -> int:
    """lj_default_lanes: the lanes_per_row lj_force_step uses for this many rows."""
    return int(load().lj_default_lanes(int(rows), int(half)))


def force_step(q: torch.Tensor, p: torch.Tensor, g: Geom, dt: float, lst: CSRList, lanes_per_row: int = 0,
               ordered: bool = False, n_interactions: torch.Tensor | None = None) -> None:
    """p += impulses of one force step (in place).  PAPER.md Alg. 1 + Alg. 3."""
    _rec(q, "q")
    _rec(p, "p")
    if n_interactions is not None and not (n_interactions.is_cuda and n_interactions.dtype == torch.int64):
        raise TypeError("n_interactions must be a CUDA int64 tensor")
    _check(load().lj_force_step_ex(_ptr(q), _ptr(p), q.shape[0], g, float(dt), int(lst.half), *_list_args(lst),
                                   int(lanes_per_row), int(ordered), _ptr(n_interactions), _stream()))


class MDGraph:
    """lj_md_graph: `steps` leapfrog steps (kick, drift + displacement, device-side rebuild
    decision, conditional rebuild) as one CUDA graph.  Holds references to every buffer."""

    def __init__(self, q, p, q_alt, p_alt, q_ref, perm, g: Geom, dt: float, builder: "ListBuilder",
                 disp, counter, status, reorder: bool, steps: int, energy_every: int = 0, energies=None):
        for t, name in ((q, "q"), (p, "p"), (q_ref, "q_ref")):
            _rec(t, name)
        if not builder.padded:
            raise ValueError("MDGraph: needs the padded list layout")
        self._keep = (q, p, q_alt, p_alt, q_ref, perm, builder, disp, counter, status, energies)
        self.steps = int(steps)
        d = MDGraphDesc(_ptr(q).value, _ptr(p).value, _ptr(q_alt).value if q_alt is not None else None,
                        _ptr(p_alt).value if p_alt is not None else None, _ptr(q_ref).value, _ptr(perm).value,
                        q.shape[0], g, float(dt), _ptr(builder.npart).value, _ptr(builder.pointer).value,
                        _ptr(builder.sorted_list).value, builder.sorted_list.numel(), _ptr(builder.workspace).value,
                        builder.workspace.numel(), _ptr(disp).value, _ptr(counter).value if counter is not None
                        else None, _ptr(status).value, int(bool(reorder)), self.steps, int(energy_every),
                        _ptr(energies).value if energies is not None else None, int(builder.interleaved))
        h = ctypes.c_void_p()
        _check(load().lj_md_graph_create(ctypes.byref(d), ctypes.byref(h)))
        self._h = h

    def launch(self):
        _check(load().lj_md_graph_launch(self._h, _stream()))

    def force_ms(self) -> list[float]:
        """Per-step force-kernel durations of the last (completed) launch."""
        out = (ctypes.c_float * self.steps)()
        _check(load().lj_md_graph_force_ms(self._h, out, self.steps))
        return list(out)

    def kernels(self) -> tuple[int, int]:
        """(kernels of all unrolled steps without rebuilds, kernels per rebuild)."""
        a, b = ctypes.c_longlong(), ctypes.c_longlong()
        _check(load().lj_md_graph_kernels(self._h, ctypes.byref(a), ctypes.byref(b)))
        return a.value, b.value

    def close(self):
        if self._h is not None:
            load().lj_md_graph_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:  # noqa: BLE001 -- interpreter shutdown
            pass


def md_capture_rebuild(q: torch.Tensor, q_ref: torch.Tensor, g: Geom, builder: "ListBuilder",
                       disp: torch.Tensor, disp_count: int, disp_stride: int, status: torch.Tensor,
                       resort: dict | None = None) -> int:
    """lj_md_capture_rebuild on the current (capturing) stream: the device-side bookkeeping
    decision + an IF node whose body wraps q (q_ref = q), optionally re-sorts every atom into
    cell order (resort = dict(q_alt, p, p_alt, perm, p_peers (int64 CUDA tensor of P device
    pointers), n_own)), and rebuilds builder's own rows (padded layout).  disp: a float64
    CUDA tensor; the decision reads disp.data_ptr()[k * disp_stride] for k < disp_count.
    Returns the kernels per rebuild."""
    _rec(q, "q")
    _rec(q_ref, "q_ref")
    if not builder.padded:
        raise ValueError("md_capture_rebuild: needs the padded list layout")
    r = resort or {}
    if resort is not None:
        for name in ("q_alt", "p", "p_alt"):
            _rec(r[name], name)
        if not (r["p_peers"].is_cuda and r["p_peers"].dtype == torch.int64):
            raise TypeError("md_capture_rebuild: p_peers must be a CUDA int64 tensor of device pointers")
    d = MDRebuildDesc(_ptr(q).value, _ptr(q_ref).value, q.shape[0], g, builder.row_begin, builder.row_end,
                      _ptr(builder.npart).value, _ptr(builder.pointer).value, _ptr(builder.sorted_list).value,
                      builder.sorted_list.numel(), _ptr(builder.workspace).value, builder.workspace.numel(),
                      _ptr(disp).value, int(disp_count), int(disp_stride), _ptr(status).value,
                      int(resort is not None), _addr(r.get("q_alt")), _addr(r.get("p")), _addr(r.get("p_alt")),
                      _addr(r.get("perm")), _addr(r.get("p_peers")), int(r.get("n_own", 0)), int(builder.interleaved))
    k = ctypes.c_longlong(0)
    _check(load().lj_md_capture_rebuild(ctypes.byref(d), _stream(), ctypes.byref(k)))
    return k.value


def copy_records(src: torch.Tensor, dst: torch.Tensor) -> None:
    """lj_copy_records: dst[:] = src[:] (n AoS4 records, device, stream-ordered)."""
    _rec(src, "src")
    _rec(dst, "dst")
    if src.shape[0] != dst.shape[0]:
        raise ValueError("copy_records: shapes differ")
    _check(load().lj_copy_records(_ptr(src), _ptr(dst), src.shape[0], _stream()))


def copy_bytes(dst: torch.Tensor, src: torch.Tensor) -> None:
    """lj_copy_bytes: dst[:] = src[:] (same dtype and element count; device or pinned host
    memory on either side; stream-ordered on the current stream; capturable)."""
    if dst.dtype != src.dtype or dst.numel() != src.numel() or not (dst.is_contiguous() and src.is_contiguous()):
        raise ValueError("copy_bytes: contiguous tensors of the same dtype and size")
    for t in (dst, src):
        if not (t.is_cuda or t.is_pinned()):
            raise ValueError("copy_bytes: device or pinned host tensors")
    _check(load().lj_copy_bytes(ctypes.c_void_p(dst.data_ptr()), ctypes.c_void_p(src.data_ptr()),
                                dst.numel() * dst.element_size(), _stream()))


def permute_rows_peers(q: torch.Tensor, q_out: torch.Tensor, q_ref: torch.Tensor | None, p_out: torch.Tensor,
                       p_peers: torch.Tensor, n_own: int, own_lo: int, own_hi: int, perm: torch.Tensor, g: Geom,
                       workspace: torch.Tensor) -> None:
    """lj_permute_rows_peers: the multi-rank re-sort (q wrapped in place; perm, q_out, q_ref and
    the own new rows of p_out, their momenta read from the owner ranks' buffers p_peers)."""
    for t, name in ((q, "q"), (q_out, "q_out"), (p_out, "p_out")):
        _rec(t, name)
    if q_ref is not None:
        _rec(q_ref, "q_ref")
    if not (p_peers.is_cuda and p_peers.dtype == torch.int64):
        raise TypeError("permute_rows_peers: p_peers must be a CUDA int64 tensor of device pointers")
    _check(load().lj_permute_rows_peers(_ptr(q), _ptr(q_out), _ptr(q_ref), _ptr(p_out), _ptr(p_peers), int(n_own),
                                        int(own_lo), int(own_hi), _ptr(perm), q.shape[0], g, _ptr(workspace),
                                        workspace.numel(), _stream()))


def publish_scalar(src: torch.Tensor, dst: torch.Tensor) -> None:
    """lj_publish_scalar: dst[0] = src[0] on the device (float64 CUDA tensors/views)."""
    for t in (src, dst):
        if not (t.is_cuda and t.dtype == torch.float64):
            raise TypeError("publish_scalar: float64 CUDA tensors")
    _check(load().lj_publish_scalar(_ptr(src), _ptr(dst), _stream()))


def force_step_half_cells(q: torch.Tensor, p: torch.Tensor, g: Geom, dt: float, lst: CSRList,
                          cell_start: torch.Tensor, lanes_per_row: int = 0,
                          n_interactions: torch.Tensor | None = None) -> None:
    """Half-list force step without per-entry global atomics (lj_force_step_half_cells):
    per-cell shared-memory windows over the 27 neighbour cells, flushed once."""
    _rec(q, "q")
    _rec(p, "p")
    if not lst.half or lst.row_begin != 0 or lst.row_end != q.shape[0]:
        raise ValueError("force_step_half_cells: needs a half list over all rows")
    if not (cell_start.is_cuda and cell_start.dtype == torch.int64):
        raise TypeError("cell_start must be a CUDA int64 tensor")
    if n_interactions is not None and not (n_interactions.is_cuda and n_interactions.dtype == torch.int64):
        raise TypeError("n_interactions must be a CUDA int64 tensor")
    _check(load().lj_force_step_half_cells(_ptr(q), _ptr(p), q.shape[0], g, float(dt), _ptr(lst.number_of_partners),
                                           _ptr(lst.pointer), _ptr(lst.sorted_list), _ptr(cell_start),
                                           int(lanes_per_row), _ptr(n_interactions), _stream()))


def force_step_variant(layout: str, rcp: str, q: torch.Tensor, p: torch.Tensor | None, n: int, g: Geom,
                       dt: float, lst: CSRList, lanes_per_row: int = 4,
                       n_interactions: torch.Tensor | None = None) -> None:
    """Paper-variant ablation (lj_force_step_variant): q/p are flat float64 CUDA
    tensors in `layout` ("aos4", "soa", "aos3", "aos8"; p unused for aos8), 1/r^2
    by `rcp` ("newton3", "newton2", "approx", "ieee")."""
    for t in (q, p):
        if t is not None and not (t.is_cuda and t.dtype == torch.float64 and t.is_contiguous()):
            raise TypeError("force_step_variant: q/p must be contiguous CUDA float64 tensors")
    if lst.half:
        raise ValueError("force_step_variant: full lists only")
    _check(load().lj_force_step_variant(LAYOUTS[layout], RECIPROCALS[rcp], _ptr(q), _ptr(p), int(n), g, float(dt),
                                        *_list_args(lst), int(lanes_per_row), _ptr(n_interactions), _stream()))


def gather_probe(q: torch.Tensor, lst: CSRList, lanes_per_row: int = 0, sink: torch.Tensor | None = None) -> None:
    """Roofline probe: the force kernel's memory traffic without its arithmetic."""
    _rec(q, "q")
    if sink is None:
        sink = torch.zeros(1, dtype=torch.float64, device=q.device)
    _check(load().lj_gather_probe(_ptr(q), q.shape[0], lst.row_begin, lst.row_end, _ptr(lst.number_of_partners),
                                  _ptr(lst.pointer), _ptr(lst.sorted_list), int(lanes_per_row), _ptr(sink),
                                  _stream()))


def list_interior(lst: CSRList) -> tuple[int, int]:
    """(A, B): rows [A, B) of the list's range have all partners inside the range
    (lj_list_interior; one 16-byte readback)."""
    out = torch.empty(2, dtype=torch.int64, device=lst.pointer.device)
    _check(load().lj_list_interior(lst.row_begin, lst.row_end, _ptr(lst.number_of_partners), _ptr(lst.pointer),
                                   _ptr(lst.sorted_list), _ptr(out), _stream()))
    a, b = out.tolist()
    return int(a), int(b)


def list_partner_ranges(lst: CSRList, bounds: list[int]) -> list[tuple[int, int]]:
    """For every owner slab s = rows [bounds[s], bounds[s+1]): (min, max) partner index of the
    list's rows inside it, or None (lj_list_partner_ranges; one readback)."""
    P = len(bounds) - 1
    dev = lst.pointer.device
    b = torch.tensor(bounds, dtype=torch.int64, device=dev)
    out = torch.empty(2 * P, dtype=torch.int64, device=dev)
    _check(load().lj_list_partner_ranges(lst.row_begin, lst.row_end, _ptr(lst.number_of_partners), _ptr(lst.pointer),
                                         _ptr(lst.sorted_list), _ptr(b), P, _ptr(out), _stream()))
    v = out.tolist()
    return [None if v[2 * s + 1] < 0 else (int(v[2 * s]), int(v[2 * s + 1])) for s in range(P)]


def integrate(q: torch.Tensor, p: torch.Tensor, dt: float, begin: int = 0, end: int | None = None) -> None:
    _rec(q, "q")
    _rec(p, "p")
    _check(load().lj_integrate(_ptr(q), _ptr(p), int(begin), q.shape[0] if end is None else int(end), float(dt),
                               _stream()))


def integrate_push(q_in: torch.Tensor, q_out: torch.Tensor, p: torch.Tensor, q_ref: torch.Tensor, dt: float,
                   begin: int, end: int, out: torch.Tensor, targets: list[tuple[int, int, int]]) -> None:
    """lj_integrate_push: q_out = q_in + p dt on rows [begin, end), out = max |q_out - q_ref| there,
    and each updated row also stored into the targets (dst device pointer, lo, hi) whose [lo, hi)
    holds it -- the drift and the position exchange in one kernel."""
    for t, name in ((q_in, "q_in"), (q_out, "q_out"), (p, "p"), (q_ref, "q_ref")):
        _rec(t, name)
    if not (out.is_cuda and out.dtype == torch.float64 and out.numel() >= 1):
        raise TypeError("integrate_push: out must be a CUDA float64 tensor")
    arr = (PushTarget * max(len(targets), 1))(*[PushTarget(int(d), int(lo), int(hi)) for d, lo, hi in targets])
    _check(load().lj_integrate_push(_ptr(q_in), _ptr(q_out), _ptr(p), _ptr(q_ref), int(begin), int(end), float(dt),
                                    _ptr(out), arr, len(targets), _stream()))


def ipc_handle(t: torch.Tensor) -> tuple[bytes, int]:
    """(64-byte CUDA IPC handle of the allocation holding t, t's byte offset in it)."""
    h = ctypes.create_string_buffer(64)
    off = ctypes.c_int64()
    _check(load().lj_ipc_get_handle(_ptr(t), h, ctypes.byref(off)))
    return h.raw, int(off.value)


def ipc_open(handle: bytes, offset: int) -> int:
    """Map another process's allocation (lj_ipc_open); returns the device pointer at offset."""
    if len(handle) != 64:
        raise ValueError("ipc_open: need a 64-byte handle")
    ptr = ctypes.c_void_p()
    _check(load().lj_ipc_open(handle, int(offset), ctypes.byref(ptr)))
    return int(ptr.value)


def ipc_close(ptr: int) -> None:
    _check(load().lj_ipc_close(ctypes.c_void_p(ptr)))


def integrate_displacement(q: torch.Tensor, p: torch.Tensor, q_ref: torch.Tensor, dt: float, begin: int, end: int,
                           out: torch.Tensor) -> None:
    """q += p dt on rows [begin, end) and out = max |q - q_ref| there, in one pass."""
    _rec(q, "q")
    _rec(p, "p")
    _rec(q_ref, "q_ref")
    _check(load().lj_integrate_displacement(_ptr(q), _ptr(p), _ptr(q_ref), int(begin), int(end), float(dt), _ptr(out),
                                            _stream()))


def wrap(q: torch.Tensor, L: float, q_ref: torch.Tensor | None = None) -> None:
    _rec(q, "q")
    if q_ref is not None:
        _rec(q_ref, "q_ref")
    _check(load().lj_wrap(_ptr(q), _ptr(q_ref), q.shape[0], float(L), _stream()))


def max_displacement(q: torch.Tensor, q_ref: torch.Tensor, begin: int = 0, end: int | None = None,
                     out: torch.Tensor | None = None) -> torch.Tensor:
    _rec(q, "q")
    _rec(q_ref, "q_ref")
    if out is None:
        out = torch.empty(1, dtype=torch.float64, device=q.device)
    _check(load().lj_max_displacement(_ptr(q), _ptr(q_ref), int(begin), q.shape[0] if end is None else int(end),
                                      _ptr(out), _stream()))
    return out


def energy(q: torch.Tensor, p: torch.Tensor, g: Geom, lst: CSRList, out: torch.Tensor | None = None) -> torch.Tensor:
    """{KE over own rows, PE over the list's entries inside r_c} as a device (2,) tensor."""
    _rec(q, "q")
    _rec(p, "p")
    if out is None:
        out = torch.empty(2, dtype=torch.float64, device=q.device)
    rb, re_, npp, ptr, sl = _list_args(lst)
    _check(load().lj_energy(_ptr(q), _ptr(p), q.shape[0], g, rb, re_, npp, ptr, sl, int(lst.half), _ptr(out),
                            _stream()))
    return out
