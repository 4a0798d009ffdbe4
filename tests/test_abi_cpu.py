"""CPU-side checks of the C-ABI library (no GPU): it loads, exports every symbol
include/liblj.h declares, and rejects bad arguments before launching anything."""
import ctypes
import re
import os

import pytest

from paper_1806_05713_b200 import build, lj

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def L():
    build.build()
    return lj.load()


def declared_symbols():
    src = open(os.path.join(ROOT, "include", "liblj.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(lj_[a-z0-9_]+)\s*\(", src)))


def test_header_declares_the_binding_exports():
    assert declared_symbols() == sorted(lj.EXPORTS)


def test_library_exports_every_declared_symbol(L):
    for name in declared_symbols():
        assert hasattr(L, name), name
    out = os.popen(f"nm -D --defined-only {lj.LIB_PATH}").read()
    for name in declared_symbols():
        assert re.search(rf"\bT {name}\b", out), f"{name} not exported as a text symbol"


def test_library_is_sm100a(L):
    out = os.popen(f"/usr/local/cuda/bin/cuobjdump --list-elf {lj.LIB_PATH}").read()
    assert "sm_100a" in out


def test_version_and_counters(L):
    assert b"sm_100a" in L.lj_version()
    assert L.lj_launch_count() >= 0
    assert L.lj_status_string(2) == b"LJ_ERR_CAPACITY"


def test_validation_before_launch(L):
    g_bad = lj.Geom(10.0, 3.3, 3.0)          # rc > rs
    size = ctypes.c_size_t()
    assert L.lj_build_list_workspace(100, g_bad, ctypes.byref(size)) == lj.LJ_ERR_ARG
    assert b"rc" in L.lj_last_error()
    g_small = lj.Geom(9.0, 3.0, 3.3)         # floor(9/3.3) = 2 < 3 cells
    assert L.lj_build_list_workspace(100, g_small, ctypes.byref(size)) == lj.LJ_ERR_ARG
    g_open = lj.Geom(0.0, 3.0, 3.3)          # list build needs a box
    assert L.lj_build_list_workspace(100, g_open, ctypes.byref(size)) == lj.LJ_ERR_UNSUPPORTED
    g = lj.Geom(15.874011, 3.0, 3.3)
    assert L.lj_build_list_workspace(4000, g, ctypes.byref(size)) == lj.LJ_OK and size.value > 4000 * 40
    assert L.lj_build_list_workspace(-1, g, ctypes.byref(size)) == lj.LJ_ERR_ARG
    assert L.lj_build_list_workspace(2 ** 31, g, ctypes.byref(size)) == lj.LJ_ERR_ARG
    # half list with a partial row range
    ne = ctypes.c_int64()
    st = L.lj_build_list(ctypes.c_void_p(256), 4000, g, 1, 0, 10, ctypes.c_void_p(256), ctypes.c_void_p(256), None, 0,
                         ctypes.byref(ne), ctypes.c_void_p(256), 1 << 30, None)
    assert st == lj.LJ_ERR_UNSUPPORTED
    # bad row range / misaligned records / non-finite dt
    st = L.lj_force_step(ctypes.c_void_p(256), ctypes.c_void_p(256), 10, g, 0.01, 0, 5, 3, None, None, None, None)
    assert st == lj.LJ_ERR_ARG
    st = L.lj_integrate(ctypes.c_void_p(264), ctypes.c_void_p(256), 0, 10, 0.1, None)
    assert st == lj.LJ_ERR_ARG and b"aligned" in L.lj_last_error()
    st = L.lj_integrate(ctypes.c_void_p(256), ctypes.c_void_p(256), 0, 10, float("nan"), None)
    assert st == lj.LJ_ERR_ARG
    st = L.lj_force_step_ex(ctypes.c_void_p(256), ctypes.c_void_p(256), 10, g, 0.01, 0, 0, 10, ctypes.c_void_p(256),
                            ctypes.c_void_p(256), ctypes.c_void_p(256), 3, 0, None, None)
    assert st == lj.LJ_ERR_ARG and b"lanes" in L.lj_last_error()
    st = L.lj_force_step_ex(ctypes.c_void_p(256), ctypes.c_void_p(256), 10, g, 0.01, 1, 0, 10, ctypes.c_void_p(256),
                            ctypes.c_void_p(256), ctypes.c_void_p(256), 0, 1, None, None)
    assert st == lj.LJ_ERR_UNSUPPORTED
    assert L.lj_wrap(None, None, 0, 0.0, None) == lj.LJ_ERR_ARG
    # LJ_LIST_INTERLEAVED needs the padded layout; its capacity is counted in blocks of 8 rows
    ws = ctypes.c_size_t()
    assert L.lj_build_list_workspace(4000, g, ctypes.byref(ws)) == lj.LJ_OK
    st = L.lj_build_list_ex(ctypes.c_void_p(256), 4000, g, 0, 0, 4000, lj.LJ_LIST_INTERLEAVED, ctypes.c_void_p(256), ctypes.c_void_p(256),
                            ctypes.c_void_p(256), 1 << 30, ctypes.byref(ne), ctypes.c_void_p(256), ws.value, None)
    assert st == lj.LJ_ERR_ARG and b"PADDED" in L.lj_last_error()
    st = L.lj_build_list_ex(ctypes.c_void_p(256), 4000, g, 0, 0, 3999, lj.LJ_LIST_PADDED | lj.LJ_LIST_INTERLEAVED,
                            ctypes.c_void_p(256), ctypes.c_void_p(256), ctypes.c_void_p(256), 3999 * 196,
                            ctypes.byref(ne), ctypes.c_void_p(256), ws.value, None)
    assert st == lj.LJ_ERR_CAPACITY and ne.value == 4000 * 196   # 3,999 rows -> 500 blocks of 8
    st = L.lj_build_list_ex(ctypes.c_void_p(256), 4000, g, 0, 0, 3999, 8, ctypes.c_void_p(256),
                            ctypes.c_void_p(256), ctypes.c_void_p(256), 1 << 30, ctypes.byref(ne),
                            ctypes.c_void_p(256), ws.value, None)
    assert st == lj.LJ_ERR_ARG and b"flags" in L.lj_last_error()
    # lj_copy_bytes: null pointers with a non-zero size; zero bytes is a no-op
    assert L.lj_copy_bytes(None, ctypes.c_void_p(256), 8, None) == lj.LJ_ERR_ARG
    assert L.lj_copy_bytes(None, None, 0, None) == lj.LJ_OK


def test_validation_of_the_step_entry_points(L):
    """Host-side argument checks of lj_rebuild, the ablation / probe / overlap /
    halo entry points: all return before any device work, so they run here."""
    g = lj.Geom(15.874011, 3.0, 3.3)
    a, b, c, d = (ctypes.c_void_p(256 * k) for k in (1, 2, 3, 4))
    ne = ctypes.c_int64()
    # rebuild: q_out aliasing q, then p without p_out
    st = L.lj_rebuild(a, b, a, c, None, d, 100, g, 0, 0, 100, 0, a, b, c, 1 << 20, ctypes.byref(ne), d, 1 << 20,
                      None)
    assert st == lj.LJ_ERR_ARG and b"distinct" in L.lj_last_error()
    st = L.lj_rebuild(a, b, c, None, None, d, 100, g, 0, 0, 100, 0, a, b, c, 1 << 20, ctypes.byref(ne), d, 1 << 20,
                      None)
    assert st == lj.LJ_ERR_ARG
    # variant: layout / reciprocal / lanes out of range
    for layout, rcp, lanes, word in ((4, 0, 4, b"layout"), (0, 4, 4, b"reciprocal"), (0, 0, 2, b"lanes")):
        st = L.lj_force_step_variant(layout, rcp, a, b, 10, g, 0.01, 0, 10, a, b, c, lanes, None, None)
        assert st == lj.LJ_ERR_ARG and word in L.lj_last_error()
    # probe: misaligned q, unsupported G|U
    st = L.lj_gather_probe(ctypes.c_void_p(264), 10, 0, 10, a, b, c, 0, d, None)
    assert st == lj.LJ_ERR_ARG and b"aligned" in L.lj_last_error()
    st = L.lj_gather_probe(a, 10, 0, 10, a, b, c, 32 | (2 << 8), d, None)
    assert st == lj.LJ_ERR_ARG and b"lanes" in L.lj_last_error()
    # interior / partner ranges: bad ranges, P out of [1, 64], null pointers
    assert L.lj_list_interior(5, 4, a, b, c, d, None) == lj.LJ_ERR_ARG
    assert L.lj_list_interior(0, 4, None, b, c, d, None) == lj.LJ_ERR_ARG
    for P in (0, 65):
        st = L.lj_list_partner_ranges(0, 4, a, b, c, d, P, a, None)
        assert st == lj.LJ_ERR_ARG and b"P" in L.lj_last_error()
    assert L.lj_list_partner_ranges(0, 4, a, b, c, None, 2, a, None) == lj.LJ_ERR_ARG
    # fused drift + displacement: null max_disp, misaligned q_ref, nan dt, bad range
    assert L.lj_integrate_displacement(a, b, c, 0, 10, 0.01, None, None) == lj.LJ_ERR_ARG
    st = L.lj_integrate_displacement(a, b, ctypes.c_void_p(264), 0, 10, 0.01, d, None)
    assert st == lj.LJ_ERR_ARG and b"aligned" in L.lj_last_error()
    assert L.lj_integrate_displacement(a, b, c, 0, 10, float("inf"), d, None) == lj.LJ_ERR_ARG
    assert L.lj_integrate_displacement(a, b, c, 10, 0, 0.01, d, None) == lj.LJ_ERR_ARG
    # fused drift + push: target count, target rows / alignment, null max_disp
    T = (lj.PushTarget * 2)(lj.PushTarget(512, 0, 10), lj.PushTarget(264, 0, 10))
    assert L.lj_integrate_push(a, b, c, d, 0, 10, 0.01, a, T, 64, None) == lj.LJ_ERR_ARG
    assert L.lj_integrate_push(a, b, c, d, 0, 10, 0.01, a, None, 1, None) == lj.LJ_ERR_ARG
    st = L.lj_integrate_push(a, b, c, d, 0, 10, 0.01, a, T, 2, None)
    assert st == lj.LJ_ERR_ARG and b"target 1" in L.lj_last_error()
    T[1] = lj.PushTarget(768, 5, 4)
    st = L.lj_integrate_push(a, b, c, d, 0, 10, 0.01, a, T, 2, None)
    assert st == lj.LJ_ERR_ARG and b"bad rows" in L.lj_last_error()
    assert L.lj_integrate_push(a, b, c, d, 0, 10, 0.01, None, T, 1, None) == lj.LJ_ERR_ARG
    # IPC: argument checks only (a real handle needs a device)
    assert L.lj_ipc_get_handle(None, ctypes.create_string_buffer(64), ctypes.byref(ne)) == lj.LJ_ERR_ARG
    assert L.lj_ipc_open(None, 0, ctypes.byref(ctypes.c_void_p())) == lj.LJ_ERR_ARG
    assert L.lj_ipc_open(b"\0" * 64, -1, ctypes.byref(ctypes.c_void_p())) == lj.LJ_ERR_ARG
    assert L.lj_ipc_close(None) == lj.LJ_ERR_ARG
    # NEXT-3 entry points: null workspace / cell starts, unsupported lanes, open box
    assert L.lj_list_cell_starts(None, 0, 100, g, a, None) == lj.LJ_ERR_ARG
    assert L.lj_list_cell_starts(a, 16, 100, g, a, None) == lj.LJ_ERR_ARG   # workspace too small
    st = L.lj_force_step_half_cells(a, b, 10, g, 0.01, a, b, c, d, 16 | 512, None, None)
    assert st == lj.LJ_ERR_ARG and b"lanes" in L.lj_last_error()
    assert L.lj_force_step_half_cells(a, b, 10, g, 0.01, a, b, c, None, 0, None, None) == lj.LJ_ERR_ARG
    assert L.lj_force_step_half_cells(a, b, 10, lj.Geom(0.0, 3.0, 3.3), 0.01, a, b, c, d, 0, None,
                                      None) != lj.LJ_OK
    # LJ_LIST_DEFERRED needs the padded layout; unknown flags
    for fl in (lj.LJ_LIST_DEFERRED, 8):
        st = L.lj_build_list_ex(a, 100, g, 0, 0, 100, fl, a, b, c, 1 << 20, ctypes.byref(ne), d, 1 << 30, None)
        assert st == lj.LJ_ERR_ARG
    # lj_md_graph: descriptor checks before any CUDA call
    h = ctypes.c_void_p()
    assert L.lj_md_graph_create(None, ctypes.byref(h)) == lj.LJ_ERR_ARG
    dsc = lj.MDGraphDesc(256, 512, 768, 1024, 1280, 1536, 100, g, 0.01, 256, 512, 768, 100 * 196, 1024, 1 << 30,
                         256, None, 512, 1, 0)
    st = L.lj_md_graph_create(ctypes.byref(dsc), ctypes.byref(h))
    assert st == lj.LJ_ERR_ARG and b"steps" in L.lj_last_error()
    dsc.steps = 5
    dsc.capacity = 100
    assert L.lj_md_graph_create(ctypes.byref(dsc), ctypes.byref(h)) == lj.LJ_ERR_CAPACITY
    dsc.capacity = 100 * 196
    dsc.q_alt = None
    assert L.lj_md_graph_create(ctypes.byref(dsc), ctypes.byref(h)) == lj.LJ_ERR_ARG   # reorder needs q_alt
    assert L.lj_md_graph_launch(None, None) == lj.LJ_ERR_ARG
    assert L.lj_md_graph_destroy(None) == lj.LJ_OK
    # nothing above reached the device
    assert L.lj_launch_count() == 0


def test_product_binding_has_no_cpu_fallback():
    """The product package never imports the oracle or a CPU path."""
    pkg = os.path.join(ROOT, "paper_1806_05713_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith(".py"):
                src = open(os.path.join(dirpath, f)).read()
                assert "import oracle" not in src and "from oracle" not in src, f


def test_bounds_checked_build_has_the_checks():
    """liblj_check.so (-DLJ_CHECK, the memory-safety build run by tests/test_gpu_checked.py)
    carries device-side traps in the force, energy and list kernels; liblj.so has none."""
    import shutil
    import subprocess
    from paper_1806_05713_b200 import build
    if shutil.which("cuobjdump") is None and not os.path.exists("/usr/local/cuda/bin/cuobjdump"):
        pytest.skip("cuobjdump not available")
    tool = shutil.which("cuobjdump") or "/usr/local/cuda/bin/cuobjdump"
    lib, chk = build.build(), build.build(check=True)

    def traps(path):
        out = subprocess.run([tool, "-sass", path], capture_output=True, text=True).stdout
        fn, hits = None, {}
        for line in out.splitlines():
            if "Function :" in line:
                fn = line.split("Function :")[1].strip()
            elif "BPT.TRAP" in line and fn:
                hits[fn] = hits.get(fn, 0) + 1
        return hits

    assert not traps(lib)
    hits = traps(chk)
    for kernel in ("k_force", "k_energy", "k_list_v4", "k_list_fallback", "k_force_ordered"):
        assert any(kernel in f for f in hits), kernel
