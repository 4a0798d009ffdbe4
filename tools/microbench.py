"""Roofline denominators measured on the box (SURVEY B-15): FP64 DFMA rate,
gather-only replay of the real CSR list (config 4 lattice and config 3 cell
order), HBM stream of the index array.  Prints JSON lines."""
import ctypes
import json
import os
import subprocess
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import lj_inputs  # noqa: E402
from paper_1806_05713_b200 import lj  # noqa: E402

SRC = os.path.join(ROOT, "tools", "microbench.cu")
LIB = os.path.join(ROOT, "tools", "libljmicro.so")


def build():
    if not os.path.exists(LIB) or os.path.getmtime(LIB) < os.path.getmtime(SRC):
        subprocess.check_call(["/usr/local/cuda/bin/nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-O3",
                               "-lineinfo", "-shared", "-Xcompiler", "-fPIC", "-o", LIB, SRC])
    return ctypes.CDLL(LIB)


def timeit(fn, reps=10, warm=2):
    for _ in range(warm):
        fn()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    s.record()
    for _ in range(reps):
        fn()
    e.record()
    torch.cuda.synchronize()
    return s.elapsed_time(e) / reps


def main():
    M = build()
    vp = ctypes.c_void_p
    M.mb_fp64_fma.argtypes = [vp, ctypes.c_int, ctypes.c_int, ctypes.c_int, vp]
    M.mb_gather.argtypes = [vp, ctypes.c_int64, vp, vp, vp, vp, ctypes.c_int, vp]
    M.mb_stream.argtypes = [vp, ctypes.c_int64, vp, vp]
    M.mb_gather_smem.argtypes = [vp, ctypes.c_int64, vp, vp, vp, vp, ctypes.c_int, ctypes.c_int, vp]
    M.mb_gather_vec.argtypes = [vp, ctypes.c_int64, vp, vp, vp, vp, ctypes.c_int, vp]
    which = sys.argv[1].split(",") if len(sys.argv) > 1 else ["fma", "4", "4c", "3"]
    dev = torch.device("cuda:0")
    st = vp(torch.cuda.current_stream().cuda_stream)
    out = torch.zeros(4, dtype=torch.float64, device=dev)
    # FP64 FMA: blocks x threads x iters x 16 x 8 FMAs
    blocks, threads, iters = 148 * 8, 256, 2000
    if "fma" in which:
        ms = timeit(lambda: M.mb_fp64_fma(vp(out.data_ptr()), blocks, threads, iters, st))
        fmas = blocks * threads * iters * 16 * 8
        print(json.dumps({"what": "fp64_fma", "ms": ms, "TFMA_s": fmas / ms / 1e9,
                          "TFLOP_s": 2 * fmas / ms / 1e9}), flush=True)
    for cname in [x for x in which if x != "fma"]:
        c = int(cname[0])
        w = lj_inputs.config(c)
        g = lj.geom(w.L, w.rc, w.rs)
        q = lj.pack_aos4(torch.from_numpy(w.q).to(dev))
        if c == 3 or cname.endswith("c"):
            q = lj.permute_rows(q, lj.cell_order(q, g))
        lst = lj.build_list(q, g, False)
        E = lst.n_entries
        for G in (1, 2, 4, 8, 16):
            ms = timeit(lambda: M.mb_gather(vp(q.data_ptr()), lst.rows, vp(lst.number_of_partners.data_ptr()),
                                            vp(lst.pointer.data_ptr()), vp(lst.sorted_list.data_ptr()),
                                            vp(out.data_ptr()), G, st))
            print(json.dumps({"what": "gather_replay", "cfg": cname, "G": G, "ms": ms, "G_entries_s": E / ms / 1e6,
                              "gather_GBs_32B": 32 * E / ms / 1e6, "index_GBs": 4 * E / ms / 1e6}), flush=True)
        args = (vp(q.data_ptr()), lst.rows, vp(lst.number_of_partners.data_ptr()), vp(lst.pointer.data_ptr()),
                vp(lst.sorted_list.data_ptr()), vp(out.data_ptr()))
        for R in (64, 128):
            ms = timeit(lambda: M.mb_gather_smem(*args, R, 14000 if R == 64 else 26000, st))
            print(json.dumps({"what": "gather_smem_g1", "cfg": cname, "rows_per_cta": R, "ms": ms,
                              "G_entries_s": E / ms / 1e6}), flush=True)
        for G in (1, 2, 4, 8):
            ms = timeit(lambda: M.mb_gather_vec(*args, G, st))
            print(json.dumps({"what": "gather_vec_int4", "cfg": cname, "G": G, "ms": ms,
                              "G_entries_s": E / ms / 1e6}), flush=True)
        ms = timeit(lambda: M.mb_stream(vp(lst.sorted_list.data_ptr()), 4 * E, vp(out.data_ptr()), st))
        print(json.dumps({"what": "stream_list", "cfg": cname, "ms": ms, "GBs": 4 * E / ms / 1e6}), flush=True)
        del q, lst
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
