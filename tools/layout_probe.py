"""Index-stream layout probe (development tool): does the row-major padded index
stream cost L1 wavefronts the force kernel could save?  On the bench's config-4
padded list (cell order), per (G, U): the gather replay with the row-major list
(the force kernel's layout), the same with a warp-tiled copy of the list (every
warp index load one coalesced 128-B line), and both with the index loads only.

    python tools/layout_probe.py [cfg]
"""
import ctypes
import json
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tools"))
import lj_inputs  # noqa: E402
from microbench import build, timeit  # noqa: E402
from paper_1806_05713_b200 import lj  # noqa: E402


def main():
    cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 4
    M = build()
    vp, i64, ci = ctypes.c_void_p, ctypes.c_int64, ctypes.c_int
    M.mb_tile_list.argtypes = [vp, vp, ci, i64, ci, vp, ci, ci, vp]
    M.mb_probe_layout.argtypes = [vp, i64, vp, vp, ci, vp, ci, vp, ci, ci, ci, vp]
    dev = torch.device("cuda:0")
    st = vp(torch.cuda.current_stream().cuda_stream)
    w = lj_inputs.config(cfg)
    g = lj.geom(w.L, w.rc, w.rs)
    q = lj.pack_aos4(torch.from_numpy(w.q).to(dev))
    q = lj.permute_rows(q, lj.cell_order(q, g))
    p = lj.pack_aos4(torch.from_numpy(w.p).to(dev))
    lst = lj.ListBuilder(w.n, g, False, device=dev, padded=True).build(q)
    stride = int(lst.pointer[1].item() - lst.pointer[0].item())
    assert int(lst.pointer[-1].item()) == stride * w.n
    sink = torch.zeros(4, dtype=torch.float64, device=dev)
    npart, slist = lst.number_of_partners, lst.sorted_list
    for G, U in ((4, 3), (4, 2), (8, 2), (8, 3), (16, 2)):
        C = -(-stride // (U * G))
        warps = -(-w.n * G // 32)
        tiled = torch.empty(warps * C * U * 32, dtype=torch.int32, device=dev)
        assert M.mb_tile_list(vp(npart.data_ptr()), vp(slist.data_ptr()), stride, w.n, C, vp(tiled.data_ptr()),
                              G, U, st) == 0
        rec = {"cfg": cfg, "G": G, "U": U, "entries": lst.n_entries, "stride": stride, "C": C}
        for mode, name in ((0, "rows_gather"), (1, "rows_index_only"), (2, "tiled_gather"), (3, "tiled_index_only")):
            def run():
                assert M.mb_probe_layout(vp(q.data_ptr()), w.n, vp(npart.data_ptr()), vp(slist.data_ptr()), stride,
                                         vp(tiled.data_ptr()), C, vp(sink.data_ptr()), G, U, mode, st) == 0
            rec[name + "_ms"] = round(min(timeit(run, reps=20) for _ in range(3)), 4)
        rec["lj_gather_probe_ms"] = round(min(timeit(lambda: lj.gather_probe(q, lst, G | (U << 8), sink), reps=20)
                                              for _ in range(3)), 4)
        pc = p.clone()
        rec["force_ms"] = round(min(timeit(lambda: lj.force_step(q, pc, g, w.dt, lst, lanes_per_row=G | (U << 8)),
                                           reps=20) for _ in range(3)), 4)
        print(json.dumps(rec), flush=True)
        del tiled


if __name__ == "__main__":
    main()
