"""B-15 roofline denominators, measured on the box, written as one
JSON document (profiles/r02_b15.json) that bench.py's roofline cites:

  * fp64_fma        -- FP64 pipe issue rate (independent DFMA chains);
  * random_gather   -- uniform random 32-B record gathers (hash-indexed, no index
                       stream) over 3.8 / 65.5 / 524 MB arrays (configs 2-3 / 4 / 5 q);
  * random_red      -- fp64 REDs (3 per record = the half list's 24-B p_j RMW,
                       PAPER.md:176-181) to random records of 3.8 / 65.5 MB arrays;
  * half_red_replay -- the half list's exact RED pattern (3 REDs per entry + 3 per
                       row, no gathers, no arithmetic) on configs 2 and 3;
  * gather_replay   -- lj_gather_probe, the force kernel's access pattern without
                       arithmetic, for every lanes/unroll/index-vector variant on the
                       bench's padded config-4 list (cell order) and configs 2/3; the
                       minimum is the "best same-list replay" the force kernel is
                       measured against;
  * force           -- lj_force_step for the same variants (same list), for the table.

    python tools/roofline_b15.py [out.json]
"""
import ctypes
import json
import os
import sys
import time

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tools"))
import lj_inputs  # noqa: E402
from microbench import build, timeit  # noqa: E402
from paper_1806_05713_b200 import lj  # noqa: E402

VARIANTS = ([(G, U, 0) for G, U in ((2, 2), (2, 3), (4, 2), (4, 3), (4, 4), (8, 2), (8, 3), (8, 4), (16, 2), (16, 3))]
            + [(G, V, lj.LJ_LANES_IDXV) for G in (2, 4, 8) for V in (2, 4)] + [(16, 4, lj.LJ_LANES_IDXV)])


def main():
    out_path = sys.argv[1] if len(sys.argv) > 1 else os.path.join(ROOT, "profiles", "r02_b15.json")
    M = build()
    vp, i64, ci = ctypes.c_void_p, ctypes.c_int64, ctypes.c_int
    M.mb_fp64_fma.argtypes = [vp, ci, ci, ci, vp]
    M.mb_random_gather.argtypes = [vp, i64, ci, ci, ci, vp, vp]
    M.mb_random_red.argtypes = [vp, i64, ci, ci, ci, vp]
    M.mb_half_red_replay.argtypes = [vp, i64, vp, vp, vp, ci, vp]
    dev = torch.device("cuda:0")
    st = vp(torch.cuda.current_stream().cuda_stream)
    sink = torch.zeros(4, dtype=torch.float64, device=dev)
    doc = {"what": "B-15 roofline microbenchmarks (SURVEY §8(d)); CUDA-event times, warm, best of repeats",
           "device": torch.cuda.get_device_name(0), "when": time.strftime("%Y-%m-%dT%H:%M:%SZ", time.gmtime())}

    blocks, threads, iters = 148 * 8, 256, 2000
    ms = min(timeit(lambda: M.mb_fp64_fma(vp(sink.data_ptr()), blocks, threads, iters, st)) for _ in range(3))
    fmas = blocks * threads * iters * 16 * 8
    doc["fp64_fma"] = {"ms": ms, "T_dfma_per_s": fmas / ms / 1e9, "TFLOP_s": 2 * fmas / ms / 1e9}
    print(json.dumps(doc["fp64_fma"]), flush=True)

    doc["random_gather"] = []
    for label, n in (("3.8 MB (119,164 records, configs 2-3)", 119164), ("65.5 MB (2,048,000, config 4)", 2048000),
                     ("524 MB (16,384,000, config 5)", 16384000)):
        q = torch.rand((n, 4), dtype=torch.float64, device=dev)
        gb, gt, gi = 148 * 16, 256, 32
        ms = min(timeit(lambda: M.mb_random_gather(vp(q.data_ptr()), n, gb, gt, gi, vp(sink.data_ptr()), st))
                 for _ in range(3))
        ng = gb * gt * gi * 8
        r = {"array": label, "records": n, "ms": ms, "G_gathers_per_s": ng / ms / 1e6, "GB_s_32B": 32 * ng / ms / 1e6}
        doc["random_gather"].append(r)
        print(json.dumps(r), flush=True)
        del q

    doc["random_red"] = []
    for label, n in (("3.8 MB (119,164 records)", 119164), ("65.5 MB (2,048,000)", 2048000)):
        p = torch.zeros((n, 4), dtype=torch.float64, device=dev)
        rb, rt, ri = 148 * 16, 256, 8
        ms = min(timeit(lambda: M.mb_random_red(vp(p.data_ptr()), n, rb, rt, ri, st)) for _ in range(3))
        nrec = rb * rt * ri * 4
        r = {"array": label, "records": n, "ms": ms, "G_red_f64_per_s": 3 * nrec / ms / 1e6,
             "G_records_rmw_per_s": nrec / ms / 1e6, "GB_s_24B_rmw": 24 * nrec / ms / 1e6}
        doc["random_red"].append(r)
        print(json.dumps(r), flush=True)
        del p

    doc["half_red_replay"] = []
    doc["gather_replay"] = []
    doc["force"] = []
    for cfg in (2, 3, 4):
        w = lj_inputs.config(cfg)
        g = lj.geom(w.L, w.rc, w.rs)
        q = lj.pack_aos4(torch.from_numpy(w.q).to(dev))
        if cfg in (3, 4):
            q = lj.permute_rows(q, lj.cell_order(q, g))
        p = lj.pack_aos4(torch.from_numpy(w.p).to(dev))
        if cfg in (2, 3):
            half = lj.build_list(q, g, True)
            pr = torch.zeros((w.n, 4), dtype=torch.float64, device=dev)
            for G in (4, 8):
                ms = min(timeit(lambda: M.mb_half_red_replay(vp(pr.data_ptr()), w.n, vp(half.number_of_partners.data_ptr()),
                                                             vp(half.pointer.data_ptr()), vp(half.sorted_list.data_ptr()),
                                                             G, st)) for _ in range(3))
                E = half.n_entries
                r = {"cfg": cfg, "G": G, "entries": E, "ms": ms, "G_entries_per_s": E / ms / 1e6,
                     "G_red_f64_per_s": 3 * (E + w.n) / ms / 1e6}
                doc["half_red_replay"].append(r)
                print(json.dumps(r), flush=True)
            del half, pr
        for il in (False, True):   # the row-major padded list and the interleaved one (the MD driver's)
          lst = lj.ListBuilder(w.n, g, False, device=dev, padded=True, interleaved=il).build(q)
          E = lst.n_entries
          for G, U, X in VARIANTS:
            lanes = G | (U << 8) | X
            rec = {"cfg": cfg, "order": "cell" if cfg in (3, 4) else "shuffled",
                   "list": "full, padded" + (", interleaved" if il else ""),
                   "G": G, "U": U, "idxv": bool(X), "lanes_per_row": lanes, "entries": E}
            try:
                rec["probe_ms"] = min(timeit(lambda: lj.gather_probe(q, lst, lanes, sink), reps=20)
                                      for _ in range(3))
            except lj.LJError:
                rec["probe_ms"] = None
            try:
                pc = p.clone()
                rec["force_ms"] = min(timeit(lambda: lj.force_step(q, pc, g, w.dt, lst, lanes_per_row=lanes), reps=20)
                                      for _ in range(3))
            except lj.LJError:
                rec["force_ms"] = None
            doc["gather_replay"].append(rec)
            print(json.dumps(rec), flush=True)
          del lst
        del q, p
        torch.cuda.empty_cache()

    best = {}
    for r in doc["gather_replay"]:
        k = (r["cfg"], r["list"])
        if r["probe_ms"] is not None and (k not in best or r["probe_ms"] < best[k]["probe_ms"]):
            best[k] = r
    doc["best_replay"] = {f"{k[0]} ({k[1]})": {"probe_ms": v["probe_ms"], "lanes_per_row": v["lanes_per_row"],
                                               "G": v["G"], "U": v["U"], "idxv": v["idxv"], "entries": v["entries"]}
                          for k, v in best.items()}
    with open(out_path, "w") as f:
        json.dump(doc, f, indent=1)
    print("wrote", out_path, flush=True)


if __name__ == "__main__":
    main()
