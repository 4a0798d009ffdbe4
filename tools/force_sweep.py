"""Kernel-variant sweep on one GPU: list-build time and force-step time per
lanes_per_row for configs 2 (shuffled), 3 (cell order) and 4 (lattice, 2.048M).
Prints one JSON object per measurement.  Development tool, not the bench."""
import json
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import lj_inputs  # noqa: E402
from paper_1806_05713_b200 import lj  # noqa: E402


def timeit(fn, reps=20, warm=3):
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
    dev = torch.device("cuda:0")
    cfgs = sys.argv[1].split(",") if len(sys.argv) > 1 else ["2", "3", "4", "4c"]
    for cname in cfgs:
        c = int(cname[0])
        w = lj_inputs.config(c)
        g = lj.geom(w.L, w.rc, w.rs)
        q = lj.pack_aos4(torch.from_numpy(w.q).to(dev))
        if c == 3 or cname.endswith("c"):
            perm = lj.cell_order(q, g)
            q = lj.permute_rows(q, perm)
        p = lj.pack_aos4(torch.from_numpy(w.p).to(dev))
        for half in ([True, False] if c != 4 else [False]):
            b = lj.ListBuilder(w.n, g, half, device=dev)
            lst = b.build(q)
            t_build = timeit(lambda: b.build(q), reps=5, warm=1)
            cnt = torch.zeros(1, dtype=torch.int64, device=dev)
            lj.force_step(q, p, g, w.dt, lst, n_interactions=cnt)
            inter = int(cnt.item())
            pairs = inter if half else inter // 2
            print(json.dumps(dict(cfg=cname, half=half, what="build", ms=round(t_build, 4), entries=lst.n_entries)),
                  flush=True)
            for lanes in (4, 8, 4 | 1024, 8 | 1024, 16 | 1024):
                ms = timeit(lambda: lj.force_step(q, p, g, w.dt, lst, lanes_per_row=lanes))
                print(json.dumps(dict(cfg=cname, half=half, what="force", lanes=lanes, ms=round(ms, 4),
                                      G_entries_s=round(lst.n_entries / ms / 1e6, 2),
                                      G_pairs_s=round(pairs / ms / 1e6, 2))), flush=True)
            if not half:
                ms = timeit(lambda: lj.force_step(q, p, g, w.dt, lst, ordered=True), reps=5)
                print(json.dumps(dict(cfg=cname, half=half, what="force_ordered", ms=round(ms, 4))), flush=True)
        del q, p
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
