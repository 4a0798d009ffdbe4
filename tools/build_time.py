"""List-build timing on one GPU (development tool): compact and padded layouts
(lj_build_list_ex) and the padded lj_rebuild,
configs 3 (cell order) and 4 (cell order).  One JSON object per measurement."""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import lj_inputs  # noqa: E402
from paper_1806_05713_b200 import lj  # noqa: E402


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
    dev = torch.device("cuda:0")
    for c in [int(x) for x in (sys.argv[1] if len(sys.argv) > 1 else "3,4").split(",")]:
        w = lj_inputs.config(c)
        g = lj.geom(w.L, w.rc, w.rs)
        q = lj.pack_aos4(torch.from_numpy(w.q).to(dev))
        perm = lj.cell_order(q, g)
        q = lj.permute_rows(q, perm)
        for padded in (False, True, "il"):
            for half in ((False, True) if c < 4 else (False,)):
                b = lj.ListBuilder(w.n, g, half, device=dev, padded=bool(padded), interleaved=padded == "il")
                lst = b.build(q)
                ms = timeit(lambda: b.build(q))
                print(json.dumps(dict(cfg=c, half=half, padded=padded, what="build", ms=round(ms, 4),
                                      entries=lst.n_entries)), flush=True)
                if padded and not half:   # (the interleaved layout: also the force step on it)
                    # lj_rebuild (wrap + cell-order permutation + list): the MD path's builder
                    q_out, p_in = torch.empty_like(q), torch.zeros_like(q)
                    p_out, perm = torch.empty_like(q), torch.empty(w.n, dtype=torch.int64, device=dev)
                    lst = b.rebuild(q, p_in, q_out, p_out, None, perm)
                    ms = timeit(lambda: b.rebuild(q, p_in, q_out, p_out, None, perm))
                    print(json.dumps(dict(cfg=c, half=half, padded=padded, what="rebuild", ms=round(ms, 4),
                                          entries=lst.n_entries)), flush=True)
                    for lanes in (0, 4 | 512, 8 | 512):
                        ms = min(timeit(lambda: lj.force_step(q_out, p_out, g, w.dt, lst, lanes_per_row=lanes),
                                        reps=20) for _ in range(3))
                        print(json.dumps(dict(cfg=c, padded=padded, what="force", lanes=lanes, ms=round(ms, 4),
                                              entries=lst.n_entries)), flush=True)
                    del q_out, p_in, p_out, perm
                del b, lst
                torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
