"""Force / build timing on one GPU (development tool): config 4 (or argv[1])
re-sorted into cell order; padded and compact lists; 4 and 8 lanes per row;
the gather probe."""
import json
import os
import sys

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
    c = int(sys.argv[1]) if len(sys.argv) > 1 else 4
    w = lj_inputs.config(c)
    g = lj.geom(w.L, w.rc, w.rs)
    q0 = lj.pack_aos4(torch.from_numpy(w.q).to(dev))
    p = lj.pack_aos4(torch.from_numpy(w.p).to(dev))
    for fine in (False,):
        q = lj.permute_rows(q0, lj.cell_order(q0, g))
        for padded in (True, False):
            b = lj.ListBuilder(w.n, g, False, device=dev, padded=padded)
            lst = b.build(q)
            ms_b = timeit(lambda: b.build(q), reps=5, warm=1)
            out = dict(cfg=c, fine=fine, padded=padded, build_ms=round(ms_b, 4))
            for lanes in (4, 8):
                out[f"force_G{lanes}_ms"] = round(timeit(lambda: lj.force_step(q, p, g, w.dt, lst, lanes_per_row=lanes)), 4)
            sink = torch.zeros(1, dtype=torch.float64, device=dev)
            out["probe_G8_ms"] = round(timeit(lambda: lj.gather_probe(q, lst, 8, sink)), 4)
            print(json.dumps(out), flush=True)
            del b, lst
            torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
