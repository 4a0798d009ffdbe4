"""Builder cost when the storage order has drifted from cell order (development tool):
config 4 sorted into cell order once, then K eager MD steps WITHOUT re-sorting (fixed
ownership, as graph_collective), then lj_build_list timed on that state, against the
same positions re-sorted into cell order.  One JSON line per K."""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import lj_inputs  # noqa: E402
from paper_1806_05713_b200 import lj, md  # noqa: E402
from build_time import timeit  # noqa: E402


def main():
    dev = torch.device("cuda:0")
    w = lj_inputs.config(4)
    g = lj.geom(w.L, w.rc, w.rs)
    sim = md.LeapfrogMD(md.LibBackend(w.n, g, 0, w.n, dev), w.q, w.p, g, w.dt, reorder=True)
    sim.reorder = False
    done = 0
    for K in (0, 10, 50, 100, 200):
        while done < K:
            sim.step()
            done += 1
        sim._resolve()
        q = sim.q.clone()
        lj.wrap(q, w.L)
        b = lj.ListBuilder(w.n, g, False, device=dev, padded=True)
        b.build(q)
        ms_drift = timeit(lambda: b.build(q))
        qs = lj.permute_rows(q, lj.cell_order(q, g))
        ms_sorted = timeit(lambda: b.build(qs))
        print(json.dumps(dict(steps_since_sort=K, rebuilds=sim.stats.rebuilds, build_ms_drifted=round(ms_drift, 4),
                              build_ms_cell_order=round(ms_sorted, 4))), flush=True)
        del b
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
