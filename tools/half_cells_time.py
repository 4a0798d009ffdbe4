"""Half-list force step: CSR kernel with per-entry REDs (lj_force_step, half = 1) vs the
per-cell shared-memory windows (lj_force_step_half_cells), configs 3 and 4 in cell
order (development tool).  One JSON object per measurement."""
import json
import os
import sys

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
    for cfg in [int(x) for x in (sys.argv[1] if len(sys.argv) > 1 else "3,4").split(",")]:
        w = lj_inputs.config(cfg)
        g = lj.geom(w.L, w.rc, w.rs)
        q0 = lj.pack_aos4(torch.from_numpy(w.q).cuda())
        p0 = lj.pack_aos4(torch.from_numpy(np.random.default_rng(1).normal(0, 1, (w.n, 3))).cuda())
        q = torch.empty_like(q0)
        p = torch.empty_like(p0)
        perm = torch.empty(w.n, dtype=torch.int64, device="cuda")
        for half in (True, False):
            b = lj.ListBuilder(w.n, g, half, device="cuda", padded=True)
            lst = b.rebuild(q0.clone(), p0, q, p, None, perm)
            cnt = torch.zeros(1, dtype=torch.int64, device="cuda")
            lj.force_step(q, p.clone(), g, w.dt, lst, n_interactions=cnt)
            pairs = int(cnt.item()) // (1 if half else 2)
            if half:
                cst = b.cell_starts()
                for name, fn in (("half_csr_red", lambda: lj.force_step(q, p, g, w.dt, lst)),
                                 ("half_cells", lambda: lj.force_step_half_cells(q, p, g, w.dt, lst, cst)),
                                 ("half_cells_g8", lambda: lj.force_step_half_cells(q, p, g, w.dt, lst, cst, 8 | 512)),
                                 ("half_cells_u3", lambda: lj.force_step_half_cells(q, p, g, w.dt, lst, cst, 4 | 768)),
                                 ("half_cells_g2", lambda: lj.force_step_half_cells(q, p, g, w.dt, lst, cst, 2 | 512))):
                    ms = timeit(fn)
                    print(json.dumps({"cfg": cfg, "kernel": name, "ms": round(ms, 4), "G_pairs_s": round(pairs / ms / 1e6, 2)}))
            else:
                ms = timeit(lambda: lj.force_step(q, p, g, w.dt, lst))
                print(json.dumps({"cfg": cfg, "kernel": "full", "ms": round(ms, 4), "G_pairs_s": round(pairs / ms / 1e6, 2)}))


if __name__ == "__main__":
    main()
