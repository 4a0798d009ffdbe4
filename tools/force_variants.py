"""Force kernel variants on the bench's list (config 4, cell order, padded): k_force G/U
(round 2 also timed a 4-rowsets-per-warp kernel here, since removed:
profiles/r02_force_rowsets_experiment_*.jsonl).  Development tool; one JSON line per variant."""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import lj_inputs  # noqa: E402
from paper_1806_05713_b200 import lj  # noqa: E402
from build_time import timeit  # noqa: E402


def main():
    cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 4
    dev = torch.device("cuda:0")
    w = lj_inputs.config(cfg)
    g = lj.geom(w.L, w.rc, w.rs)
    q = lj.pack_aos4(torch.from_numpy(w.q).to(dev))
    q = lj.permute_rows(q, lj.cell_order(q, g))
    p = lj.pack_aos4(torch.from_numpy(w.p).to(dev))
    lst = lj.ListBuilder(w.n, g, False, device=dev, padded=True).build(q)
    variants = [(4, 2, 0), (4, 3, 0), (8, 2, 0), (16, 2, 0)]
    ref = p.clone()
    lj.force_step(q, ref, g, w.dt, lst, lanes_per_row=4 | 3 << 8)
    for G, U, X in variants:
        lanes = G | U << 8 | X
        pc = p.clone()
        lj.force_step(q, pc, g, w.dt, lst, lanes_per_row=lanes)
        diff = float((pc - ref).abs().max())
        f = min(timeit(lambda: lj.force_step(q, pc, g, w.dt, lst, lanes_per_row=lanes), reps=20) for _ in range(3))
        print(json.dumps({"cfg": cfg, "G": G, "U": U, "force_ms": round(f, 4),
                          "max_abs_diff_vs_G4U3": diff}), flush=True)


if __name__ == "__main__":
    main()
