"""A/B of the index-stream cache hints (LJ_LANES_IDX_STREAM) on the bench's list (config 4,
cell order, padded): the force kernel alone back to back, and as in the MD step -- right
after a drift + displacement pass over q, p, q_ref (196 MB streamed through L2).
Development tool; one JSON line per variant."""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import lj_inputs  # noqa: E402
from paper_1806_05713_b200 import lj  # noqa: E402


def main():
    dev = torch.device("cuda:0")
    w = lj_inputs.config(4)
    g = lj.geom(w.L, w.rc, w.rs)
    q = lj.pack_aos4(torch.from_numpy(w.q).to(dev))
    q = lj.permute_rows(q, lj.cell_order(q, g))
    p = lj.pack_aos4(torch.from_numpy(w.p).to(dev))
    lst = lj.ListBuilder(w.n, g, False, device=dev, padded=True).build(q)
    qd, pd, qr = q.clone(), p.clone(), q.clone()
    disp = torch.zeros(1, dtype=torch.float64, device=dev)
    S = lj.LJ_LANES_IDX_STREAM
    st = torch.cuda.current_stream()
    for lanes in (4 | 3 << 8, 4 | 3 << 8 | S, 4 | 2 << 8, 4 | 2 << 8 | S, 8 | 2 << 8, 8 | 2 << 8 | S):
        pc = p.clone()
        for _ in range(3):
            lj.force_step(q, pc, g, w.dt, lst, lanes_per_row=lanes)
        ts = []
        for _ in range(20):
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(st)
            lj.force_step(q, pc, g, w.dt, lst, lanes_per_row=lanes)
            b.record(st)
            ts.append((a, b))
        ins = []
        for _ in range(20):
            lj.integrate_displacement(qd, pd, qr, 0.0, 0, w.n, disp)   # dt 0: streams the arrays, q unchanged
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(st)
            lj.force_step(q, pc, g, w.dt, lst, lanes_per_row=lanes)
            b.record(st)
            ins.append((a, b))
        torch.cuda.synchronize()
        iso = sorted(a.elapsed_time(b) for a, b in ts)[len(ts) // 2]
        aft = sorted(a.elapsed_time(b) for a, b in ins)[len(ins) // 2]
        print(json.dumps({"G": lanes & 0xff, "U": (lanes >> 8) & 0xff, "idx_stream": bool(lanes & S),
                          "force_ms_back_to_back": round(iso, 4), "force_ms_after_drift": round(aft, 4)}), flush=True)


if __name__ == "__main__":
    main()
