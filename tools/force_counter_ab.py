"""The force kernel with and without the interaction counter (development tool; config 4, the
bench's list): back-to-back medians of 20 launches."""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import lj_inputs  # noqa: E402
from paper_1806_05713_b200 import lj  # noqa: E402

dev = torch.device("cuda:0")
w = lj_inputs.config(4)
g = lj.geom(w.L, w.rc, w.rs)
q = lj.pack_aos4(torch.from_numpy(w.q).to(dev))
q = lj.permute_rows(q, lj.cell_order(q, g))
p = lj.pack_aos4(torch.from_numpy(w.p).to(dev))
lst = lj.ListBuilder(w.n, g, False, device=dev, padded=True).build(q)
cnt = torch.zeros(1, dtype=torch.int64, device=dev)
st = torch.cuda.current_stream()
for counter in (None, cnt, None, cnt):
    pc = p.clone()
    for _ in range(3):
        lj.force_step(q, pc, g, w.dt, lst, n_interactions=counter)
    ev = []
    for _ in range(20):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(st)
        lj.force_step(q, pc, g, w.dt, lst, n_interactions=counter)
        b.record(st)
        ev.append((a, b))
    torch.cuda.synchronize()
    t = sorted(a.elapsed_time(b) for a, b in ev)
    print(json.dumps({"counter": counter is not None, "median_ms": round(t[10], 4), "min_ms": round(t[0], 4)}))
