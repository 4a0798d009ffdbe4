"""A few force launches on config 4 (cell order, padded list) for ncu captures:
    python tools/one_force.py [il|plain] [lanes,...]   (default: il, 4|768)"""
import os
import sys

import torch

sys.path.insert(0, os.getcwd())
import lj_inputs  # noqa: E402
from paper_1806_05713_b200 import lj  # noqa: E402

layout = sys.argv[1] if len(sys.argv) > 1 else "il"
lanes_list = [int(x) for x in (sys.argv[2] if len(sys.argv) > 2 else str(4 | 768)).split(",")]
w = lj_inputs.config(4)
g = lj.geom(w.L, w.rc, w.rs)
q0 = lj.pack_aos4(torch.from_numpy(w.q).cuda())
p = lj.pack_aos4(torch.from_numpy(w.p).cuda())
q = lj.permute_rows(q0, lj.cell_order(q0, g))
lst = lj.ListBuilder(w.n, g, False, device="cuda", padded=True, interleaved=layout == "il").build(q)
cnt = torch.zeros(1, dtype=torch.int64, device="cuda")
for lanes in lanes_list:
    for _ in range(3):
        lj.force_step(q, p, g, w.dt, lst, lanes_per_row=lanes, n_interactions=cnt)
torch.cuda.synchronize()
