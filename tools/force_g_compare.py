"""Two force kernels on the bench's list (config 4, cell order, padded), for an ncu
capture of both: k_force<4,3> and k_force<16,3> (development tool)."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import lj_inputs  # noqa: E402
from paper_1806_05713_b200 import lj  # noqa: E402

w = lj_inputs.config(4)
g = lj.geom(w.L, w.rc, w.rs)
q = lj.pack_aos4(torch.from_numpy(w.q).cuda())
q = lj.permute_rows(q, lj.cell_order(q, g))
p = lj.pack_aos4(torch.from_numpy(w.p).cuda())
lst = lj.ListBuilder(w.n, g, False, device="cuda", padded=True).build(q)
for lanes in (4 | 3 << 8, 16 | 3 << 8, 8 | 2 << 8):
    for _ in range(2):
        lj.force_step(q, p, g, w.dt, lst, lanes_per_row=lanes)
torch.cuda.synchronize()
print("ok")
