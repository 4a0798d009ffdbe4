import os, sys, torch
sys.path.insert(0, os.getcwd())
import lj_inputs
from paper_1806_05713_b200 import lj
w = lj_inputs.config(4); g = lj.geom(w.L, w.rc, w.rs)
q0 = lj.pack_aos4(torch.from_numpy(w.q).cuda()); p = lj.pack_aos4(torch.from_numpy(w.p).cuda())
q = lj.permute_rows(q0, lj.cell_order(q0, g))
lst = lj.ListBuilder(w.n, g, False, device="cuda", padded=True).build(q)
for lanes in (4 | 768, 8 | 512):
    for _ in range(3):
        lj.force_step(q, p, g, w.dt, lst, lanes_per_row=lanes)
torch.cuda.synchronize()
