import sys, json, torch
sys.path.insert(0, '/root/repo')
import lj_inputs
from paper_1806_05713_b200 import lj
sys.path.insert(0, '/root/repo/tools')
from order_time import timeit
dev = torch.device('cuda:0')
w = lj_inputs.config(4); g = lj.geom(w.L, w.rc, w.rs)
q = lj.pack_aos4(torch.from_numpy(w.q).to(dev)); q = lj.permute_rows(q, lj.cell_order(q, g))
p = lj.pack_aos4(torch.from_numpy(w.p).to(dev))
lst = lj.ListBuilder(w.n, g, False, device=dev, padded=True).build(q)
for G in (2, 4, 8):
    for U in (2, 3, 4):
        ms = timeit(lambda: lj.force_step(q, p, g, w.dt, lst, lanes_per_row=G | (U << 8)))
        print(json.dumps(dict(G=G, U=U, ms=round(ms, 4))), flush=True)
