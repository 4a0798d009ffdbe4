"""Build the config-4 list (cell order) a few times -- for ncu launch lists of the builder."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import lj_inputs  # noqa: E402
from paper_1806_05713_b200 import lj  # noqa: E402

c = sys.argv[1] if len(sys.argv) > 1 else "4c"
w = lj_inputs.config(int(c[0]))
g = lj.geom(w.L, w.rc, w.rs)
q = lj.pack_aos4(torch.from_numpy(w.q).cuda())
if c.endswith("c"):
    q = lj.permute_rows(q, lj.cell_order(q, g))
b = lj.ListBuilder(w.n, g, False, device=q.device)
for _ in range(3):
    lst = b.build(q)
torch.cuda.synchronize()
print("entries", lst.n_entries)
