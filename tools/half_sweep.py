import json, sys, os, torch, numpy as np
sys.path.insert(0, os.getcwd())
import lj_inputs
from paper_1806_05713_b200 import lj
def timeit(fn, reps=30, warm=3):
    for _ in range(warm): fn()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize(); s.record()
    for _ in range(reps): fn()
    e.record(); torch.cuda.synchronize()
    return s.elapsed_time(e) / reps
for c in (2, 3):
    w = lj_inputs.config(c); g = lj.geom(w.L, w.rc, w.rs)
    q = lj.pack_aos4(torch.from_numpy(w.q).cuda())
    p = lj.pack_aos4(torch.from_numpy(w.p).cuda())
    lst = lj.ListBuilder(w.n, g, True, device="cuda", padded=True).build(q)
    for lanes in (1, 2 | 512, 4 | 512, 4 | 768, 4 | 1024, 8 | 512, 8 | 768, 16 | 512, 32 | 512):
        ms = timeit(lambda: lj.force_step(q, p, g, w.dt, lst, lanes_per_row=lanes))
        print(json.dumps(dict(cfg=c, lanes=lanes, ms=round(ms, 4))), flush=True)
    cnt = torch.zeros(1, dtype=torch.int64, device="cuda")
    ms = timeit(lambda: lj.force_step(q, p, g, w.dt, lst, n_interactions=cnt))
    print(json.dumps(dict(cfg=c, lanes="default+counter", ms=round(ms, 4))), flush=True)
