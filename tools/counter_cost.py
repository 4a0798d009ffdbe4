"""Force step with and without the interaction counter (development tool)."""
import json, os, sys
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


for c in (3, 4):
    w = lj_inputs.config(c)
    g = lj.geom(w.L, w.rc, w.rs)
    q0 = lj.pack_aos4(torch.from_numpy(w.q).cuda())
    p = lj.pack_aos4(torch.from_numpy(w.p).cuda())
    q = lj.permute_rows(q0, lj.cell_order(q0, g))
    lst = lj.ListBuilder(w.n, g, False, device="cuda", padded=True).build(q)
    cnt = torch.zeros(1, dtype=torch.int64, device="cuda")
    a = timeit(lambda: lj.force_step(q, p, g, w.dt, lst))
    b = timeit(lambda: lj.force_step(q, p, g, w.dt, lst, n_interactions=cnt))
    print(json.dumps({"cfg": c, "no_counter_ms": round(a, 4), "counter_ms": round(b, 4)}))
