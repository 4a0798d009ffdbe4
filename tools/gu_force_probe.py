"""Force kernel vs gather probe per lanes-per-row G and gathers in flight U (config 4,
cell order, padded list; development tool)."""
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


cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 4
w = lj_inputs.config(cfg)
g = lj.geom(w.L, w.rc, w.rs)
q0 = lj.pack_aos4(torch.from_numpy(w.q).cuda())
p = lj.pack_aos4(torch.from_numpy(w.p).cuda())
q = lj.permute_rows(q0, lj.cell_order(q0, g))
lst = lj.ListBuilder(w.n, g, False, device="cuda", padded=True).build(q)
sink = torch.zeros(1, dtype=torch.float64, device="cuda")
IDXV = lj.LJ_LANES_IDXV
variants = [(G, U, 0) for G, U in ((2, 2), (2, 3), (4, 2), (4, 3), (4, 4), (8, 2), (8, 3), (8, 4), (16, 2), (16, 3))]
variants += [(G, V, IDXV) for G in (2, 4, 8) for V in (2, 4)] + [(16, 4, IDXV)]
for G, U, X in variants:
    lanes = G | (U << 8) | X
    try:
        f = timeit(lambda: lj.force_step(q, p, g, w.dt, lst, lanes_per_row=lanes))
    except lj.LJError as e:
        f = None
    try:
        pr = timeit(lambda: lj.gather_probe(q, lst, lanes, sink))
    except lj.LJError:
        pr = None
    print(json.dumps({"cfg": cfg, "G": G, "U": U, "idxv": bool(X), "force_ms": f and round(f, 4),
                      "probe_ms": pr and round(pr, 4), "entries": lst.n_entries}), flush=True)
