"""Force-step timing with and without the interaction counter, cold and warm
(development tool): config 4 in cell order, padded list."""
import json
import os
import sys

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


def main():
    dev = torch.device("cuda:0")
    w = lj_inputs.config(4)
    g = lj.geom(w.L, w.rc, w.rs)
    q = lj.pack_aos4(torch.from_numpy(w.q).to(dev))
    q = lj.permute_rows(q, lj.cell_order(q, g))
    p = lj.pack_aos4(torch.from_numpy(w.p).to(dev))
    lst = lj.ListBuilder(w.n, g, False, device=dev, padded=True).build(q)
    cnt = torch.zeros(1, dtype=torch.int64, device=dev)
    print(json.dumps(dict(what="no counter", ms=round(timeit(lambda: lj.force_step(q, p, g, w.dt, lst)), 4))))
    print(json.dumps(dict(what="counter", ms=round(timeit(
        lambda: lj.force_step(q, p, g, w.dt, lst, n_interactions=cnt)), 4))))
    # one launch at a time after a host sync (the bench's per-step pattern)
    ts = []
    for _ in range(20):
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        lj.force_step(q, p, g, w.dt, lst, n_interactions=cnt)
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    print(json.dumps(dict(what="counter, synced launches", ms=round(sum(ts) / len(ts), 4))))
    flush = torch.empty(512 * 1024 * 1024, dtype=torch.uint8, device=dev)
    ts = []
    for _ in range(20):
        flush.fill_(1)   # evict L2 (the bench's steps run between other kernels)
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        lj.force_step(q, p, g, w.dt, lst, n_interactions=cnt)
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    print(json.dumps(dict(what="counter, synced, L2 flushed", ms=round(sum(ts) / len(ts), 4))))


if __name__ == "__main__":
    main()
