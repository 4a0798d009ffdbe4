"""Experiment (development tool): would an interleaved padded row layout -- slot
8c + 2g + u holds entry 8c + 4u + g, so that lane g of a 4-lane group gets its two
entries of a chunk with ONE 64-bit index load -- make the force kernel faster?
k_force_idxv<4, 2> on the interleaved list reproduces k_force<4, 2>'s gather pattern
exactly with half the index requests.  Rows are rounded up to a multiple of 8 entries
(the padding slots point at the row's own atom: r = 0, masked by the cutoff test), so
the interleaved runs do ~2 % more entries.  Timing only."""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import lj_inputs  # noqa: E402
from paper_1806_05713_b200 import lj  # noqa: E402
from build_time import timeit  # noqa: E402


def main():
    dev = torch.device("cuda:0")
    w = lj_inputs.config(4)
    g = lj.geom(w.L, w.rc, w.rs)
    q = lj.pack_aos4(torch.from_numpy(w.q).to(dev))
    q = lj.permute_rows(q, lj.cell_order(q, g))
    p = lj.pack_aos4(torch.from_numpy(w.p).to(dev))
    lst = lj.ListBuilder(w.n, g, False, device=dev, padded=True).build(q)
    S = lj.LJ_PADDED_ROW_STRIDE
    n = w.n
    L2 = lst.sorted_list[: n * S].view(n, S)
    npart = lst.number_of_partners.long()
    n8 = (npart + 7) // 8 * 8
    assert int(n8.max()) <= S
    own = torch.arange(n, device=dev, dtype=torch.int32).unsqueeze(1).expand(n, S)
    slot = torch.arange(S, device=dev).unsqueeze(0)
    filled = torch.where(slot < npart.unsqueeze(1), L2, own)               # pad slots -> own atom
    e = torch.arange(S, device=dev)
    c, rem = e // 8, e % 8
    src = c * 8 + (rem % 2) * 4 + rem // 2                                  # slot s holds entry src[s]
    src = torch.where(src < S, src, e)
    il = torch.gather(filled, 1, src.unsqueeze(0).expand(n, S).contiguous())
    lst8 = lj.CSRList(n8.to(torch.int32), lst.pointer, filled.reshape(-1).contiguous(), -1, 0, n, False, True)
    lsti = lj.CSRList(n8.to(torch.int32), lst.pointer, il.reshape(-1).contiguous(), -1, 0, n, False, True)
    sink = torch.zeros(1, dtype=torch.float64, device=dev)
    out = {}
    for name, L_, lanes in (("k_force<4,2> plain", lst, 4 | 2 << 8), ("k_force<4,3> plain", lst, 4 | 3 << 8),
                            ("k_force<4,2> rows rounded to 8", lst8, 4 | 2 << 8),
                            ("k_force_idxv<4,2> interleaved", lsti, 4 | 2 << 8 | lj.LJ_LANES_IDXV),
                            ("k_force_idxv<4,2> plain (entries 2g, 2g+1)", lst8, 4 | 2 << 8 | lj.LJ_LANES_IDXV)):
        pc = p.clone()
        f = min(timeit(lambda: lj.force_step(q, pc, g, w.dt, L_, lanes_per_row=lanes), reps=20) for _ in range(3))
        pr = min(timeit(lambda: lj.gather_probe(q, L_, lanes, sink), reps=20) for _ in range(3))
        out[name] = (f, pr)
        print(json.dumps({"variant": name, "force_ms": round(f, 4), "probe_ms": round(pr, 4)}), flush=True)


if __name__ == "__main__":
    main()
