"""Paper-variant ablation on one GPU (development tool):
the full-list force step with the paper's layouts (AoS with padding = the
library's layout, SoA, AoS without padding, AoS8 = q and p in one 64-B record)
and four 1/r^2 evaluations, on config 4 (and 3) in cell order.  Prints one JSON
object per variant: ms per step and, on config 3, the C-12 parity error
against the CPU oracle."""
import json
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import lj_inputs  # noqa: E402
from paper_1806_05713_b200 import lj  # noqa: E402


def to_layout(rec: torch.Tensor, layout: str, p: torch.Tensor | None = None) -> torch.Tensor:
    """AoS4 records (n,4) -> the flat layout (argument marshalling for the ablation only)."""
    if layout == "aos4":
        return rec.contiguous().view(-1)
    if layout == "soa":
        return rec[:, :3].t().contiguous().view(-1)
    if layout == "aos3":
        return rec[:, :3].contiguous().view(-1)
    out = torch.cat([rec, p], dim=1)           # aos8: q record then p record
    return out.contiguous().view(-1)


def from_layout(flat: torch.Tensor, layout: str, n: int) -> torch.Tensor:
    """Momenta (n,3) from a layout's p (or, for aos8, from q's records)."""
    if layout == "aos4":
        return flat.view(n, 4)[:, :3]
    if layout == "soa":
        return flat.view(3, n).t()
    if layout == "aos3":
        return flat.view(n, 3)
    return flat.view(n, 8)[:, 4:7]


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
    cfgs = [int(c) for c in (sys.argv[1] if len(sys.argv) > 1 else "3,4").split(",")]
    for c in cfgs:
        w = lj_inputs.config(c)
        g = lj.geom(w.L, w.rc, w.rs)
        q0 = lj.pack_aos4(torch.from_numpy(w.q).to(dev))
        perm = lj.cell_order(q0, g)
        q = lj.permute_rows(q0, perm)
        rng = np.random.default_rng(7)
        p_np = rng.normal(0, 1, (w.n, 3))
        p = lj.pack_aos4(torch.from_numpy(p_np).to(dev))
        lst = lj.ListBuilder(w.n, g, False, device=dev, padded=True).build(q)
        ref = S = None
        if c == 3:   # C-12 parity against the oracle (cell-ordered storage)
            import oracle
            qn = q[:, :3].cpu().numpy().copy()
            ol = oracle.list_cells(qn, w.L, w.rs, False)
            ref = oracle.force_step(qn, p_np, w.L, w.rc, w.dt, ol)
            S = oracle.abs_contrib(qn, p_np, w.L, w.rc, w.dt, ol)
        for layout in ("aos4", "soa", "aos3", "aos8"):
            for rcp in (("newton3", "newton2", "approx", "ieee") if layout == "aos4" else ("newton3",)):
                for lanes in (4, 8):
                    pc = p.clone()
                    ql = to_layout(q, layout, pc)
                    pl = None if layout == "aos8" else to_layout(pc, layout)
                    ms = timeit(lambda: lj.force_step_variant(layout, rcp, ql, pl, w.n, g, 0.0, lst, lanes))
                    out = dict(cfg=c, layout=layout, rcp=rcp, lanes=lanes, ms=round(ms, 4),
                               G_entries_s=round(lst.n_entries / ms / 1e6, 1))
                    if ref is not None:   # one real step from p0 (fresh copies) for the parity error
                        pc = p.clone()
                        ql = to_layout(q.clone(), layout, pc)
                        pl = None if layout == "aos8" else to_layout(pc, layout)
                        lj.force_step_variant(layout, rcp, ql, pl, w.n, g, w.dt, lst, lanes)
                        got = from_layout(ql if layout == "aos8" else pl, layout, w.n).cpu().numpy()
                        out["c12_error"] = float(oracle.parity_error(got, ref, S))
                    print(json.dumps(out), flush=True)
        del lst
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
