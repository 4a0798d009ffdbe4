"""Small end-to-end run of every kernel (development tool; compute-sanitizer is
closed on the GPU pool, so this is the all-kernels smoke run instead):
lists (fast v4, exact v2 on unwrapped input, fallback on a dense gas, compact
and padded), lj_rebuild, force (full/half/ordered/variants), integrate, wrap,
displacement, energy, cell order, a few MD steps."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import lj_inputs  # noqa: E402
from paper_1806_05713_b200 import lj, md  # noqa: E402


def main():
    dev = torch.device("cuda:0")
    w = lj_inputs.config(1)
    g = lj.geom(w.L, w.rc, w.rs)
    q = lj.pack_aos4(torch.from_numpy(w.q).to(dev))
    p = lj.pack_aos4(torch.from_numpy(np.random.default_rng(1).normal(0, 1, (w.n, 3))).to(dev))
    for half in (False, True):
        for padded in (False, True):
            lst = lj.ListBuilder(w.n, g, half, device=dev, padded=padded).build(q)
            lj.force_step(q, p, g, w.dt, lst)
            if not half:
                lj.force_step(q, p, g, w.dt, lst, ordered=True)
                lj.energy(q, p, g, lst)
                lj.gather_probe(q, lst)
    # exact kernel (unwrapped input) and the fallback (dense gas)
    qu = lj.pack_aos4(torch.from_numpy(w.q + 0.12).to(dev))
    lj.build_list(qu, g, False)
    qd = lj.pack_aos4(torch.from_numpy(lj_inputs.random_gas(3000, 9.9, 3)).to(dev))
    lj.build_list(qd, lj.geom(9.9, 3.0, 3.3), False)
    # cell-ordered system: v4 staging by runs, rebuild, variants
    w3 = lj_inputs.config(1)
    q3 = lj.permute_rows(q, lj.cell_order(q, g))
    b = lj.ListBuilder(w3.n, g, False, device=dev, padded=True)
    lst = b.build(q3)
    for layout in ("aos4", "soa", "aos3", "aos8"):
        qs = q3.clone().view(-1) if layout == "aos4" else (
            q3[:, :3].t().contiguous().view(-1) if layout == "soa" else
            (q3[:, :3].contiguous().view(-1) if layout == "aos3" else torch.cat([q3, p], 1).contiguous().view(-1)))
        ps = None if layout == "aos8" else torch.zeros_like(qs)
        lj.force_step_variant(layout, "newton3", qs, ps, w3.n, g, w3.dt, lst, 8)
    qa, pa, qr = torch.empty_like(q), torch.empty_like(p), torch.empty_like(q)
    perm = torch.empty(w.n, dtype=torch.int64, device=dev)
    b.rebuild(q.clone(), p, qa, pa, qr, perm)
    lj.list_interior(lst.rows_view(1000, 3000))
    lj.integrate(q3, p, w.dt)
    lj.wrap(q3, w.L, qr)
    lj.max_displacement(q3, qr)
    # MD through the driver
    wm = lj_inputs.make_system(8, jitter_seed=1, T=1.0, mom_seed=5, dt=0.01)
    gm = lj.geom(wm.L, wm.rc, wm.rs)
    sim = md.LeapfrogMD(md.LibBackend(wm.n, gm, 0, wm.n, dev), wm.q, wm.p, gm, wm.dt)
    sim.start_leapfrog()
    for k in range(12):
        sim.step(sample=(k == 5))
    # NEXT-3 half list with shared-memory windows, NEXT-2 fused drift + push (emulated
    # peer), the MD step as a CUDA graph with the conditional rebuild
    bh = lj.ListBuilder(w3.n, g, True, device=dev, padded=True)
    lh = bh.build(q3)
    lj.force_step_half_cells(q3, p.clone(), g, w3.dt, lh, bh.cell_starts())
    peer = torch.zeros_like(q3)
    lj.integrate_push(q3, q3.clone(), p, qr, w3.dt, 0, w3.n, torch.zeros(1, dtype=torch.float64, device=dev),
                      [(peer.data_ptr(), 100, 900)])
    gr = md.LeapfrogMD(md.LibBackend(wm.n, gm, 0, wm.n, dev), wm.q, wm.p, gm, wm.dt).graph(8)
    gr.launch()
    torch.cuda.synchronize()
    gr.finish()
    gr.close()
    torch.cuda.synchronize()
    print("sanitize run ok, launches", lj.launch_count())


if __name__ == "__main__":
    main()
