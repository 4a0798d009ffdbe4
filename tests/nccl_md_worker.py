"""Worker for tests/test_gpu_nccl.py, launched under torch.distributed.run with
the NCCL backend (P = 1 on the one-GPU pool: LJ_FORCE_COLLECTIVES=1 makes the
driver issue every collective of the P > 1 path).  Prints one JSON line.

Checks:
  * eager NCCL steps (all-gather + all-reduce MAX, host decision) against the
    oracle's KDK loop (reading O8; energies and trajectory before chaos);
  * the captured multi-rank step (graph_collective: NCCL all-gather inside a
    CUDA graph, decision from the published pads, conditional rebuild) bit for
    bit against the same eager NCCL steps;
  * the asynchronous all-gather with interior/boundary row split (overlap) bit
    for bit against the blocking exchange.
"""
import json
import os
import sys

import numpy as np
import torch
import torch.distributed as dist

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import lj_inputs  # noqa: E402
import oracle  # noqa: E402
from paper_1806_05713_b200 import lj, md  # noqa: E402


def main():
    assert os.environ.get("LJ_FORCE_COLLECTIVES") == "1"
    local = int(os.environ.get("LOCAL_RANK", "0"))
    dev = torch.device("cuda", local)
    torch.cuda.set_device(dev)
    dist.init_process_group("nccl", device_id=dev)
    rank, world = dist.get_rank(), dist.get_world_size()
    out = {"world": world, "backend": dist.get_backend()}
    w = lj_inputs.make_system(10, jitter_seed=1, T=1.0, mom_seed=5, dt=0.005)
    g = lj.geom(w.L, w.rc, w.rs)
    rb, re_ = md.row_range(w.n, rank, world)

    def sim(overlap=False, reorder=False):
        return md.LeapfrogMD(md.LibBackend(w.n, g, rb, re_, dev), w.q, w.p, g, w.dt, rank, world,
                             dist.group.WORLD, reorder=reorder, overlap=overlap)

    # 1. eager NCCL steps vs the oracle (KDK energies at sample steps, no re-sort)
    steps, every = 200, 10
    _, _, e_ref, rb_ref = oracle.md_run(w.q, w.p, w.L, w.rc, w.rs, w.dt, steps, every)
    s = sim()
    out["collective"] = s.collective
    s.start_leapfrog()
    E = []
    for k in range(steps + 1):
        e = s.step(sample=(k % every == 0))
        if e is not None:
            E.append(e[0] + e[1])
    E, Er = np.array(E), e_ref[:, 2]
    out["energy_points"] = len(E) == len(Er)
    out["energy_start_rel"] = float(abs(E[0] - Er[0]) / abs(Er[0]))
    out["energy_first10_max_rel"] = float(np.max(np.abs(E[:11] - Er[:11]) / np.abs(Er[:11])))
    out["rebuilds"] = [s.stats.rebuilds, int(rb_ref)]

    # 2. captured multi-rank step == eager NCCL steps, bit for bit (two launches), with the
    #    re-sort at every rebuild (momenta read from the share buffers) and with fixed ownership
    for resort in (True, False):
        a, b = sim(reorder=True), sim(reorder=True)    # both start with one re-sort
        a.reorder = resort
        n_steps = 30
        gr = b.graph_collective(n_steps, resort=resort)
        ok = True
        for launch in range(2):
            for _ in range(n_steps):
                a.kick(w.dt, a.counter)
                a.drift_and_exchange()
            gr.launch()
            torch.cuda.synchronize()
            gr.finish()
            ok = ok and torch.equal(a.q[:, :3], b.q[:, :3]) and torch.equal(a.p, b.p)
            ok = ok and a.stats.rebuilds == b.stats.rebuilds
        tag = "resort" if resort else "fixed"
        out[f"graph_equals_eager_{tag}"] = bool(ok)
        out[f"graph_rebuilds_{tag}"] = b.stats.rebuilds
        out[f"graph_interactions_equal_{tag}"] = a.interactions() == b.interactions()
        gr.close()
        b.close()

    # 3. asynchronous all-gather + interior/boundary split == blocking exchange
    c, d = sim(overlap=False), sim(overlap=True)
    out["overlap_active"] = d.overlap
    for x in (c, d):
        x.start_leapfrog()
        for _ in range(40):
            x.step()
        x.sync_positions()
    out["overlap_equals_blocking"] = bool(torch.equal(c.q, d.q) and torch.equal(c.p, d.p))
    if rank == 0:
        print(json.dumps(out), flush=True)
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
