"""Per-phase timeline of the end-to-end step graph (development tool): graph_host_io on
config 4 with timing events at the phase boundaries; prints, per step, each event's time
relative to the step's start, and the means over steps without / with a rebuild."""
import json
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import lj_inputs  # noqa: E402
from paper_1806_05713_b200 import lj, md  # noqa: E402


def main():
    K = int(sys.argv[1]) if len(sys.argv) > 1 else 30
    w = lj_inputs.config(4)
    g = lj.geom(w.L, w.rc, w.rs)
    dev = torch.device("cuda:0")
    sim = md.LeapfrogMD(md.LibBackend(w.n, g, 0, w.n, dev), w.q, w.p, g, w.dt, reorder=True)
    for _ in range(5):
        sim.kick(w.dt, sim.counter)
        sim.drift_and_exchange()
    qh = torch.empty((w.n, 3), dtype=torch.float64, pin_memory=True)
    ph = torch.empty((w.n, 3), dtype=torch.float64, pin_memory=True)
    qh.copy_(sim.q[:, :3])
    ph.copy_(sim.p[:, :3])
    tl = []
    gr = sim.graph_host_io(K, qh, ph, timeline=tl)
    gr.launch()
    torch.cuda.synchronize()
    gr.finish()
    tl.clear()
    gr = sim.graph_host_io(K, qh, ph, timeline=tl)   # (a fresh capture: events of this launch)
    gr.launch()
    torch.cuda.synchronize()
    gr.finish()
    rows = []
    for k, t in enumerate(tl):
        s0 = t["start"]
        r = {name: round(s0.elapsed_time(e), 4) for name, e in t.items() if name != "start"}
        if k + 1 < len(tl):
            r["next_start"] = round(s0.elapsed_time(tl[k + 1]["start"]), 4)
        rows.append(r)
        print(json.dumps({"step": k, **r}), flush=True)
    for reb in (False, True):
        sel = [r for r in rows if "next_start" in r and ((r["rebuild"] - r["q_in"]) > 0.5) == reb]
        if sel:
            mean = {k: round(sum(r[k] for r in sel) / len(sel), 4) for k in sel[0]}
            print(json.dumps({"rebuild_steps": reb, "n": len(sel), "mean": mean}), flush=True)


if __name__ == "__main__":
    main()
