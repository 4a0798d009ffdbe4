"""Where the end-to-end step's time goes (development tool), config 4, one GPU:
the device-only step graph (lj_md_graph), graph_host_io as bench.py runs it, and
graph_host_io with 1 / 8 / 16 row chunks, and with the momenta's copies left out.  One JSON line each (ms per step over K steps)."""
import json
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import lj_inputs  # noqa: E402
from paper_1806_05713_b200 import lj, md  # noqa: E402


def run(sim, gr, K):
    gr.launch()
    torch.cuda.synchronize()
    gr.finish()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    gr.launch()
    e.record()
    torch.cuda.synchronize()
    gr.finish()
    gr.close()
    return s.elapsed_time(e) / K


def main():
    K = int(sys.argv[1]) if len(sys.argv) > 1 else 40
    w = lj_inputs.config(4)
    g = lj.geom(w.L, w.rc, w.rs)
    dev = torch.device("cuda:0")
    sim = md.LeapfrogMD(md.LibBackend(w.n, g, 0, w.n, dev), w.q, w.p, g, w.dt, reorder=True)
    for _ in range(5):
        sim.kick(w.dt, sim.counter)
        sim.drift_and_exchange()
    print(json.dumps({"what": "lj_md_graph (device only)", "ms_per_step": round(run(sim, sim.graph(K), K), 4)}),
          flush=True)
    qh = torch.empty((w.n, 3), dtype=torch.float64, pin_memory=True)
    ph = torch.empty((w.n, 3), dtype=torch.float64, pin_memory=True)
    for chunks in (4, 1, 8):
        qh.copy_(sim.q[:, :3])
        ph.copy_(sim.p[:, :3])
        ms = run(sim, sim.graph_host_io(K, qh, ph, chunks=chunks), K)
        print(json.dumps({"what": "graph_host_io", "chunks": chunks, "ms_per_step": round(ms, 4)}), flush=True)
    for chunks in (16,):
        qh.copy_(sim.q[:, :3])
        ph.copy_(sim.p[:, :3])
        ms = run(sim, sim.graph_host_io(K, qh, ph, chunks=chunks), K)
        print(json.dumps({"what": "graph_host_io", "chunks": chunks, "ms_per_step": round(ms, 4)}), flush=True)
    # the momenta's copies left out (D2H and H2D of p patched to no-ops at capture; the device p
    # is then re-packed from p_in's stale contents every step -- a timing-only variant)
    real = lj.copy_bytes
    lj.copy_bytes = lambda dst, src: None if (dst.data_ptr() == ph.data_ptr() or src.data_ptr() == ph.data_ptr()
                                              or _in_p(dst, src, ph)) else real(dst, src)
    try:
        qh.copy_(sim.q[:, :3])
        ph.copy_(sim.p[:, :3])
        ms = run(sim, sim.graph_host_io(K, qh, ph, chunks=8), K)
        print(json.dumps({"what": "graph_host_io, q round trip only (timing variant)", "chunks": 8,
                          "ms_per_step": round(ms, 4)}), flush=True)
    finally:
        lj.copy_bytes = real


def _in_p(dst, src, ph):
    lo, hi = ph.data_ptr(), ph.data_ptr() + ph.numel() * 8
    return lo <= dst.data_ptr() < hi or lo <= src.data_ptr() < hi


if __name__ == "__main__":
    main()
