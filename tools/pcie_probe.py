"""Host <-> device copy rates on the box (development tool): pinned (n, 3) float64
arrays of config 4's size, H2D alone, D2H alone, both at once on two streams, and the
e2e step's volume (q and p each way).  One JSON line per measurement."""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1806_05713_b200 import lj  # noqa: E402


def timed(fn, reps=10):
    fn()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(reps):
        fn()
    e.record()
    torch.cuda.synchronize()
    return s.elapsed_time(e) / reps


def main():
    n = 2048000
    dev = torch.device("cuda:0")
    hs = [torch.empty((n, 3), dtype=torch.float64, pin_memory=True) for _ in range(4)]
    ds = [torch.empty((n, 3), dtype=torch.float64, device=dev) for _ in range(4)]
    nb = n * 24
    main_s = torch.cuda.current_stream()
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()

    def h2d():
        lj.copy_bytes(ds[0], hs[0])

    def d2h():
        lj.copy_bytes(hs[1], ds[1])

    def both():
        s1.wait_stream(main_s)
        s2.wait_stream(main_s)
        with torch.cuda.stream(s1):
            lj.copy_bytes(ds[0], hs[0])
        with torch.cuda.stream(s2):
            lj.copy_bytes(hs[1], ds[1])
        main_s.wait_stream(s1)
        main_s.wait_stream(s2)

    def step_volume():   # q and p each way, the two directions on two streams
        s1.wait_stream(main_s)
        s2.wait_stream(main_s)
        with torch.cuda.stream(s1):
            lj.copy_bytes(ds[0], hs[0])
            lj.copy_bytes(ds[2], hs[2])
        with torch.cuda.stream(s2):
            lj.copy_bytes(hs[1], ds[1])
            lj.copy_bytes(hs[3], ds[3])
        main_s.wait_stream(s1)
        main_s.wait_stream(s2)

    def two_h2d():   # two H2D at once on two streams
        s1.wait_stream(main_s)
        s2.wait_stream(main_s)
        with torch.cuda.stream(s1):
            lj.copy_bytes(ds[0], hs[0])
        with torch.cuda.stream(s2):
            lj.copy_bytes(ds[2], hs[2])
        main_s.wait_stream(s1)
        main_s.wait_stream(s2)

    for name, fn, b in (("h2d", h2d, nb), ("d2h", d2h, nb), ("h2d+d2h concurrent", both, 2 * nb),
                        ("two h2d concurrent", two_h2d, 2 * nb), ("e2e step volume (2 each way)", step_volume, 4 * nb)):
        ms = min(timed(fn) for _ in range(3))
        print(json.dumps({"what": name, "bytes": b, "ms": round(ms, 4), "GB_s": round(b / ms / 1e6, 2)}), flush=True)
    # the same step volume captured into a CUDA graph (as graph_host_io's memcpy nodes)
    g = torch.cuda.CUDAGraph()
    cs = torch.cuda.Stream()
    cs.wait_stream(main_s)
    with torch.cuda.graph(g, stream=cs):
        step_volume()
    ms = min(timed(g.replay) for _ in range(3))
    print(json.dumps({"what": "e2e step volume, graph-captured", "bytes": 4 * nb, "ms": round(ms, 4),
                      "GB_s": round(4 * nb / ms / 1e6, 2)}), flush=True)
    g2 = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g2, stream=cs):   # 8 chunks per array, each direction on its own stream
        s1.wait_stream(cs)
        s2.wait_stream(cs)
        for a in range(2):
            for c in range(8):
                lo, hi = n * c // 8, n * (c + 1) // 8
                with torch.cuda.stream(s1):
                    lj.copy_bytes(ds[2 * a][lo:hi], hs[2 * a][lo:hi])
                with torch.cuda.stream(s2):
                    lj.copy_bytes(hs[2 * a + 1][lo:hi], ds[2 * a + 1][lo:hi])
        cs.wait_stream(s1)
        cs.wait_stream(s2)
    ms = min(timed(g2.replay) for _ in range(3))
    print(json.dumps({"what": "e2e step volume, graph-captured, 8 chunks", "bytes": 4 * nb, "ms": round(ms, 4),
                      "GB_s": round(4 * nb / ms / 1e6, 2)}), flush=True)


if __name__ == "__main__":
    main()
