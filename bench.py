#!/usr/bin/env python
"""Benchmark of the LJ fp64 force hot path (arXiv 1806.05713) on B200.

Default workload (BASELINE.json metric "pair-interactions/sec ... at 1/2/4/8
B200"): config 4 -- N = 2,048,000 FCC atoms, rho = 1, jitter +-0.05, Gaussian
momenta T = 1, r_c = 3.0, r_s = 3.3, full list, rows split across ranks with a
per-step all-gather of positions, leapfrog dt = 0.01 with bookkeeping rebuilds.
A step = force + integrate + all-gather + displacement check (+ rebuild when
triggered), i.e. every §8(a) row of the path.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config 4] [--impl ours|reference]

Prints ONE JSON line on rank 0.  --impl reference times the CPU oracle
(oracle/, plain C, single thread) on a bounded sample of the same workload.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import lj_inputs  # noqa: E402

METRIC = "LJ fp64 pair-interactions/sec (G/s) and ms/force-step at 1/2/4/8 B200"
FLOP_PER_ENTRY = 22          # 21 add/mul + 1 division per full-list entry (no p_j update)
BYTES_PER_ENTRY = 36         # 4-B index + one 32-B record gather per full-list entry
BYTES_PER_ROW = 108          # q_i 32 + p_i 32 in + 32 out + pointer 8 + count 4
FP64_LANES_PER_SM = 64       # B200: 64 FP64 lanes per SM
N_SM = 148


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=None,
                    help="timed steps (default: the config's own, BASELINE.json: 100 for configs 2-4, 1000 for 5)")
    ap.add_argument("--warmup", type=int, default=10)
    ap.add_argument("--config", type=int, default=4, choices=[2, 3, 4, 5])
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--list", default=None, choices=["half", "full"], help="configs 2/3 only (default full)")
    ap.add_argument("--order", default=None, choices=["lattice", "shuffled", "cell"],
                    help="storage order; default: config 2 shuffled, 3 cell, 4/5 cell (re-sorted at every rebuild)")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--repeats", type=int, default=5,
                    help="graph step control: time the K steps this many times (min / median reported; "
                         "the headline value is the first)")
    ap.add_argument("--no-graph", action="store_true",
                    help="launch every step eagerly (configs 2/3: no force replay; MD configs: host-side step control)")
    ap.add_argument("--no-overlap", action="store_true", help="P > 1: blocking all-gather (no comm/compute overlap)")
    ap.add_argument("--exchange", default="allgather", choices=["allgather", "halo", "push"],
                    help="P > 1: position exchange between rebuilds (halo = only the rows each rank's list reads, "
                         "over NCCL send/recv; push = the same rows stored into the peers' replicas by the "
                         "integrate kernel itself over CUDA IPC / NVLink)")
    ap.add_argument("--energy-every", type=int, default=None,
                    help="NVE energy sample interval in timed steps (default: config 5 -> steps/20, else off)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    a = ap.parse_args()
    if a.steps is None:
        a.steps = lj_inputs.CONFIGS[a.config]["steps"]
    return a


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return json.load(f), "measured"
    except OSError:
        return {"hbm_gbs": 6650.0, "sm_max_mhz": 1965.0}, "fallback"


# ---- clocks sampler (NVML, during the timed region) ------------------------------

class ClockSampler:
    def __init__(self, index):
        self.samples, self.power_w, self.reasons, self.max_mhz = [], [], set(), None
        self._stop = threading.Event()
        self._t = None
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
        except Exception:  # noqa: BLE001 -- NVML missing: report no clocks
            self.nv = None

    def _run(self):
        nv = self.nv
        names = {
            "hw_slowdown": getattr(nv, "nvmlClocksEventReasonHwSlowdown", 0x8),
            "hw_thermal_slowdown": getattr(nv, "nvmlClocksEventReasonHwThermalSlowdown", 0x40),
            "sw_thermal_slowdown": getattr(nv, "nvmlClocksEventReasonSwThermalSlowdown", 0x20),
            "sw_power_cap": getattr(nv, "nvmlClocksEventReasonSwPowerCap", 0x4),
            "hw_power_brake_slowdown": getattr(nv, "nvmlClocksEventReasonHwPowerBrakeSlowdown", 0x80),
        }
        while not self._stop.is_set():
            try:
                self.samples.append(nv.nvmlDeviceGetClockInfo(self.h, nv.NVML_CLOCK_SM))
                r = nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                for k, bit in names.items():
                    if r & bit:
                        self.reasons.add(k)
            except Exception:  # noqa: BLE001
                pass
            try:
                self.power_w.append(nv.nvmlDeviceGetPowerUsage(self.h) / 1000.0)
            except Exception:  # noqa: BLE001
                pass
            time.sleep(0.005)

    def start(self):
        if self.nv is not None:
            self._t = threading.Thread(target=self._run, daemon=True)
            self._t.start()

    def stop(self):
        self._stop.set()
        if self._t is not None:
            self._t.join()
        if not self.samples:
            return None
        out = {"sm_mhz": statistics.median(self.samples), "sm_max_mhz": self.max_mhz,
               "reasons": sorted(self.reasons), "samples": len(self.samples)}
        if self.power_w:
            out["power_w"] = statistics.median(self.power_w)
        return out


# ---- the oracle as the CPU baseline / reference arm ---------------------------------

# One bounded sample of the workload for every CPU leg (cpu_baseline and --impl reference):
# rows [0, N/frac) of the config, the oracle's list of those rows built once (untimed).
SAMPLE_FRAC = {2: 1, 3: 1, 4: 8, 5: 64}


def host_info():
    """Cores this process may use and the host CPU model (the GPU box's host, not the build box)."""
    cores = len(os.sched_getaffinity(0))
    model = None
    try:
        import subprocess
        out = subprocess.run(["lscpu"], capture_output=True, text=True, timeout=10).stdout
        for line in out.splitlines():
            if line.startswith("Model name:"):
                model = line.split(":", 1)[1].strip()
                break
    except Exception:  # noqa: BLE001 -- lscpu missing
        pass
    return {"cores_available": cores, "cpu_model": model}


def oracle_sample(w, steps, frac=8, warmup=0, timings=None, threads=None):
    """Oracle (plain C) leapfrog steps on rows [0, N/frac) of the workload:
    force + integrate + displacement check per step, list built once (not timed).
    threads=None: the oracle as it stands (1 thread, the paper's protocol);
    threads=C: the all-core timing build of the full-list force step (OpenMP over rows,
    bit-identical results).  Returns (pairs/s, seconds, pairs)."""
    import oracle
    rows = w.n // frac
    q = oracle.wrap(w.q, w.L)   # a fresh contiguous copy
    lst = oracle.list_cells(q, w.L, w.rs, False, 0, rows)
    p = w.p.copy()
    qref = q.copy()
    pairs = 0.0
    t_total = 0.0
    for s in range(warmup + steps):
        t0 = time.perf_counter()
        if threads is None:
            oracle.force_step(q, p, w.L, w.rc, w.dt, lst, inplace=True)
        else:
            oracle.force_step_full_rows_parallel(q, p, w.L, w.rc, w.dt, lst, threads=threads)
        oracle.integrate(q, p, w.dt, 0, rows, inplace=True)
        oracle.max_displacement(q, qref, 0, rows)
        dt_s = time.perf_counter() - t0
        if s >= warmup:
            t_total += dt_s
            if timings is not None:
                timings.append(dt_s)
    # interactions in the sample (entries inside r_c; each pair counted from both
    # rows in a full list -> unique pairs = entries / 2, as for the GPU line)
    pr = lst.pairs()
    d = q[pr[:, 1]] - q[pr[:, 0]]
    d = np.where(d > 0.5 * w.L, d - w.L, np.where(d < -0.5 * w.L, d + w.L, d))
    inside = np.count_nonzero((d[:, 0] * d[:, 0] + d[:, 1] * d[:, 1]) + d[:, 2] * d[:, 2] < w.rc * w.rc)
    pairs = inside / 2.0 * steps
    return pairs / t_total, t_total, pairs


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    w = lj_inputs.config(args.config)
    frac = SAMPLE_FRAC[args.config]
    step_times = []
    t0 = time.perf_counter()
    value, secs, pairs = oracle_sample(w, args.steps, frac=frac, warmup=args.warmup, timings=step_times)
    sample = (f"config {args.config} rows [0, N/{frac}) = {w.n // frac} of {w.n} atoms (the same sample as "
              f"cpu_baseline); oracle list built once (untimed); {args.steps} timed leapfrog steps "
              f"(force + integrate + displacement), {args.warmup} warm-up")
    line = {
        "impl": "reference", "metric": METRIC, "value": value / 1e9, "unit": "G pair-interactions/s",
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": 1e3 * secs / args.steps, "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": f"config{args.config}", "n_atoms": w.n, "sample_rows": w.n // frac},
        "cpu_baseline": {"value": value / 1e9, "unit": "G pair-interactions/s", "cores": 1,
                         "kind": "oracle", "sample": sample, "host": host_info()},
        "e2e": {"value": value / 1e9, "unit": "G pair-interactions/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
        "wall_s": time.perf_counter() - t0,
    }
    print(json.dumps(line), flush=True)


# ---- our arm ----------------------------------------------------------------------

# the five fastest gather-replay variants of the B-15 sweep (profiles/r02_b15.json, config 4)
PROBE_VARIANTS = [4 | 3 << 8, 8 | 2 << 8, 8 | 3 << 8, 16 | 2 << 8, 16 | 3 << 8]


def lanes_str(lanes):
    s = f"G{lanes & 0xff}/U{(lanes >> 8) & 0xff}"
    return s + ("/idxv" if lanes & (1 << 16) else "")


def load_b15():
    p = os.path.join(ROOT, "profiles", "r02_b15.json")
    if not os.path.exists(p):
        return None
    with open(p) as f:
        return json.load(f)


def timed_ms(fn, stream):
    import torch
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(stream)
    fn()
    b.record(stream)
    b.synchronize()
    return a.elapsed_time(b)


def spawn_ranks(n):
    """`bench.py --gpus N` launched as a single process: re-execute it as N ranks, one
    per GPU, under torch.distributed.run (the driver's own launch line).  Fails loudly
    if fewer than N GPUs are visible -- never silently times one rank."""
    import socket

    import torch
    have = torch.cuda.device_count()
    if have < n:
        raise SystemExit(f"bench.py --gpus {n}: only {have} CUDA device(s) visible")
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.abspath(__file__), *sys.argv[1:]]
    sys.stdout.flush()
    os.execv(sys.executable, cmd)


def main():
    args = parse()
    if args.impl == "reference":
        run_reference(args)
        return

    import torch
    import torch.distributed as dist

    from paper_1806_05713_b200 import lj, md

    lj.load()   # fails loudly without the CUDA library
    if "WORLD_SIZE" not in os.environ and args.gpus > 1:
        spawn_ranks(args.gpus)   # re-executes this command under torchrun (never returns)
    world = int(os.environ.get("WORLD_SIZE", "1"))
    if world != args.gpus:
        raise SystemExit(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world}")
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if not torch.cuda.is_available():
        raise SystemExit("bench.py needs a CUDA GPU (no CPU fallback)")
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    comm = None
    if world > 1 or "MASTER_ADDR" in os.environ:   # torchrun (any N): NCCL process group
        # failure detection: NCCL errors/timeouts abort the collective instead of hanging the job
        os.environ.setdefault("TORCH_NCCL_ASYNC_ERROR_HANDLING", "1")
        import datetime
        dist.init_process_group("nccl", device_id=dev, timeout=datetime.timedelta(seconds=600))
        comm = dist.group.WORLD

    def barrier():
        if comm is not None:
            dist.barrier()

    w = lj_inputs.config(args.config)
    g = lj.geom(w.L, w.rc, w.rs)
    pk, pk_kind = peaks()
    force_only = args.config in (2, 3)
    half = (args.list == "half") if force_only else False
    if force_only and world > 1:
        raise SystemExit("configs 2/3 are single-GPU force-only benchmarks")

    order = args.order or {2: "shuffled", 3: "cell"}.get(args.config, "cell")
    rb, re_ = md.row_range(w.n, rank, world)
    be = md.LibBackend(w.n, g, rb, re_, dev, half=half)
    sim = md.LeapfrogMD(be, w.q, w.p, g, w.dt, rank, world, comm, reorder=(order == "cell"),
                        overlap=not args.no_overlap, exchange=args.exchange)
    if not force_only:
        sim.start_leapfrog()   # p_0 -> p_{-1/2}

    stream = torch.cuda.current_stream()
    f_ev = []

    def one_step(record, sample=False):
        """One step of the hot path; sample=True splits the kick around an energy
        evaluation at synchronised momenta (config 5 NVE samples)."""
        rec = record and not sample
        if rec:
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(stream)
        e = None
        if sample:
            sim.sync_positions()
            be.force(sim.q, sim.p, 0.5 * w.dt, sim.lst, sim.counter)
            e = sim.energy()
            be.force(sim.q, sim.p, 0.5 * w.dt, sim.lst)
        else:
            sim.kick(w.dt, sim.counter)   # interior rows overlap the pending all-gather (P > 1)
        if rec:
            b.record(stream)
            f_ev.append((a, b))
        if force_only:
            return e
        sim.drift_and_exchange()          # integrate, displacement check, all-gather / rebuild
        return e

    every = args.energy_every if args.energy_every is not None else (max(2, args.steps // 20) if args.config == 5 else 0)
    energies = []

    for _ in range(args.warmup):
        one_step(False)
    # force-only configs 2/3: the step is one kernel launch on a fixed list -- capture
    # it in a CUDA graph and replay it (no per-step host launch work)
    graph = None
    counted_once = None
    if force_only and not args.no_graph:
        # q is fixed in the force-only configs, so the interactions of a step are the same
        # every step: count them in one extra (untimed) launch and replay the force step
        # without the counter's atomics
        sim.interactions()
        pc = sim.p.clone()
        be.force(sim.q, pc, w.dt, sim.lst, sim.counter)
        counted_once = sim.interactions()
        del pc
        graph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(graph):
            be.force(sim.q, sim.p, w.dt, sim.lst)
        launches_per_replay = 1

        def one_step(record, sample=False):   # noqa: F811 -- the graph replay replaces the eager step
            if record:
                a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                a.record(stream)
            graph.replay()
            if record:
                b.record(stream)
                f_ev.append((a, b))
            lj_graph_launches[0] += launches_per_replay
    # MD configs on one rank: the whole step -- kick, drift + displacement, the rebuild
    # decision and the conditional rebuild -- as one CUDA graph over the K timed steps
    # (lj_md_graph, device-side decision: no host round trip per step or rebuild)
    # (P > 1, or P = 1 with LJ_FORCE_COLLECTIVES=1: graph_collective -- the NCCL all-gather captured
    # in the same graph, the decision from the displacements the all-gather carries in the q pads)
    md_graph = None
    graph_note = ""
    if not force_only and not args.no_graph:
        try:
            if sim.collective:
                if every > 0:
                    raise ValueError("energy samples at P > 1 run eagerly")
                if args.exchange != "allgather":
                    raise ValueError(f"--exchange {args.exchange} runs eagerly")
                md_graph = sim.graph_collective(args.steps)
            else:
                md_graph = sim.graph(args.steps, energy_every=every)
        except Exception as ex:   # noqa: BLE001 -- any capture failure: eager GPU steps instead, said in the line
            torch.cuda.synchronize()
            graph_note = f" (graph unavailable: {type(ex).__name__}: {ex})"
    lj_graph_launches = [0]
    sim.interactions()   # reset counter
    reb0 = sim.stats.rebuilds
    clocks = ClockSampler(local)
    barrier()
    torch.cuda.synchronize()
    clocks.start()
    launches0 = lj.launch_count()
    t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t0.record(stream)
    if md_graph is not None:
        md_graph.launch()
    else:
        for k in range(args.steps):
            e = one_step(True, sample=(every > 0 and not force_only and k % every == 0))
            if e is not None:
                energies.append((k, e[0], e[1]))
    sim.sync_positions()
    t1.record(stream)
    torch.cuda.synchronize()
    barrier()
    if md_graph is not None:
        graph_rebuilds = md_graph.finish()
        per_step, per_rebuild = md_graph.g.kernels()   # (all unrolled steps, per rebuild)
        lj_graph_launches[0] = per_step + per_rebuild * graph_rebuilds
        f_ms_graph = [t for t in md_graph.g.force_ms() if t > 0]   # sample steps are not timed
        energies = md_graph.energies()
    launches = lj.launch_count() - launches0 + lj_graph_launches[0]   # graph replays launch without the host
    ck = clocks.stop()
    ms = t0.elapsed_time(t1)
    ms_t = torch.tensor([ms], dtype=torch.float64, device=dev)
    if comm is not None:
        dist.all_reduce(ms_t, op=dist.ReduceOp.MAX)
    ms_max = float(ms_t.item())
    entries_inside = sim.interactions()           # summed over ranks and timed steps
    if counted_once is not None:                  # force-only graph replay: constant per step
        entries_inside = counted_once * args.steps
    pairs = entries_inside if half else entries_inside / 2.0
    value = pairs / (ms_max * 1e-3)
    rebuilds = sim.stats.rebuilds - reb0
    force_ms = f_ms_graph if md_graph is not None else [a.elapsed_time(b) for a, b in f_ev]
    force_note = "CUDA-event nodes around every timed step's force kernel (inside the timed region)"
    if not force_ms:
        # graph_collective has no per-step event nodes: time the same kernel on the final list,
        # on a scratch copy of p, right after the timed region
        pc = sim.p.clone()
        force_ms = [timed_ms(lambda: be.force(sim.q, pc, w.dt, sim.lst), stream) for _ in range(10)]
        force_note = "10 launches of the same kernel on the final list after the timed region"
        del pc
    force_avg = sum(force_ms) / len(force_ms)
    entries_per_launch = sim.lst.n_entries       # own rows (last list)

    # ---- roofline of the dominant kernel (the force step) ----
    # The full-list force kernel is bound by its partner gathers: every entry is one random
    # 32-B record load served by L1/L2 (the L1TEX data pipe runs at ~93 % of its wavefront peak,
    # ncu; FP64 at ~40 %).  Its floor is the force kernel's own access pattern without the
    # arithmetic -- lj_gather_probe on this list -- timed live here for the five fastest
    # lanes/unroll variants of the B-15 sweep (profiles/r02_b15.json); the fastest is the
    # "best same-list replay" (not the kernel's own G/U).  achieved / peak are the
    # algorithmic bytes of a launch (36 B per entry + 108 B per row) over the
    # force kernel's and the best replay's durations, so frac = best replay / force.
    sm_mhz = pk.get("sm_max_mhz", 1965.0)
    peak_tflops = N_SM * FP64_LANES_PER_SM * 2 * sm_mhz * 1e6 / 1e12
    E = entries_per_launch
    rows_own = re_ - rb
    gather_bytes = BYTES_PER_ENTRY * E + BYTES_PER_ROW * rows_own   # SURVEY §8(d) algorithmic bytes per launch
    fp64_ms = FLOP_PER_ENTRY * E / (peak_tflops * 1e12) * 1e3
    b15 = load_b15()
    tp = os.path.join(ROOT, "profiles", f"traffic_config{args.config}.json")
    tj = {}
    if os.path.exists(tp):
        with open(tp) as f:
            tj = json.load(f)
    traffic = tj.get("dram_bytes_per_launch")
    roof = None
    if not half:
        sink = torch.zeros(1, dtype=torch.float64, device=dev)
        probes = {}
        for lanes in PROBE_VARIANTS + [lj.default_lanes(rows_own, False)]:
            lj.gather_probe(sim.q, sim.lst, lanes, sink)
            probes[lanes] = min(timed_ms(lambda: lj.gather_probe(sim.q, sim.lst, lanes, sink), stream)
                                for _ in range(10))
        best_lanes = min(probes, key=probes.get)
        best_ms = probes[best_lanes]
        dram = None
        if traffic:
            dram = {"bytes_per_launch": traffic, "achieved_gbs": traffic / (force_avg * 1e-3) / 1e9,
                    "peak_gbs": pk.get("hbm_gbs"), "peak_kind": pk_kind,
                    "frac": traffic / (force_avg * 1e-3) / 1e9 / pk.get("hbm_gbs", 6448.4),
                    "source": f"profiles/traffic_config{args.config}.json (ncu --set full of this kernel)"}
        roof = {"bound": "l1_data_pipe",
                "achieved": gather_bytes / (force_avg * 1e-3) / 1e9,
                "peak": gather_bytes / (best_ms * 1e-3) / 1e9,
                "unit": "GB/s", "frac": best_ms / force_avg, "traffic": traffic,
                "peak_kind": "measured live: best same-list gather replay (lj_gather_probe: index loads + one "
                             "256-bit record gather per entry, no arithmetic) over lanes variants "
                             + ", ".join(lanes_str(x) for x in probes),
                "kernel": f"k_force (full list, lanes_per_row {lanes_str(lj.default_lanes(rows_own, False))})",
                "force_ms": force_avg, "force_ms_source": force_note,
                "force_ms_median": statistics.median(force_ms), "force_ms_min": min(force_ms),
                "best_replay": {"lanes_per_row": lanes_str(best_lanes), "ms": best_ms},
                "replay_ms": {lanes_str(k): v for k, v in probes.items()},
                "bytes_per_entry": BYTES_PER_ENTRY, "bytes_per_row": BYTES_PER_ROW, "entries_per_launch": E,
                "l1_data_pipe_pct_of_peak": tj.get("l1tex_lsu_wavefront_pct_of_peak"),
                "dram": dram,
                "fp64": {"achieved_tflops": FLOP_PER_ENTRY * E / (force_avg * 1e-3) / 1e12,
                         "peak_tflops": peak_tflops, "frac": fp64_ms / force_avg, "flop_per_entry": FLOP_PER_ENTRY,
                         "peak_kind": f"derived: {N_SM} SM x {FP64_LANES_PER_SM} FP64 lanes x 2 x {sm_mhz:.0f} MHz"
                                      + (f"; measured DFMA {b15['fp64_fma']['TFLOP_s']:.1f} TFLOP/s" if b15 else "")},
                "random_gather_context": (b15 or {}).get("random_gather")}
    else:
        # half list (Alg. 3): 3 fp64 REDs per entry (the 24-B p_j RMW) + 3 per row;
        # the denominator is the measured RED throughput (profiles/r02_b15.json random_red)
        reds = 3.0 * (E + rows_own)
        red_peak = None
        if b15:
            red_peak = max(r["G_red_f64_per_s"] for r in b15["random_red"])
        roof = {"bound": "red", "achieved": reds / (force_avg * 1e-3) / 1e9, "peak": red_peak,
                "unit": "G RED.F64/s", "frac": (reds / (force_avg * 1e-3) / 1e9 / red_peak) if red_peak else None,
                "traffic": traffic, "kernel": f"k_force (half list, lanes_per_row {lanes_str(lj.default_lanes(rows_own, True))})",
                "peak_kind": "measured: fp64 RED throughput to random records (tools/roofline_b15.py, "
                             "profiles/r02_b15.json)",
                "force_ms": force_avg, "reds_per_launch": reds,
                "half_list_red_replay": (b15 or {}).get("half_red_replay")}

    # ---- repeats of the timed steps (SURVEY §8(d) timing protocol: min and median) ----
    repeats = None
    if md_graph is not None and args.repeats > 1:
        rms = [ms_max / args.steps]
        for _ in range(args.repeats - 1):
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(stream)
            md_graph.launch()
            b.record(stream)
            torch.cuda.synchronize()
            md_graph.finish()
            rms.append(a.elapsed_time(b) / args.steps)
        srt = sorted(rms)
        repeats = {"n": len(rms), "ms_per_step_min": srt[0], "ms_per_step_median": srt[len(srt) // 2],
                   "note": "repeat 1 is the timed line; later repeats continue the trajectory (more rebuilds "
                           "may fall in a window)"}

    # ---- e2e: same steps through the public API with host buffers ----
    e2e = None
    if not args.no_e2e and world == 1 and not force_only and not args.no_graph and not half:
        # one rank: the K steps as ONE CUDA graph in which the state round-trips through the
        # user's (n, 3) arrays in pinned host memory every step (md.LeapfrogMD.graph_host_io):
        # H2D of p and q in 8 row chunks on a copy stream, pack, the device-side decision and
        # conditional re-sorting rebuild, the kick per chunk with that chunk's momenta sent back
        # at once, drift + displacement, q sent back; a chunk's H2D in step k+1 waits only for
        # the same chunk's D2H in step k.  One replay warms up (the trajectory
        # continues), the second is timed.
        qh = torch.empty((w.n, 3), dtype=torch.float64, pin_memory=True)
        ph = torch.empty((w.n, 3), dtype=torch.float64, pin_memory=True)
        qh.copy_(sim.q[:, :3])
        ph.copy_(sim.p[:, :3])
        sim.interactions()
        hg = sim.graph_host_io(args.steps, qh, ph)
        hg.launch()
        torch.cuda.synchronize()
        hg.finish()
        sim.interactions()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        hg.launch()
        e1.record(stream)
        torch.cuda.synchronize()
        e_reb = hg.finish()
        hg.close()
        ems = e0.elapsed_time(e1)
        e_pairs = sim.interactions() / 2.0
        nbytes = 2 * w.n * 24
        e2e = {"value": e_pairs / (ems * 1e-3) / 1e9, "unit": "G pair-interactions/s",
               "h2d_bytes_per_step": nbytes, "d2h_bytes_per_step": nbytes, "ms_per_step": ems / args.steps,
               "path": "md.LeapfrogMD.graph_host_io (one CUDA graph launch for the K steps; host arrays "
                       "round-trip every step)", "rebuilds": e_reb}
    elif not args.no_e2e:
        # host side: the user's (n, 3) position / momentum arrays in pinned memory;
        # the device packs them into the AoS4 records (lj_pack_aos4) and unpacks the
        # result (lj_unpack_aos4), so 24 B per atom and array cross PCIe, not 32.
        # The own rows are streamed in K chunks: H2D and D2H run on two copy streams
        # (PCIe is full duplex) and overlap the force on the other chunks; a chunk's
        # H2D of step k+1 waits only for the same chunk's D2H of step k (the state
        # round-trips through the host buffers every step).
        nl = re_ - rb
        K = 4 if (nl >= 1 << 20 and not half) else 1   # small systems and half lists: one chunk
        cb = [rb + (nl * c) // K for c in range(K + 1)]
        cs = [slice(cb[c] - rb, cb[c + 1] - rb) for c in range(K)]
        qh = torch.empty((nl, 3), dtype=torch.float64, pin_memory=True)
        ph = torch.empty((nl, 3), dtype=torch.float64, pin_memory=True)
        qh.copy_(sim.q[rb:re_, :3])
        ph.copy_(sim.p[rb:re_, :3])
        q_in, p_in, q_out, p_out, p_out2 = (torch.empty((nl, 3), dtype=torch.float64, device=dev) for _ in range(5))
        sim.interactions()
        barrier()
        torch.cuda.synchronize()
        ci, co = torch.cuda.Stream(), torch.cuda.Stream()
        ev_pout, ev_qout = [None] * K, [None] * K
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        ci.wait_stream(stream)
        co.wait_stream(stream)

        def h2d(dst, src, c, after):
            with torch.cuda.stream(ci):
                if after[c] is not None:
                    ci.wait_event(after[c])
                dst[cs[c]].copy_(src[cs[c]], non_blocking=True)
                return ci.record_event()

        def d2h(dst, src, c):
            return d2h_after(dst, src, c, stream.record_event())

        def d2h_after(dst, src, c, ready):
            co.wait_event(ready)
            with torch.cuda.stream(co):
                dst[cs[c]].copy_(src[cs[c]], non_blocking=True)
                return co.record_event()

        p_ready = [None] * K

        resorts = 0
        for _ in range(args.steps):
            sim.sync_positions()                  # the exchange of the previous step (P > 1)
            qd, pd = sim.q, sim.p
            ev_q = [h2d(q_in, qh, c, ev_qout) for c in range(K)]
            ev_p = [h2d(p_in, ph, c, ev_pout) for c in range(K)]
            for c in range(K):
                stream.wait_event(ev_q[c])
                lj.pack_aos4(q_in[cs[c]], out=qd[cb[c]:cb[c + 1]])
            for c in range(K):   # force per chunk as soon as its momenta have arrived
                stream.wait_event(ev_p[c])
                lj.pack_aos4(p_in[cs[c]], out=pd[cb[c]:cb[c + 1]])
                if K == 1:
                    be.force(sim.q, sim.p, w.dt, sim.lst, sim.counter)
                else:
                    be.force_rows(sim.q, sim.p, w.dt, sim.lst, cb[c], cb[c + 1], sim.counter)
                lj.unpack_aos4(pd[cb[c]:cb[c + 1]], out=p_out[cs[c]])
                p_ready[c] = stream.record_event()   # p is final after the kick (unless re-sorted)
            if not force_only:
                sim.drift_and_exchange()
            p_src = p_out
            if sim.p is not pd:                   # a rebuild re-sorted the atoms: p again
                resorts += 1
                lj.unpack_aos4(sim.p[rb:re_], out=p_out2)
                p_ready = [stream.record_event()] * K
                p_src = p_out2
            # q leaves first: the next step's force needs all of it back, while p's way back
            # (and the next H2D of a p chunk) only gates that chunk's force
            for c in range(K):
                lj.unpack_aos4(sim.q[cb[c]:cb[c + 1]], out=q_out[cs[c]])
                ev_qout[c] = d2h(qh, q_out, c)
            for c in range(K):
                ev_pout[c] = d2h_after(ph, p_src, c, p_ready[c])
        for c in range(K):
            stream.wait_event(ev_qout[c])
            stream.wait_event(ev_pout[c])
        e1.record(stream)
        torch.cuda.synchronize()
        barrier()
        ems = torch.tensor([e0.elapsed_time(e1)], dtype=torch.float64, device=dev)
        if comm is not None:
            dist.all_reduce(ems, op=dist.ReduceOp.MAX)
        e_pairs = sim.interactions()
        e_pairs = e_pairs if half else e_pairs / 2.0
        nbytes = 2 * (re_ - rb) * 24
        e2e = {"value": e_pairs / (float(ems.item()) * 1e-3) / 1e9, "unit": "G pair-interactions/s",
               "h2d_bytes_per_step": nbytes, "d2h_bytes_per_step": nbytes + resorts * (re_ - rb) * 24 / args.steps,
               "ms_per_step": float(ems.item()) / args.steps}

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        # ~10 s of single-thread oracle work (the contract's 10-30 s bounded sample), on the same
        # sample the --impl reference arm times; then the all-core OpenMP timing build on it
        frac, nst = SAMPLE_FRAC[args.config], 30
        v, secs, _ = oracle_sample(w, nst, frac=frac)
        hi = host_info()
        cpu = {"value": v / 1e9, "unit": "G pair-interactions/s", "cores": 1, "kind": "oracle",
               "sample": f"config {args.config} rows [0,N/{frac}) ({w.n // frac} atoms), {nst} oracle leapfrog steps "
                         f"(force+integrate+displacement; list built once, untimed, not rebuilt), {secs:.1f} s",
               "host": hi}
        if not half:
            nth = hi["cores_available"]
            va, secs_a, _ = oracle_sample(w, nst, frac=frac, threads=nth)
            cpu["all_core"] = {"value": va / 1e9, "cores": nth, "seconds": secs_a,
                               "kind": "oracle all-core timing build (OpenMP over full-list rows, bit-identical)"}

    if rank == 0:
        line = {
            "metric": METRIC, "value": value / 1e9, "unit": "G pair-interactions/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_max / args.steps,
            # the workload is a fixed system (config 4: 2.048 M atoms) whose rows are split over the
            # ranks, with a real exchange step: total work fixed as N grows
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
            "dtype": "f64", "data": "synthetic",
            "config": {"workload": f"config{args.config}", "n_atoms": w.n, "list": "half" if half else "full",
                       "order": order + ((" (re-sorted at every rebuild)" if sim.reorder else
                                          " (sorted once, then fixed row ownership)")
                                         + (", new own rows' momenta read from the owner ranks over NVLink"
                                            if sim.reorder and sim.collective and md_graph is not None else "")
                                         if order == "cell" and not force_only else ""),
                       "dt": w.dt, "rc": w.rc, "rs": w.rs, "parallelism": f"rows/{world}",
                       "exchange": (("fused integrate + NVLink push" if sim.push else "halo" if sim.halo else "all-gather")
                                    + (" (async, overlapped with the interior rows' force)" if sim.overlap else "")
                                    if (world > 1 or sim.collective) else "none (1 rank)"),
                       "l2": "inputs larger than L2 (list %.2f GB of entries in a %.2f GB padded array + %.0f MB of records)"
                             % (4 * sim.lst.n_entries / 1e9, 4 * sim.lst.sorted_list.numel() / 1e9, 64 * w.n / 1e6),
                       "rebuilds_in_timed_steps": rebuilds},
            "ms_per_force_step": force_avg,
            "cuda_graph": (graph is not None or md_graph is not None),
            "interactions_counted": ("once (q fixed in the force-only configs), x steps" if counted_once is not None
                                     else "live, every timed step (kernel counter)"),
            "step_control": (("device (graph_collective: NCCL all-gather + conditional rebuild node captured in one "
                              "graph for the timed steps; decision from the displacements carried in the q pads)"
                              if sim.collective else
                              "device (lj_md_graph: conditional rebuild node, one graph launch for the timed steps)")
                             if md_graph is not None else "host" + graph_note),
            "roofline": roof,
            "repeats": repeats,
            "cpu_baseline": cpu, "e2e": e2e, "gpu_launches": launches, "clocks": ck,
        }
        if energies:
            E = np.array([ke + pe for _, ke, pe in energies])
            ks = np.array([k for k, _, _ in energies], dtype=np.float64)
            slope = float(np.polyfit(ks * w.dt, E / w.n, 1)[0]) if len(E) > 2 else None
            line["nve"] = {"samples": len(E), "every": every, "E0_per_atom": float(E[0] / w.n),
                           "drift_end_per_atom": float((E[-1] - E[0]) / w.n),
                           "max_abs_dev_per_atom": float(np.abs(E - E[0]).max() / w.n),
                           "slope_per_atom_per_time": slope, "note": "energy samples split the kick (KDK) at "
                           "sample steps; their force time is excluded from ms_per_force_step"}
        print(json.dumps(line), flush=True)
    if comm is not None:
        barrier()
        sim.close()   # unmap the peers' replicas (push exchange)
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
