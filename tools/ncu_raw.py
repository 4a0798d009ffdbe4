"""Print key metrics of an `ncu --page raw --csv` export and the hot SASS lines of a
`--page source --csv --print-source sass` export (development tool)."""
import csv
import sys

KEYS = ["gpu__time_duration.sum", "smsp__inst_executed.sum", "sm__inst_executed.avg.per_cycle_active",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
        "launch__occupancy_limit_registers", "launch__occupancy_limit_shared_mem",
        "l1tex__data_pipe_lsu_wavefronts.avg.pct_of_peak_sustained_elapsed",
        "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
        "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "l1tex__t_sector_hit_rate.pct",
        "lts__t_sector_hit_rate.pct", "dram__bytes_read.sum", "dram__bytes_write.sum", "sm__cycles_elapsed.avg.per_second"]


def raw(path):
    rows = list(csv.reader(open(path)))
    h, units = rows[0], rows[1]
    for v in rows[2:]:
        print("#", v[h.index("Kernel Name")][:100] if "Kernel Name" in h else "")
        for k in KEYS:
            if k in h:
                print(f"  {k} = {v[h.index(k)]} {units[h.index(k)]}")
        for i, k in enumerate(h):
            if k.startswith("smsp__average_warps_issue_stalled") and k.endswith("per_issue_active.ratio"):
                try:
                    if float(v[i]) > 0.2:
                        print(f"  {k[34:-29]} = {v[i]}")
                except ValueError:
                    pass


def source(path, thresh=0.004):
    rows = list(csv.reader(open(path)))
    h = rows[1]
    ai, si, ie, sp = h.index("Address"), h.index("Source"), h.index("Instructions Executed"), \
        h.index("Warp Stall Sampling (All Samples)")
    data = [(r[ai], r[si], int(r[ie] or 0), int(r[sp] or 0)) for r in rows[2:] if len(r) > sp]
    tot, ts = sum(d[2] for d in data), sum(d[3] for d in data)
    print("total warp instructions", tot, "stall samples", ts)
    for k, d in enumerate(data):
        if d[2] > thresh * tot or d[3] > thresh * ts:
            print(f"{k:5d} {d[2] / tot * 100:5.2f}% {d[3] / ts * 100:5.2f}%  {d[1][:90]}")


if __name__ == "__main__":
    raw(sys.argv[1])
    if len(sys.argv) > 2:
        source(sys.argv[2], float(sys.argv[3]) if len(sys.argv) > 3 else 0.004)
