"""Summaries of ncu captures for profiles/.

    python tools/ncu_summary.py full REPORT.ncu-rep KERNEL_REGEX      # --set full sections + traffic
    python tools/ncu_summary.py launches LAUNCHES.csv                 # per-kernel launch-list table
"""
import csv
import io
import subprocess
import sys
from collections import defaultdict

SECTIONS = ("GPU Speed Of Light Throughput", "Compute Workload Analysis", "Memory Workload Analysis",
            "Scheduler Statistics", "Warp State Statistics", "Occupancy", "Launch Statistics")
RAW = ("gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
       "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
       "smsp__issue_active.avg.pct_of_peak_sustained_active", "smsp__inst_executed.sum",
       "l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum", "launch__registers_per_thread")


def ncu_csv(args):
    out = subprocess.run(["ncu", "-i", *args, "--csv"], capture_output=True, text=True).stdout
    return list(csv.reader(io.StringIO(out)))


def full(rep, regex):
    rows = ncu_csv([rep, "--page", "details", "-k", f"regex:{regex}"])
    h = rows[0]
    ki, si, mi, vi, ui = (h.index(x) for x in ("Kernel Name", "Section Name", "Metric Name", "Metric Value",
                                               "Metric Unit"))
    last = None
    for r in rows[1:]:
        if r[ki] != last:
            print(f"===== {r[ki][:160]}")
            last = r[ki]
        if r[si] in SECTIONS and r[mi] and not any(x in r[mi] for x in ("Cluster", "TPC", "Green", "Stack")):
            print(f"{r[si][:28]:28s} | {r[mi]:45s} | {r[vi]:>16s} {r[ui]}")
    raw = ncu_csv([rep, "--page", "raw", "-k", f"regex:{regex}"])
    h = raw[0]
    print("===== raw counters (per launch)")
    for r in raw[2:]:
        d = dict(zip(h, r))
        print(d.get("Kernel Name", "")[:100])
        for k in RAW:
            print(f"  {k:62s} {d.get(k)}")
        stalls = []
        for k in h:
            if k.startswith("smsp__average_warps_issue_stalled") and k.endswith("per_issue_active.ratio"):
                try:
                    stalls.append((float(d[k]), k))
                except ValueError:
                    pass
        for v, k in sorted(stalls, reverse=True)[:8]:
            print(f"  {k:62s} {v:.3f}")


def launches(path):
    rows = list(csv.reader(open(path)))
    i = next(j for j, r in enumerate(rows) if r and r[0] == "ID")
    h = rows[i]
    agg = defaultdict(lambda: [0, 0.0, 0.0, 0.0])
    for r in rows[i + 1:]:
        d = dict(zip(h, r))
        a = agg[d["Kernel Name"][:110]]
        v = float(d["Metric Value"].replace(",", ""))
        m = d["Metric Name"]
        if m == "gpu__time_duration.sum":
            a[0] += 1
            a[1] += v / 1e3
        elif m == "dram__bytes_read.sum":
            a[2] += v
        elif m == "dram__bytes_write.sum":
            a[3] += v
    tot = sum(a[1] for a in agg.values())
    print(f"{'launches':>8s} {'avg us':>10s} {'share':>6s} {'rd B/launch':>12s} {'wr B/launch':>12s}  kernel")
    for k, a in sorted(agg.items(), key=lambda kv: -kv[1][1]):
        n = max(a[0], 1)
        print(f"{a[0]:8d} {a[1] / n:10.1f} {a[1] / tot * 100:5.1f}% {a[2] / n:12.4g} {a[3] / n:12.4g}  {k}")


if __name__ == "__main__":
    if sys.argv[1] == "full":
        full(sys.argv[2], sys.argv[3])
    else:
        launches(sys.argv[2])
