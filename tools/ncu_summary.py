"""Summarise ncu artefacts for profiles/: per-kernel launch times from a
`--metrics gpu__time_duration.sum --csv` log and key counters of a `--set full`
report.  Usage: python tools/ncu_summary.py launches.csv [report.ncu-rep ...]"""
import csv
import subprocess
import sys
from collections import defaultdict

KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "sm__inst_executed.sum", "sm__inst_issued.avg.pct_of_peak_sustained_active",
        "sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed",
        "TPC.TriageCompute.sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "dram__throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
        "launch__grid_size", "smsp__warps_issue_stalled_long_scoreboard_per_issue_active.ratio",
        "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_shared_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_tensor_subpipe_hmma_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_tensor_subpipe_imma_cycles_active.avg.pct_of_peak_sustained_active"]


def launches(path):
    rows = list(csv.reader(open(path)))
    start = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    h = rows[start]
    ki, vi = h.index("Kernel Name"), h.index("Metric Value")
    gi = h.index("Grid Size") if "Grid Size" in h else None
    mi = h.index("Metric Name") if "Metric Name" in h else None
    agg = defaultdict(list)
    for r in rows[start + 1:]:
        if mi is not None and r[mi] != "gpu__time_duration.sum":
            continue
        key = r[ki].split("(")[0] + (f"  grid={r[gi]}" if gi is not None else "")
        agg[key].append(float(r[vi].replace(",", "")))
    tot = sum(sum(v) for k, v in agg.items() if "ta::" in k)
    print(f"# per-kernel device time (ncu, cold cache, serialised) from {path}")
    for k, v in sorted(agg.items(), key=lambda kv: -sum(kv[1])):
        share = f"{100 * sum(v) / tot:5.1f}% of ta:: time" if "ta::" in k else ""
        print(f"{k[:96]:96s} n={len(v):3d} mean={sum(v) / len(v) / 1e3:10.2f} us {share}")


def report(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    h, units = rows[0], rows[1]
    print(f"\n# {path}")
    for r in rows[2:]:
        name = r[h.index("Kernel Name")] if "Kernel Name" in h else "?"
        print(f"kernel: {name[:90]}")
        for k in KEYS:
            if k in h:
                i = h.index(k)
                print(f"  {k:90s} {r[i]:>16s} {units[i]}")


if __name__ == "__main__":
    if sys.argv[1] != "/dev/null":  # (no launch list: report captures only)
        launches(sys.argv[1])
    for p in sys.argv[2:]:
        report(p)
