#!/usr/bin/env python3
"""Summarise ncu captures into markdown for profiles/ (run here, no GPU).

  python tools/ncu_summary.py rep1.ncu-rep [rep2 ...] > profiles/xxx.md
  python tools/ncu_summary.py --launches launches.csv > profiles/xxx_launches.md
"""
import collections
import csv
import io
import subprocess
import sys

KEYS = [
    ("gpu__time_duration.sum", "duration"),
    ("launch__grid_size", "grid"),
    ("launch__block_size", "block"),
    ("launch__registers_per_thread", "regs"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "warps active %"),
    ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue active %"),
    ("smsp__inst_executed.sum", "warp instr"),
    ("smsp__thread_inst_executed_per_inst_executed.ratio", "threads/instr"),
    ("sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active", "fp64 pipe %"),
    ("sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active", "fma pipe %"),
    ("sm__inst_executed_pipe_tensor_subpipe_hmma.avg.pct_of_peak_sustained_active", "tensor hmma %"),
    ("dram__bytes_read.sum", "dram read"),
    ("dram__bytes_write.sum", "dram write"),
    ("l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", "smem wavefronts"),
    ("smsp__average_warps_issue_stalled_barrier_per_issue_active.ratio", "stall barrier"),
    ("smsp__average_warps_issue_stalled_membar_per_issue_active.ratio", "stall membar"),
    ("smsp__average_warps_issue_stalled_short_scoreboard_per_issue_active.ratio", "stall short_sb"),
    ("smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio", "stall long_sb"),
    ("smsp__average_warps_issue_stalled_wait_per_issue_active.ratio", "stall wait"),
    ("smsp__average_warps_issue_stalled_math_pipe_throttle_per_issue_active.ratio", "stall math_throttle"),
    ("smsp__average_warps_issue_stalled_mio_throttle_per_issue_active.ratio", "stall mio_throttle"),
    ("smsp__average_warps_issue_stalled_branch_resolving_per_issue_active.ratio", "stall branch"),
]


def raw(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    h, units = rows[0], rows[1]
    res = []
    for row in rows[2:]:
        d = dict(zip(h, row))
        u = dict(zip(h, units))
        res.append((d, u))
    return res


def fmt(v, unit):
    try:
        x = float(v.replace(",", ""))
    except (ValueError, AttributeError):
        return v
    if unit in ("ns", "us", "ms", "s") or unit.endswith("second"):
        return f"{x:.3f} {unit}"
    if unit == "byte" or unit.startswith("Kbyte") or unit.startswith("Mbyte"):
        return f"{x:.4g} {unit}"
    if abs(x) >= 1e6:
        return f"{x:.4g}"
    return f"{x:.3f}".rstrip("0").rstrip(".")


def summarize(reps):
    cols = []
    for rep in reps:
        for d, u in raw(rep):
            name = d.get("Kernel Name", "?")
            cols.append((rep.split("/")[-1].replace(".ncu-rep", ""), name, d, u))
    print("| metric | " + " | ".join(f"{c[0]}<br>`{c[1][:60]}`" for c in cols) + " |")
    print("|---|" + "---|" * len(cols))
    for key, label in KEYS:
        vals = [fmt(c[2].get(key, "n/a"), c[3].get(key, "")) for c in cols]
        print(f"| {label} | " + " | ".join(vals) + " |")


def launches(path):
    rows = list(csv.reader(open(path)))
    hi = [i for i, r in enumerate(rows) if "Kernel Name" in r][0]
    h = rows[hi]
    ki, vi, ui = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
    agg = collections.defaultdict(lambda: [0, 0.0])
    for r in rows[hi + 1:]:
        if len(r) <= vi:
            continue
        name = r[ki].split("(")[0]
        v = float(r[vi].replace(",", ""))
        v = v / 1e3 if r[ui] == "ns" else (v * 1e3 if r[ui] == "ms" else v)  # -> us
        agg[name][0] += 1
        agg[name][1] += v
    tot = sum(a[1] for a in agg.values())
    print("| kernel | launches | total us | share |")
    print("|---|---|---|---|")
    for k, (n, t) in sorted(agg.items(), key=lambda x: -x[1][1]):
        print(f"| `{k}` | {n} | {t:.1f} | {100 * t / tot:.1f}% |")


if __name__ == "__main__":
    if sys.argv[1] == "--launches":
        launches(sys.argv[2])
    else:
        summarize(sys.argv[1:])
