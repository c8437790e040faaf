#!/usr/bin/env python3
"""Top source lines of an ncu capture by warp-stall samples (cuda,sass view).

  python tools/ncu_lines.py rep.ncu-rep [N]
"""
import csv
import io
import subprocess
import sys


def main():
    rep, n = sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 30
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    agg, fname, hdr = {}, "", None
    for r in rows:
        if r and r[0] == "File Path":
            fname = r[1].split("/")[-1]
            continue
        if r and r[0] == "Line No":
            hdr = r
            continue
        if hdr is None or len(r) < len(hdr) or not r[0].isdigit():
            continue
        s = int(r[4] or 0) if r[4].isdigit() else 0
        ins = int(r[7] or 0) if r[7].isdigit() else 0
        key = (fname, int(r[0]))
        a = agg.setdefault(key, [0, 0, r[1].strip()[:100]])
        a[0] += s
        a[1] += ins
    tot = sum(v[0] for v in agg.values()) or 1
    toti = sum(v[1] for v in agg.values()) or 1
    print(f"| stall % | instr % | line | source |\n|---|---|---|---|")
    for (f, ln), (s, i, src) in sorted(agg.items(), key=lambda kv: -kv[1][0])[:n]:
        print(f"| {100 * s / tot:.1f} | {100 * i / toti:.1f} | {f}:{ln} | `{src}` |")


if __name__ == "__main__":
    main()
