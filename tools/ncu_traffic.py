#!/usr/bin/env python3
"""DRAM traffic per launch of one ncu --set full capture, as JSON for
bench.py's roofline "traffic" field (run on the box right after the capture).

  python tools/ncu_traffic.py rep.ncu-rep > profiles/r1_ls_kernel_traffic.json
"""
import json
import sys

from ncu_summary import raw

SCALE = {"byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}


def main():
    rows = raw(sys.argv[1])
    d, u = rows[0]
    b = 0.0
    for key in ("dram__bytes_read.sum", "dram__bytes_write.sum"):
        b += float(d[key].replace(",", "")) * SCALE[u[key]]
    print(json.dumps({"kernel": d.get("Kernel Name"), "dram_bytes_per_launch": b,
                      "duration": d.get("gpu__time_duration.sum") + " " + u.get("gpu__time_duration.sum", ""),
                      "source": sys.argv[1].split("/")[-1]}, indent=1))


if __name__ == "__main__":
    main()
