#!/usr/bin/env python3
"""C4 analytic measurement alone (bench.py c4_analytic_measure), with the
reference arm on this host's cores unless --no-cpu."""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import torch

    import bench
    from paper_2410_10447_b200._lib import load

    lib = load()
    s = torch.cuda.Stream()
    torch.cuda.set_stream(s)
    out = bench.c4_analytic_measure(lib, torch, 0, cpu_seconds=0.0 if "--no-cpu" in sys.argv else 12.0)
    print(json.dumps(out, indent=1))
    os.makedirs(os.path.join(ROOT, "gpurun_out"), exist_ok=True)
    with open(os.path.join(ROOT, "gpurun_out", os.environ.get("C4A_OUT", "c4a_probe.json")), "w") as f:
        json.dump(out, f, indent=1)


if __name__ == "__main__":
    main()
