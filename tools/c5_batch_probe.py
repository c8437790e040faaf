#!/usr/bin/env python3
"""C5 screening throughput vs ligands per mdr_grid_screen_batch call."""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import torch

    import bench

    s = torch.cuda.Stream()
    torch.cuda.set_stream(s)
    n = int(os.environ.get("C5_N", "2048"))
    out = {}
    for b in [int(x) for x in sys.argv[1:]] or [256, 512, 1024]:
        r = bench.c5_measure(torch, 0, n_ligands=n, batch=b)
        out[b] = {"ligands_per_hour": r["ligands_per_hour"], "seconds": r["seconds"]}
        print(b, out[b], flush=True)
    with open(os.path.join(ROOT, "gpurun_out", "c5_batch_probe.json"), "w") as f:
        json.dump(out, f, indent=1)


if __name__ == "__main__":
    main()
