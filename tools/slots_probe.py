#!/usr/bin/env python3
"""C3 docking rate per concurrent search at 7 vs 6 searches per SM: 100 runs
(900 searches per generation -> 129 CTAs x 7 slots) against 88 runs (792 ->
132 x 6).  Proxy for what spreading the searches over more SMs would buy."""
import ctypes as C
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import torch

    import bench
    from paper_2410_10447_b200 import SINGLE, Device, LgaSettings
    from paper_2410_10447_b200._lib import load

    lib = load()
    dev = Device(0)
    s = torch.cuda.Stream()
    torch.cuda.set_stream(s)
    dev.set_stream(s.cuda_stream)
    inst = bench.workload()
    st = LgaSettings()
    di = lib.mdr_instance_upload(dev.ctx, C.byref(inst.c()))
    out = {}
    for runs in [int(x) for x in sys.argv[1:]] or (100, 88, 74):
        b = lib.mdr_lga_batch_create(dev.ctx, di, bench.METHODS["baseline"], SINGLE, C.byref(st), runs)
        seeds = torch.from_numpy(bench.run_seeds(0)[:runs].view(np.int64)).cuda()
        tot = torch.zeros(1, dtype=torch.int64, device="cuda")
        for _ in range(3):
            lib.mdr_lga_batch_run_dev(dev.ctx, b, C.c_void_p(seeds.data_ptr()))
        lib.mdr_lga_batch_total_evals_dev(dev.ctx, b, C.c_void_p(tot.data_ptr()))
        torch.cuda.synchronize()
        ev = int(tot.item())
        ms = []
        for _ in range(15):
            a, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(s)
            lib.mdr_lga_batch_run_dev(dev.ctx, b, C.c_void_p(seeds.data_ptr()))
            e.record(s)
            e.synchronize()
            ms.append(a.elapsed_time(e))
        med = sorted(ms)[7]
        out[runs] = {"evals_per_s": ev / (med * 1e-3), "ms": med, "evals": ev,
                     "evals_per_s_per_search": ev / (med * 1e-3) / (9 * runs)}
        print(runs, out[runs], flush=True)
    os.makedirs(os.path.join(ROOT, "gpurun_out"), exist_ok=True)
    json.dump(out, open(os.path.join(ROOT, "gpurun_out", "slots_probe.json"), "w"), indent=1)


if __name__ == "__main__":
    main()
