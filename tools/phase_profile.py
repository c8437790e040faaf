#!/usr/bin/env python3
"""Per-phase cycle breakdown of the warp-pair Lamarckian search on the C3
docking (experiment build with -DMDR_PHASE_PROF=1; the numbers are clock64
sums of lane 0 of each warp, per evaluation).

    python -m paper_2410_10447_b200.build --variant prof -DMDR_PHASE_PROF=1
    MDR_LIB_PATH=paper_2410_10447_b200/variants/prof/libmdr_b200.so python tools/phase_profile.py
"""
import ctypes as C
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

NAMES = ["L0 adadelta", "L1 trig+frame+pos", "L2 wait B1", "L3 items", "L4 wait B2", "L5 combine+reduce",
         "L6 project+best", None, "H8 wait B1", "H9 items", "H10 wait B2"]
# ls_multi.cu (default search kernel): L1 = trig, frame, positions and the
# B1 arrive (no wait), L2 unused, H10 = the projection axes (last helper)


def main():
    import torch

    from paper_2410_10447_b200 import BASELINE, SINGLE, Device, LgaSettings
    from paper_2410_10447_b200.workloads import c3

    dev = Device(0)
    lib = dev.lib
    seeds = np.arange(int(os.environ.get("PHASE_RUNS", "100")), dtype=np.uint64) + np.uint64(1_000_000)
    out = (C.c_uint64 * 16)()
    dev.lga_run_batch(c3(), BASELINE, SINGLE, LgaSettings(), seeds)  # warm
    assert lib.mdr_phase_prof(out, 1) == 0, lib.mdr_last_error(None)
    sm = (C.c_uint32 * 256)()
    lib.mdr_phase_prof_sm(sm, 1)
    if os.environ.get("AB_WPB"):
        assert lib.mdr_ctx_set_warps_per_block(dev.ctx, int(os.environ["AB_WPB"])) == 0
    dev.lga_run_batch(c3(), BASELINE, SINGLE, LgaSettings(), seeds)
    assert lib.mdr_phase_prof(out, 1) == 0
    v = list(out)
    lib.mdr_phase_prof_sm(sm, 1)
    per_sm = [x for x in sm][:148]
    ev = v[7]
    rep = {"evals": ev, "searches": v[11], "cycles_per_eval": {}}
    tot = sum(v[k] for k in range(7))
    for k, n in enumerate(NAMES):
        if n:
            rep["cycles_per_eval"][n] = v[k] / ev
    rep["leader_total_per_eval"] = tot / ev
    gens = LgaSettings().generations + 1  # LS launches per docking (generations + polish uses its own kernel)
    hist = {}
    for x in per_sm:
        hist[x] = hist.get(x, 0) + 1
    rep["searches_per_sm_per_docking"] = {"histogram (searches started on an SM over the docking: SM count)": hist,
                                          "max": max(per_sm), "min": min(per_sm), "launches": gens}
    print(json.dumps(rep, indent=1))
    os.makedirs(os.path.join(ROOT, "gpurun_out"), exist_ok=True)
    with open(os.path.join(ROOT, "gpurun_out", os.environ.get("PHASE_OUT", "phase_profile.json")), "w") as f:
        json.dump(rep, f, indent=1)
    torch.cuda.synchronize()


if __name__ == "__main__":
    main()
