#!/usr/bin/env python3
"""Grid-mode parity at scale (SURVEY §8c protocol (2) for the f1 path): the
C4 workload at full size — the device builds the 126^3 x 6 maps, the oracle
scores the downloaded copy, so both sides see identical inputs — docked with
N paired seeds on the device (FP32) and by the double-precision oracle
(orc_grid_lga_run, one process per host core).  Reports the paired-seed
mean-best difference, the best energies and the 2 A clustering of the final
poses.  Writes gpurun_out/grid_parity_scale.json.

GRID_STRICT=1: the device runs the strict FP64 grid path (context pair
precision MDR_PAIR_FP64: the oracle's double arithmetic and order, correctly
rounded trig on both sides) and the report counts runs identical to the
oracle (best energy and evaluation count) and times the device docking.
"""
import json
import multiprocessing as mp
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
N = int(os.environ.get("GRID_PARITY_RUNS", "32"))
BASE = 515000
_G = {}


def _cpu(seed):
    from oracle.oracle import Oracle

    inst, params, grid, s = _G["case"]
    r = Oracle("port").grid_lga_run(inst, grid, params, s, int(seed))
    return seed, r["best_energy"], r["evaluations"], r["best_genotype"].tolist()


def main():
    from oracle.oracle import Oracle
    from paper_2410_10447_b200 import BASELINE, Device
    from paper_2410_10447_b200._abi import Grid
    from paper_2410_10447_b200.workloads import c4

    from paper_2410_10447_b200 import PAIR_FP32, PAIR_FP64

    strict = os.environ.get("GRID_STRICT") == "1"
    inst, params, fields, grid, s = c4()
    dev = Device(0, pair=PAIR_FP64 if strict else PAIR_FP32)
    dg = dev.grid_build(inst, fields, grid)
    G = Grid(grid.shape, grid.n_types, grid.origin, grid.spacing, dg.download())
    _G["case"] = (inst, params, G, s)
    seeds = np.arange(N, dtype=np.uint64) + np.uint64(BASE)
    import time

    gpu = dev.grid_lga_run_batch(dg, inst, params, BASELINE, s, seeds)
    t0 = time.perf_counter()
    gpu = dev.grid_lga_run_batch(dg, inst, params, BASELINE, s, seeds)
    dt = time.perf_counter() - t0
    with mp.get_context("fork").Pool(os.cpu_count()) as pool:
        cpu = sorted(pool.map(_cpu, [int(x) for x in seeds]))
    ge = np.array([r.best_energy for r in gpu])
    ce = np.array([c[1] for c in cpu])
    port = Oracle("port")
    gc, _, gn = dev.cluster_poses(inst, np.stack([r.best_genotype for r in gpu]), ge, 2.0)
    cc, _, cn = port.cluster_poses(inst, np.stack([np.array(c[3]) for c in cpu]), ce, 2.0)
    out = {"workload": "C4 (100 atoms / 30 torsions, 126^3 x 6 maps, intramolecular on), default LgaSettings, "
                       "partition 64", "runs": N, "base_seed": BASE,
           "mean_best_gpu": float(ge.mean()), "mean_best_oracle": float(ce.mean()),
           "rel_diff_means": float(abs(ge.mean() - ce.mean()) / abs(ce.mean())),
           "best_gpu": float(ge.min()), "best_oracle": float(ce.min()),
           "median_abs_rel_diff_per_seed": float(np.median(np.abs(ge - ce) / np.abs(ce))),
           "std_best_gpu": float(ge.std(ddof=1)), "std_best_oracle": float(ce.std(ddof=1)),
           "diff_of_means_in_standard_errors": float(abs(ge.mean() - ce.mean()) /
                                                     np.sqrt(ge.var(ddof=1) / N + ce.var(ddof=1) / N)),
           "clusters_gpu": int(gn), "clusters_oracle": int(cn),
           "clusters_identical": bool(gn == cn and np.array_equal(gc, cc)),
           "identical_runs": int(sum(g.best_energy == c[1] and g.evaluations == c[2] for g, c in zip(gpu, cpu))),
           "device_mode": "strict FP64 (MDR_PAIR_FP64)" if strict else "FP32 grid path",
           "device_evals_per_s": float(sum(r.evaluations for r in gpu) / dt),
           "evals_gpu_mean": float(np.mean([r.evaluations for r in gpu])),
           "evals_oracle_mean": float(np.mean([c[2] for c in cpu]))}
    print(json.dumps(out, indent=1))
    os.makedirs(os.path.join(ROOT, "gpurun_out"), exist_ok=True)
    with open(os.path.join(ROOT, "gpurun_out", os.environ.get("GRID_PARITY_OUT", "grid_parity_scale.json")), "w") as f:
        json.dump(out, f, indent=1)


if __name__ == "__main__":
    main()
