#!/usr/bin/env python3
"""Paired-seed parity at scale (reference acceptance.cpp:128-145 methodology,
SURVEY §8c protocol (2)): 100 LGA runs per instance (bundled s1/s2/s3 and the
C3 ligand) with default LgaSettings, every device mode against the reference
library (oracle/_ref, one process per host core), plus the RMSD clustering of
the 100 final poses (2 A) on both sides.  Writes gpurun_out/parity_scale.json.
"""
import json
import multiprocessing as mp
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

N_RUNS = 100
BASE = 777000


def _instances():
    from paper_2410_10447_b200._abi import Instance
    from paper_2410_10447_b200.workloads import c3

    raw = json.load(open(os.path.join(ROOT, "tests", "golden", "instances.json")))
    out = {k: Instance(np.array(v["atoms"]), np.array(v["torsion"]), np.array(v["sites"]), v["n_rot"], k)
           for k, v in raw.items() if k in ("s1", "s2", "s3")}
    out["c3"] = c3()
    return out


def _cpu(args):
    name, method, accum, seed = args
    from oracle.oracle import Oracle, available
    from paper_2410_10447_b200._abi import LgaSettings

    o = Oracle("reference" if available("reference") else "port")
    r = o.lga_run(_instances()[name], method, accum, LgaSettings(), seed)
    return name, method, accum, seed, r["best_energy"], r["evaluations"], r["converged"], r["best_genotype"].tolist()


def main():
    from oracle.oracle import Oracle
    from paper_2410_10447_b200 import BASELINE, HALF, PAIR_FP32, PAIR_FP64, PAIR_FP64_FAST, SINGLE, TCU, Device
    from paper_2410_10447_b200._abi import LgaSettings

    insts = _instances()
    seeds = [BASE + i for i in range(N_RUNS)]
    jobs = [(n, m, a, sd) for n in insts for (m, a) in ((BASELINE, SINGLE), (TCU, HALF)) for sd in seeds]
    with mp.get_context("fork").Pool(os.cpu_count()) as pool:
        cpu = {(n, m, a, sd): (e, ev, cv, np.array(g)) for n, m, a, sd, e, ev, cv, g in pool.map(_cpu, jobs)}
    port = Oracle("port")
    report = {"n_runs": N_RUNS, "base_seed": BASE, "cpu_reference": "oracle/_ref (the reference library)",
              "results": {}}
    modes = [("fp64", PAIR_FP64, BASELINE, SINGLE), ("fp64fast", PAIR_FP64_FAST, BASELINE, SINGLE),
             ("fp32", PAIR_FP32, BASELINE, SINGLE), ("fp64fast/tcu-half", PAIR_FP64_FAST, TCU, HALF)]
    only = os.environ.get("PARITY_MODES")  # e.g. "fp64fast" (comma separated)
    if only:
        modes = [m for m in modes if m[0] in only.split(",")]
    for mname, pair, method, accum in modes:
        dev = Device(0, pair=pair)
        for name, inst in insts.items():
            gpu = dev.lga_run_batch(inst, method, accum, LgaSettings(), seeds)
            ref = [cpu[(name, method, accum, sd)] for sd in seeds]
            ge = np.array([r.best_energy for r in gpu])
            ce = np.array([r[0] for r in ref])
            same = int(sum(g.best_energy == r[0] and g.evaluations == r[1] for g, r in zip(gpu, ref)))
            gnc = float(np.mean([not r.converged for r in gpu]))
            cnc = float(np.mean([not r[2] for r in ref]))
            # clustering of the final poses (device) vs the oracle clustering of the reference's poses
            gc, _, gn = dev.cluster_poses(inst, np.stack([r.best_genotype for r in gpu]), ge, 2.0)
            cc, _, cn = port.cluster_poses(inst, np.stack([r[3] for r in ref]), ce, 2.0)
            rec = {"identical_runs": same, "mean_best_gpu": float(ge.mean()), "mean_best_ref": float(ce.mean()),
                   "rel_diff_means": float(abs(ge.mean() - ce.mean()) / abs(ce.mean())),
                   "best_gpu": float(ge.min()), "best_ref": float(ce.min()),
                   "nonconvergent_gpu": gnc, "nonconvergent_ref": cnc,
                   "clusters_gpu": int(gn), "clusters_ref": int(cn),
                   "clusters_identical": bool(gn == cn and np.array_equal(gc, cc))}
            report["results"][f"{mname}/{name}"] = rec
            print(mname, name, rec, flush=True)
        dev.close()
    os.makedirs(os.path.join(ROOT, "gpurun_out"), exist_ok=True)
    with open(os.path.join(ROOT, "gpurun_out", os.environ.get("PARITY_OUT", "parity_scale.json")), "w") as f:
        json.dump(report, f, indent=1)


if __name__ == "__main__":
    main()
