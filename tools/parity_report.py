#!/usr/bin/env python3
"""GPU parity report (run on the B200 box): how close each device mode is to
the reference, per evaluation, per local search and per LGA run.

Writes gpurun_out/parity_report.json (copied to profiles/ by hand).  The CPU
side is the plain-C restatement (oracle/liboracle.so, bit-identical to the
reference library — tests/test_oracle.py).
"""
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from oracle.oracle import Oracle  # noqa: E402
from paper_2410_10447_b200 import (  # noqa: E402
    BASELINE,
    HALF,
    PAIR_FP32,
    PAIR_FP64,
    PAIR_FP64_FAST,
    SINGLE,
    TCU,
    TCU_SPLIT,
    Device,
    LgaSettings,
)
from paper_2410_10447_b200._abi import Instance, derive_rng, random_instance, random_pose  # noqa: E402


def bits(x):
    return np.asarray(x, np.float32).view(np.uint32)


def load_instances():
    with open(os.path.join(ROOT, "tests", "golden", "instances.json")) as f:
        raw = json.load(f)
    return {k: Instance(np.array(v["atoms"]), np.array(v["torsion"]), np.array(v["sites"]), v["n_rot"], k)
            for k, v in raw.items()}


def main():
    port = Oracle("port")
    insts = load_instances()
    rng = derive_rng(31337, "parity/report")
    cases = []
    for rep in range(60):
        inst = random_instance(rng, rep % 9, 1 + rng.next_index(100), 1 + rng.next_index(64))
        cases.append((inst, np.stack([random_pose(rng, inst.n_rot, 0.5 if k % 2 else 1.5) for k in range(20)])))
    out = {"per_eval": {}, "local_search": {}, "lga": {}}
    ref_cache, ls_cache, lga_cache = {}, {}, {}
    for inst_i, (inst, poses) in enumerate(cases):
        ref_cache[inst_i] = [port.score(inst, p, BASELINE, SINGLE, 128) for p in poses]
    for pair, pname in ((PAIR_FP64, "fp64"), (PAIR_FP64_FAST, "fp64fast"), (PAIR_FP32, "fp32")):
        dev = Device(0, pair=pair)
        for method, mname in ((BASELINE, "baseline"), (TCU_SPLIT, "split")):
            exact = total = 0
            worst_e = worst_g = 0.0
            for inst_i, (inst, poses) in enumerate(cases):
                e, g, t, _ = dev.score_batch(inst, poses, method, SINGLE, 128)
                for k, (we, wg, wt, _) in enumerate(ref_cache[inst_i]):
                    total += 1
                    exact += bool(bits(e[k]) == bits(we) and np.array_equal(bits(g[k]), bits(wg)))
                    worst_e = max(worst_e, abs(float(e[k]) - float(we)) / max(abs(float(we)), 1.0))
                    worst_g = max(worst_g, float(np.abs(g[k] - wg).max()) / max(float(np.abs(wg).max()), 1.0))
            out["per_eval"][f"{pname}/{mname}"] = {"evals": total, "bit_exact_fraction": exact / total,
                                                   "max_rel_err_energy": worst_e, "max_rel_err_grad": worst_g}
            print(pname, mname, out["per_eval"][f"{pname}/{mname}"], flush=True)
        # local searches on the C3 ligand and the bundled s3
        for name in ("synth20", "s3"):
            inst = insts[name]
            if name not in ls_cache:
                lr = derive_rng(7, "parity/ls/" + name)
                st = np.stack([random_pose(lr, inst.n_rot, 0.6) for _ in range(64)])
                ls_cache[name] = (st, [port.local_search(inst, x, 150, 1e-4, BASELINE, SINGLE, 64) for x in st])
            starts, refs = ls_cache[name]
            res = dev.local_search_batch(inst, starts, 150, 1e-4, BASELINE, SINGLE, 64)
            same = close = 0
            for s, r, w in zip(starts, res, refs):
                same += r.energy == w["energy"] and r.iterations == w["iterations"]
                close += abs(r.energy - w["energy"]) <= 1e-4 * max(abs(w["energy"]), 1.0)
            out["local_search"][f"{pname}/{name}"] = {"searches": 64, "identical_trajectory": same,
                                                      "final_energy_within_1e-4": close}
            print(pname, name, out["local_search"][f"{pname}/{name}"], flush=True)
        # full LGA runs, paired seeds
        for name in ("s2", "synth20"):
            inst = insts[name]
            s = LgaSettings()
            seeds = np.arange(40, dtype=np.uint64) + np.uint64(4242)
            gpu = dev.lga_run_batch(inst, BASELINE, SINGLE, s, seeds)
            if name not in lga_cache:
                lga_cache[name] = [port.lga_run(inst, BASELINE, SINGLE, s, int(x)) for x in seeds]
            cpu = lga_cache[name]
            same = sum(g.best_energy == c["best_energy"] and g.evaluations == c["evaluations"] for g, c in zip(gpu, cpu))
            mg = float(np.mean([g.best_energy for g in gpu]))
            mc = float(np.mean([c["best_energy"] for c in cpu]))
            out["lga"][f"{pname}/{name}"] = {"runs": 40, "identical_runs": same, "mean_best_gpu": mg,
                                             "mean_best_cpu": mc, "rel_diff_means": abs(mg - mc) / abs(mc)}
            print(pname, name, out["lga"][f"{pname}/{name}"], flush=True)
        dev.close()
    os.makedirs(os.path.join(ROOT, "gpurun_out"), exist_ok=True)
    with open(os.path.join(ROOT, "gpurun_out", os.environ.get("PARITY_OUT", "parity_report.json")), "w") as f:
        json.dump(out, f, indent=1)


if __name__ == "__main__":
    main()
