"""Regenerate tests/golden/*.json from the REFERENCE ITSELF.

Run here (where /root/reference exists):  python tests/golden/make_golden.py
It parses the bundled ligand files with the reference's own parse_instance and
records outputs of the reference library compiled in place by oracle/Makefile
(oracle/_ref/libmdr_ref.so).  The JSON fixtures travel to the GPU box; nothing
there reads /root/reference.
"""
from __future__ import annotations

import ctypes as C
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)

from oracle.oracle import Oracle, build  # noqa: E402
from paper_2410_10447_b200._abi import (  # noqa: E402
    BASELINE,
    HALF,
    SINGLE,
    TCU,
    Instance,
    LgaSettings,
    derive_rng,
    random_instance,
    random_pose,
)

DATA = "/root/reference/proj/data"
OUT = os.path.dirname(os.path.abspath(__file__))


def parse_with_reference(lib, text: str) -> Instance:
    cap = 4096
    na, ns, nr, el = C.c_int32(), C.c_int32(), C.c_int32(), C.c_int32()
    atoms = np.zeros(cap * 4)
    tors = np.zeros(cap, np.int32)
    sites = np.zeros(cap * 5)
    rc = lib.ref_parse_instance(text.encode(), cap, cap, C.byref(na), C.byref(ns), C.byref(nr),
                                atoms.ctypes.data_as(C.POINTER(C.c_double)),
                                tors.ctypes.data_as(C.POINTER(C.c_int32)),
                                sites.ctypes.data_as(C.POINTER(C.c_double)), C.byref(el))
    assert rc == 0, (rc, el.value)
    return Instance(atoms[: 4 * na.value].reshape(-1, 4), tors[: na.value],
                    sites[: 5 * ns.value].reshape(-1, 5), nr.value)


def inst_json(inst: Instance) -> dict:
    return dict(atoms=inst.atoms.tolist(), torsion=inst.torsion.tolist(), sites=inst.sites.tolist(),
                n_rot=inst.n_rot)


def main() -> None:
    build()
    ref = Oracle("reference")
    insts = {}
    for name in ("s1", "s2", "s3"):
        with open(os.path.join(DATA, name + ".mdri")) as f:
            insts[name] = parse_with_reference(ref.lib, f.read())
    insts["synth7"] = random_instance(derive_rng(6002, "dock-fd"), 3, 7, 4)
    insts["synth20"] = random_instance(derive_rng(12345, "synth/small"), 5, 20, 64)
    with open(os.path.join(OUT, "instances.json"), "w") as f:
        json.dump({k: inst_json(v) for k, v in insts.items()}, f)

    vec: dict = {}
    vec["rng_golden_42"] = [int(x) for x in ref.rng_draws(42, "golden", 10)]
    vec["normals_12345_lga"] = ref.rng_normals(12345, "lga", 16).tolist()

    # score: poses near the binding region (spread 0.35 / 0.6) and far field
    score_cases = []
    for name, inst in insts.items():
        rng = derive_rng(777, "golden/score/" + name)
        for rep in range(6):
            g = random_pose(rng, inst.n_rot, 0.35 if rep < 3 else 1.5)
            for method, accum in ((BASELINE, SINGLE), (TCU, HALF), (TCU, SINGLE)):
                e, grad, tq, st = ref.score(inst, g, method, accum, 64)
                score_cases.append(dict(inst=name, g=g.tolist(), method=method, accum=accum,
                                        partition=64, energy=float(e), grad=grad.astype(float).tolist(),
                                        torque=tq.astype(float).tolist(), stats=list(st.as_tuple())))
            er, gr, tr = ref.score_reference(inst, g)
            score_cases.append(dict(inst=name, g=g.tolist(), method="reference", energy=er,
                                    grad=gr.tolist(), torque=tr.tolist()))
    vec["score"] = score_cases

    ls_cases = []
    for name in ("s1", "s2", "s3", "synth7"):
        inst = insts[name]
        rng = derive_rng(778, "golden/ls/" + name)
        for rep in range(2):
            g = random_pose(rng, inst.n_rot, 0.6)
            for method, accum in ((BASELINE, SINGLE), (TCU, HALF)):
                r = ref.local_search(inst, g, 150, 1e-4, method, accum, 64)
                ls_cases.append(dict(inst=name, start=g.tolist(), method=method, accum=accum,
                                     max_iters=150, tol=1e-4, genotype=r["genotype"].tolist(),
                                     energy=r["energy"], iterations=r["iterations"],
                                     converged=r["converged"]))
    vec["local_search"] = ls_cases

    lga_cases = []
    small = dict(population_size=8, generations=2, ls_max_iters=30)
    for name, seed, method, accum, kw in (
        ("s1", 4242, TCU, HALF, small),
        ("s1", 99, BASELINE, SINGLE, dict(population_size=2, generations=1, mutation_sigma=0.0,
                                          ls_fraction=1.0, ls_max_iters=60)),
        ("s1", 7, BASELINE, SINGLE, dict(population_size=6, generations=50, max_evaluations=200,
                                         ls_max_iters=40)),
        ("s2", 20260816, TCU, HALF, {}),
        ("s2", 12345, BASELINE, SINGLE, {}),
        ("s3", 12346, BASELINE, SINGLE, {}),
    ):
        s = LgaSettings(**kw)
        r = ref.lga_run(insts[name], method, accum, s, seed)
        lga_cases.append(dict(inst=name, seed=seed, method=method, accum=accum, settings=kw,
                              best_energy=r["best_energy"], best_genotype=r["best_genotype"].tolist(),
                              evaluations=r["evaluations"], converged=r["converged"],
                              runs=[list(x) for x in r["runs"]],
                              total_stats=list(r["total_stats"].as_tuple())))
    vec["lga_run"] = lga_cases
    with open(os.path.join(OUT, "ref_vectors.json"), "w") as f:
        json.dump(vec, f)
    print("wrote", len(score_cases), "score,", len(ls_cases), "ls,", len(lga_cases), "lga cases")


if __name__ == "__main__":
    main()
