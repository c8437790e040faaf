"""Measure grid-mode device-vs-oracle error distributions (sets the
tolerances written in tests/test_gpu_grid.py).  Run on the GPU box:
    python tools/grid_probe.py > gpurun_out/grid_probe.json
"""
import json
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from oracle.oracle import Oracle  # noqa: E402
from paper_2410_10447_b200 import BASELINE, TCU, TCU_SPLIT, Device  # noqa: E402
from paper_2410_10447_b200._abi import (  # noqa: E402
    LgaSettings,
    centered_grid,
    derive_rng,
    random_instance,
    random_ligand_params,
    random_pose,
    random_receptor_fields,
)


def main():
    port = Oracle("port")
    dev = Device(0)
    out = {}
    for name, (na, nr, ns, seed, part) in {"small": (20, 5, 16, 7, 64), "large": (100, 30, 64, 8, 128)}.items():
        inst = random_instance(derive_rng(seed, "grid/inst"), nr, na, ns)
        rf = random_receptor_fields(derive_rng(seed, "grid/rec"), ns, 4)
        lp = random_ligand_params(derive_rng(seed, "grid/lig"), na, 4)
        G = centered_grid(41, 0.375, 4)
        G.maps = port.grid_build(inst, rf, G)
        dg = dev.grid_upload(G)
        rng = derive_rng(1, "grid/poses")
        poses = np.stack([random_pose(rng, nr, 3.0 if k % 4 else 8.0) for k in range(64)])
        rec = {}
        for mname, m in (("baseline", BASELINE), ("split", TCU_SPLIT), ("tcu", TCU)):
            e, g, _ = dev.grid_score_batch(dg, inst, lp, poses, m, part)
            er, gr = [], []
            for i, p in enumerate(poses):
                we, wg, _, _ = port.grid_score(inst, G, lp, p)
                er.append(abs(e[i] - we) / max(1.0, abs(we)))
                gr.append(np.abs(g[i] - wg).max() / max(1.0, np.abs(wg).max()))
            rec[mname] = dict(e_rel_max=float(max(er)), e_rel_med=float(np.median(er)), g_rel_max=float(max(gr)),
                              g_rel_med=float(np.median(gr)))
        starts = poses[:16]
        res = dev.grid_local_search_batch(dg, inst, lp, starts, 150, 1e-4, BASELINE, part)
        ls = []
        for s, r in zip(starts, res):
            w = port.grid_local_search(inst, G, lp, s, 150, 1e-4)
            ls.append(dict(gpu=r.energy, cpu=w["energy"], it_gpu=r.iterations, it_cpu=w["iterations"]))
        rec["local_search"] = ls
        if name == "small":
            s = LgaSettings(generations=6)
            seeds = np.arange(8, dtype=np.uint64) + 1000
            gpu = dev.grid_lga_run_batch(dg, inst, lp, BASELINE, s, seeds)
            cpu = [port.grid_lga_run(inst, G, lp, s, int(x)) for x in seeds]
            rec["lga"] = [dict(gpu=a.best_energy, cpu=b["best_energy"], ev_gpu=a.evaluations, ev_cpu=b["evaluations"])
                          for a, b in zip(gpu, cpu)]
        out[name] = rec
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
