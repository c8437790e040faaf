"""Split one C5 screen batch into host preparation vs device time."""
import json, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
from paper_2410_10447_b200 import BASELINE, Device
from paper_2410_10447_b200._abi import LgaSettings
from paper_2410_10447_b200.workloads import c4_receptor, c5_ligand

torch.cuda.set_device(0)
dev = Device(0)
sites, fields, grid = c4_receptor()
dg = dev.grid_build(sites, fields, grid)
n = int(sys.argv[1]) if len(sys.argv) > 1 else 256
t0 = time.perf_counter()
ligs, prms = zip(*[c5_ligand(j, sites) for j in range(n)])
t1 = time.perf_counter()
s = LgaSettings(partition=64)
seeds = np.arange(n * 10, dtype=np.uint64)
dev.grid_screen_batch(dg, list(ligs[:8]), list(prms[:8]), 10, BASELINE, LgaSettings(partition=64, generations=1), seeds[:80])
torch.cuda.synchronize()
t2 = time.perf_counter()
res = dev.grid_screen_batch(dg, list(ligs), list(prms), 10, BASELINE, s, seeds)
t3 = time.perf_counter()
ev = sum(int(r["evaluations"].sum()) for r in res)
print(json.dumps({"ligands": n, "python_ligand_gen_s": t1 - t0, "screen_call_s": t3 - t2,
                  "ligands_per_hour_call": n / (t3 - t2) * 3600, "evals_per_s": ev / (t3 - t2),
                  "mean_atoms": float(np.mean([l.n_atoms for l in ligs])),
                  "mean_rot": float(np.mean([l.n_rot for l in ligs]))}))
