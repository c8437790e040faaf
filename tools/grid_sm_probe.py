import ctypes as C, sys, os, json
sys.path.insert(0, os.getcwd())
import numpy as np, torch
from paper_2410_10447_b200 import Device, BASELINE
from paper_2410_10447_b200.workloads import c4
inst, params, fields, grid, s = c4()
d = Device(0); lib = d.lib
dg = d.grid_build(inst, fields, grid)
sm = (C.c_uint32 * 256)()
seeds = np.arange(100, dtype=np.uint64) + 2000000
d.grid_lga_run_batch(dg, inst, params, BASELINE, s, seeds)
lib.mdr_phase_prof_sm(sm, 1)
d.grid_lga_run_batch(dg, inst, params, BASELINE, s, seeds)
lib.mdr_phase_prof_sm(sm, 1)
v = list(sm)[:148]
h = {}
for x in v: h[x] = h.get(x, 0) + 1
print("per-SM grid LS CTAs over a docking (20 gens):", sorted(h.items()))
