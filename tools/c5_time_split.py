import os, sys, time
sys.path.insert(0, os.getcwd())
import numpy as np, torch
import bench
from paper_2410_10447_b200 import Device, LgaSettings
from paper_2410_10447_b200 import screen as sc
from paper_2410_10447_b200.workloads import c4_receptor, c5_ligand
sites, fields, grid = c4_receptor()
dev = Device(0)
dg = dev.grid_build(sites, fields, grid)
s = LgaSettings(partition=64)
n = 4096
t0 = time.perf_counter(); ligs = [c5_ligand(j, sites) for j in range(n)]; print("gen", time.perf_counter() - t0)
orig = dev.grid_screen_batch
acc = {"call": 0.0}
def timed(*a, **k):
    t = time.perf_counter(); r = orig(*a, **k); acc["call"] += time.perf_counter() - t; return r
dev.grid_screen_batch = timed
sc.screen(dev, dg, lambda j: ligs[j], 2048, 10, s, 0, batch=1024)
acc["call"] = 0.0
t0 = time.perf_counter()
sc.screen(dev, dg, lambda j: ligs[j], n, 10, s, 0, batch=1024)
tot = time.perf_counter() - t0
print("total", tot, "in grid_screen_batch", acc["call"], "lig/h", n / tot * 3600)
