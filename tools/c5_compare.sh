cd $GRAFT_REPO_ROOT
timeout 600 python tools/c5_profile.py 256 2>&1 | tail -1
timeout 600 python tools/c5_probe.py 256 2>&1 | grep -E "ligands_per_hour|evals_per_s|seconds"
timeout 600 python - <<'PY'
import sys, time, json
sys.path.insert(0, '.')
import numpy as np, torch
from paper_2410_10447_b200 import BASELINE, Device
from paper_2410_10447_b200 import screen as sc
from paper_2410_10447_b200._abi import LgaSettings
from paper_2410_10447_b200.workloads import c4_receptor, c5_ligand
torch.cuda.set_device(0)
dev = Device(0)
sites, fields, grid = c4_receptor()
dg = dev.grid_build(sites, fields, grid)
ligs = [c5_ligand(j, sites) for j in range(256)]
s = LgaSettings(partition=64)
for seedbase in (0, 12345):
    seeds = np.array([sc.run_seed(seedbase, j, k, 10) for j in range(256) for k in range(10)], np.uint64)
    t = time.perf_counter()
    res = dev.grid_screen_batch(dg, [l for l, _ in ligs], [p for _, p in ligs], 10, BASELINE, s, seeds, 2.0)
    dt = time.perf_counter() - t
    ev = sum(int(r['evaluations'].sum()) for r in res)
    print('seedbase', seedbase, 'lig/h', round(256 / dt * 3600), 'evals/s', round(ev / dt / 1e6, 1), 'evals', ev)
PY
