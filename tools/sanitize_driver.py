"""Small end-to-end pass over every kernel family, for compute-sanitizer
(memcheck / racecheck / synccheck): analytic score / LS / LGA (all pair
modes, all reduction methods), the LGA's two-warp persistent search and
polish (named-barrier arrive/sync protocol, padded site chunks) and the
other search configurations, grid build / score / LS / LGA / screen,
clustering, reductions (incl. the batched tcgen05 contraction) and the
half/mma units."""
import json, os, sys
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2410_10447_b200 import BASELINE, HALF, PAIR_FP32, PAIR_FP64, PAIR_FP64_FAST, SINGLE, TCU, TCU_SPLIT, Device
from paper_2410_10447_b200._abi import (Instance, LgaSettings, centered_grid, derive_rng, random_instance,
                                        random_ligand_params, random_pose, random_receptor_fields)
from paper_2410_10447_b200.workloads import c4_receptor, c5_ligand

raw = json.load(open("tests/golden/instances.json"))["s3"]
s3 = Instance(np.array(raw["atoms"]), np.array(raw["torsion"]), np.array(raw["sites"]), raw["n_rot"])
small = LgaSettings(generations=2, population_size=8, ls_max_iters=12)
rng = derive_rng(1, "san")
poses = np.stack([random_pose(rng, s3.n_rot, 2.0) for _ in range(6)])
for pair in (PAIR_FP64, PAIR_FP64_FAST, PAIR_FP32):
    dev = Device(0, pair=pair)
    for m, acc in ((BASELINE, SINGLE), (TCU, HALF), (TCU_SPLIT, SINGLE)):
        dev.score_batch(s3, poses, m, acc, 64)
        dev.local_search_batch(s3, poses[:3], 10, 1e-4, m, acc, 64)
        dev.lga_run_batch(s3, m, acc, small, [1, 2])
    dev.score_reference(s3, poses[0])
    dev.close()
dev = Device(0)
dev.reduce4(np.random.default_rng(0).uniform(-1, 1, (128, 4)).astype(np.float32), SINGLE, TCU)
dev.reduce7(np.random.default_rng(1).uniform(-1, 1, (64, 7)).astype(np.float32), TCU_SPLIT, SINGLE)
dev.block_reduce(np.arange(256, dtype=np.float32), 256)
c, r, nc = dev.cluster_poses(s3, poses, np.arange(6.0), 1.0)
sites, fields, _ = c4_receptor()
grid = centered_grid(33, 0.375, 4)
dg = dev.grid_build(sites, fields, grid)
lig, prm = c5_ligand(3, sites)
gp = np.stack([random_pose(rng, lig.n_rot, 2.0) for _ in range(4)])
for m in (BASELINE, TCU, TCU_SPLIT):
    dev.grid_score_batch(dg, lig, prm, gp, m, 64)
    dev.grid_local_search_batch(dg, lig, prm, gp[:2], 8, 1e-4, m, 64)
dev.grid_lga_run_batch(dg, lig, prm, BASELINE, LgaSettings(generations=2, population_size=8, ls_max_iters=8,
                                                           partition=64), [5, 6])
ligs, prms = zip(*[c5_ligand(j, sites) for j in range(3)])
dev.grid_screen_batch(dg, list(ligs), list(prms), 2, BASELINE,
                      LgaSettings(generations=1, population_size=6, ls_max_iters=6, partition=64),
                      np.arange(6, dtype=np.uint64), 2.0)
# chunked small ligand: the multi-warp persistent search (ls_multi.cu: pooled and leader + helper), its
# polish, and the one-warp / legacy-pair configurations
from paper_2410_10447_b200.workloads import c3  # noqa: E402

for warps in (3, 2, 1, 0):
    d = Device(0, pair=PAIR_FP64_FAST)
    assert d.lib.mdr_ctx_set_ls_warps(d.ctx, warps) == 0
    for m, acc in ((BASELINE, SINGLE), (TCU_SPLIT, SINGLE)):
        d.lga_run_batch(c3(), m, acc, LgaSettings(generations=2, ls_max_iters=20), [11, 12, 13])
    d.close()
# the pooled search's BIG form (dim 46 > 32: two dimensions per leader lane)
d = Device(0, pair=PAIR_FP64_FAST)
big = random_instance(derive_rng(5, "san/big"), 40, 16, 64)
d.lga_run_batch(big, BASELINE, SINGLE, LgaSettings(generations=2, ls_max_iters=12), [21, 22])
d.close()
# TcuSplit batches routed to tcgen05 (float4 and Partial7 forms, ragged tail)
n_red = 148 * 32 + 5
assert dev.lib.mdr_reduce_uses_tc05(dev.ctx, TCU_SPLIT, 32, n_red) == 1
dev.reduce4_batch(np.random.default_rng(2).uniform(-1, 1, (n_red, 32, 4)).astype(np.float32), SINGLE, TCU_SPLIT)
dev.reduce7_batch(np.random.default_rng(3).uniform(-1, 1, (n_red, 32, 7)).astype(np.float32), TCU_SPLIT, SINGLE)
print("sanitize driver done")
