"""Native multi-GPU host driver (csrc/multi.cpp): one host thread and one
context per listed device.  On a one-GPU box device 0 is listed twice, which
exercises the threading, sharding, work queue and the gather; results must be
identical to single-device calls with the same seeds."""
import numpy as np
import pytest

from paper_2410_10447_b200 import BASELINE, SINGLE
from paper_2410_10447_b200._abi import LgaSettings, centered_grid
from paper_2410_10447_b200.api import multi_lga_run_batch, multi_screen

pytestmark = pytest.mark.gpu


def test_multi_lga_equals_single_device(dev, instances):
    inst = instances["s3"]
    s = LgaSettings(generations=4)
    seeds = np.arange(11, dtype=np.uint64) + 500
    be, bg, ev, cv = multi_lga_run_batch([0, 0, 0], inst, BASELINE, SINGLE, s, seeds)
    one = dev.lga_run_batch(inst, BASELINE, SINGLE, s, seeds)
    assert np.array_equal(be, [r.best_energy for r in one])
    assert np.array_equal(ev, [r.evaluations for r in one])
    assert np.array_equal(bg, np.stack([r.best_genotype for r in one]))


def test_multi_screen_equals_single_device(dev):
    from paper_2410_10447_b200.workloads import c4_receptor, c5_ligand

    sites, fields, _ = c4_receptor()
    grid = centered_grid(41, 0.375, 4)
    ligs, params = zip(*[c5_ligand(j, sites) for j in range(10)])
    runs = 3
    s = LgaSettings(generations=2, partition=64)
    seeds = np.arange(10 * runs, dtype=np.uint64) + 9000
    be, bg, ev, cl, nc, dol = multi_screen([0, 0], sites, fields, grid, list(ligs), list(params), runs, BASELINE, s,
                                           seeds, 2.0, batch_ligands=3)
    assert set(dol.tolist()) <= {0, 1} and (dol >= 0).all()
    dg = dev.grid_build(sites, fields, grid)
    ref = dev.grid_screen_batch(dg, list(ligs), list(params), runs, BASELINE, s, seeds, 2.0)
    assert np.array_equal(be, np.concatenate([r["best_energy"] for r in ref]))
    assert np.array_equal(ev, np.concatenate([r["evaluations"] for r in ref]))
    assert np.array_equal(cl, np.concatenate([r["cluster_of"] for r in ref]))
    assert np.array_equal(nc, [r["n_clusters"] for r in ref])
    assert np.array_equal(bg, np.concatenate([r["best_genotype"].ravel() for r in ref]))


def test_multi_screen_requeues_a_failed_device(dev):
    """Fault injection: device index 1 fails on its first batch;
    its batch is re-queued, device 0 docks everything, results unchanged."""
    from paper_2410_10447_b200 import _lib
    from paper_2410_10447_b200.workloads import c4_receptor, c5_ligand

    lib = _lib.load()
    sites, fields, _ = c4_receptor()
    grid = centered_grid(33, 0.375, 4)
    ligs, params = zip(*[c5_ligand(j, sites) for j in range(8)])
    s = LgaSettings(generations=1, partition=64)
    seeds = np.arange(16, dtype=np.uint64) + 31
    ref = multi_screen([0], sites, fields, grid, list(ligs), list(params), 2, BASELINE, s, seeds, 2.0,
                       batch_ligands=2)
    lib.mdr_multi_set_fault_injection(1, 0)
    try:
        got = multi_screen([0, 0], sites, fields, grid, list(ligs), list(params), 2, BASELINE, s, seeds, 2.0,
                           batch_ligands=2)
    finally:
        lib.mdr_multi_set_fault_injection(-1, 0)
    assert np.all(got[5] == 0)  # every ligand docked by the surviving device
    for a, b in zip(ref[:5], got[:5]):
        assert np.array_equal(a, b)
    lib.mdr_multi_set_fault_injection(0, 0)
    try:
        with pytest.raises(Exception):  # the only device fails: the call fails
            multi_screen([0], sites, fields, grid, list(ligs), list(params), 2, BASELINE, s, seeds, 2.0,
                         batch_ligands=2)
    finally:
        lib.mdr_multi_set_fault_injection(-1, 0)
