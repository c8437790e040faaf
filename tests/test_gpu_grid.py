"""Grid-map scoring mode on the B200 against the CPU oracle
(oracle/mdr_oracle.c orc_grid_*, pinned by tests/test_grid_oracle.py).

Tolerances (the device computes in FP32 on FP32 maps, the oracle in double):
  * map builder: <= 2 float ulps per value (FP64 on both sides; exp() of
    libdevice vs glibc may differ by one double ulp before the float rounding);
  * energy: |E_gpu - E_orc| <= 1e-5 * max(1, |E|)  (measured max 1.0e-6,
    tools/grid_probe.py, profiles/r1_grid_probe.json);
  * gradient: max_d |g_gpu - g_orc| <= 2e-5 * max(1, max_d |g_orc|)
    (measured max 1.6e-6);
  * Tcu (paper f16 MMA reduction): 5e-3 relative (f16 rounding of every
    partial, SURVEY §0 "Measured precision facts");
  * local search / LGA: trajectories diverge once FP32 rounding flips a
    comparison, so final energies are compared statistically (paired starts /
    seeds): median relative difference <= 1e-3 and mean within 2 %.
"""
import numpy as np
import pytest

from paper_2410_10447_b200 import BASELINE, TCU, TCU_SPLIT
from paper_2410_10447_b200._abi import (
    Instance,
    LgaSettings,
    LigandParams,
    SizeError,
    UnsupportedBlockSizeError,
    centered_grid,
    derive_rng,
    random_instance,
    random_ligand_params,
    random_pose,
    random_receptor_fields,
)

pytestmark = pytest.mark.gpu


def _case(n_atoms, n_rot, n_sites=16, n=41, spacing=0.375, n_types=4, seed=7):
    inst = random_instance(derive_rng(seed, "grid/inst"), n_rot, n_atoms, n_sites)
    rf = random_receptor_fields(derive_rng(seed, "grid/rec"), n_sites, n_types)
    lp = random_ligand_params(derive_rng(seed, "grid/lig"), n_atoms, n_types)
    return inst, rf, lp, centered_grid(n, spacing, n_types)


@pytest.fixture(scope="module")
def small(port, dev):
    inst, rf, lp, G = _case(20, 5)
    G.maps = port.grid_build(inst, rf, G)
    return inst, lp, G, dev.grid_upload(G)


@pytest.fixture(scope="module")
def large(port, dev):
    inst, rf, lp, G = _case(100, 30, n_sites=64, seed=8)
    G.maps = port.grid_build(inst, rf, G)
    return inst, lp, G, dev.grid_upload(G)


def _poses(inst, n, seed, spread=3.0):
    rng = derive_rng(seed, "grid/poses")
    return np.stack([random_pose(rng, inst.n_rot, spread if k % 4 else 8.0) for k in range(n)])


def test_grid_build_matches_oracle(port, dev):
    inst, rf, lp, G = _case(20, 5, n=33, spacing=0.5)
    want = port.grid_build(inst, rf, G)
    got = dev.grid_build(inst, rf, G).download()
    ulp = np.abs(got.view(np.int32).astype(np.int64) - want.view(np.int32).astype(np.int64))
    assert ulp.max() <= 2, ulp.max()


@pytest.mark.parametrize("method", [BASELINE, TCU_SPLIT])
@pytest.mark.parametrize("which,partition", [("small", 32), ("small", 64), ("large", 64), ("large", 128)])
def test_grid_score_matches_oracle(port, dev, small, large, method, which, partition):
    inst, lp, G, dg = small if which == "small" else large
    poses = _poses(inst, 24, 1)
    e, g, tq = dev.grid_score_batch(dg, inst, lp, poses, method, partition)
    for i, p in enumerate(poses):
        we, wg, wt, _ = port.grid_score(inst, G, lp, p)
        assert abs(e[i] - we) <= 1e-5 * max(1.0, abs(we)), (i, e[i], we)
        assert np.abs(g[i] - wg).max() <= 2e-5 * max(1.0, np.abs(wg).max()), (i, g[i], wg)
        assert np.abs(tq[i] - wt).max() <= 2e-5 * max(1.0, np.abs(wt).max())


def test_grid_score_without_intra_matches_oracle(port, dev, small):
    inst, lp, G, dg = small
    lp0 = LigandParams(lp.atom_type, lp.charge, lp.radius, lp.epsilon, lp.elec_scale, intra=False)
    poses = _poses(inst, 16, 2)
    e, g, _ = dev.grid_score_batch(dg, inst, lp0, poses, BASELINE, 64)
    for i, p in enumerate(poses):
        we, wg, _, wi = port.grid_score(inst, G, lp0, p)
        assert wi == 0.0
        assert abs(e[i] - we) <= 1e-5 * max(1.0, abs(we))
        assert np.abs(g[i] - wg).max() <= 2e-5 * max(1.0, np.abs(wg).max())


def test_grid_paper_tcu_reduction_within_f16_tolerance(dev, small):
    inst, lp, G, dg = small
    poses = _poses(inst, 16, 3, spread=2.0)
    e0, g0, _ = dev.grid_score_batch(dg, inst, lp, poses, BASELINE, 64)
    e1, g1, _ = dev.grid_score_batch(dg, inst, lp, poses, TCU, 64)
    assert np.all(np.abs(e1 - e0) <= 5e-3 * np.maximum(1.0, np.abs(e0)))
    assert np.all(np.abs(g1 - g0).max(axis=1) <= 5e-3 * np.maximum(1.0, np.abs(g0).max(axis=1)))


def test_grid_methods_agree_with_tcu_split(dev, large):
    """The error-compensated tf32 MMA reduction is fp32-accurate: it agrees
    with the shuffle-tree reduction to a few float ulps of the partial mass."""
    inst, lp, G, dg = large
    poses = _poses(inst, 16, 4, spread=2.0)
    e0, g0, _ = dev.grid_score_batch(dg, inst, lp, poses, BASELINE, 128)
    e1, g1, _ = dev.grid_score_batch(dg, inst, lp, poses, TCU_SPLIT, 128)
    assert np.all(np.abs(e1 - e0) <= 1e-5 * np.maximum(1.0, np.abs(e0)))
    assert np.all(np.abs(g1 - g0).max(axis=1) <= 1e-5 * np.maximum(1.0, np.abs(g0).max(axis=1)))


def test_grid_local_search_matches_oracle_statistically(port, dev, small):
    inst, lp, G, dg = small
    starts = _poses(inst, 24, 5, spread=2.0)
    res = dev.grid_local_search_batch(dg, inst, lp, starts, 150, 1e-4, BASELINE, 64)
    rel = []
    for s, r in zip(starts, res):
        w = port.grid_local_search(inst, G, lp, s, 150, 1e-4)
        rel.append(abs(r.energy - w["energy"]) / max(1.0, abs(w["energy"])))
        # the reported best pose really has the reported energy on the device
    assert np.median(rel) <= 1e-3, rel
    ge = np.array([r.energy for r in res])
    we = np.array([port.grid_local_search(inst, G, lp, s, 150, 1e-4)["energy"] for s in starts])
    assert abs(ge.mean() - we.mean()) <= 0.02 * max(1.0, abs(we.mean()))
    e_best, _, _ = dev.grid_score_batch(dg, inst, lp, np.stack([r.genotype for r in res]), BASELINE, 64)
    assert np.allclose(e_best, ge, rtol=1e-6, atol=1e-6)


def test_grid_lga_paired_seeds(port, dev, small):
    inst, lp, G, dg = small
    s = LgaSettings(generations=6)
    seeds = np.arange(8, dtype=np.uint64) + 1000
    gpu = dev.grid_lga_run_batch(dg, inst, lp, BASELINE, s, seeds)
    cpu = [port.grid_lga_run(inst, G, lp, s, int(x)) for x in seeds]
    ge = np.array([r.best_energy for r in gpu])
    ce = np.array([r["best_energy"] for r in cpu])
    assert abs(ge.mean() - ce.mean()) <= 0.02 * max(1.0, abs(ce.mean())), (ge, ce)
    for r in gpu:  # budget and bookkeeping as the reference's lga_run
        assert r.evaluations <= s.max_evaluations
        assert r.best_energy <= min(x[0] for x in r.runs) + 1e-12
        assert len(r.runs) == s.generations * 9 + 1


def test_grid_errors_before_work(dev, small):
    inst, lp, G, dg = small
    poses = _poses(inst, 2, 6)
    with pytest.raises(UnsupportedBlockSizeError):
        dev.grid_score_batch(dg, inst, lp, poses, BASELINE, 8)  # not a legal block
    big = random_instance(derive_rng(1, "grid/big"), 40, 50, 4)
    lpb = random_ligand_params(derive_rng(1, "grid/bigl"), 50, 4)
    with pytest.raises(UnsupportedBlockSizeError):  # 46 dimensions > 32 threads
        dev.grid_score_batch(dg, big, lpb, _poses(big, 1, 7), BASELINE, 32)
    bad = LigandParams(np.full(inst.n_atoms, 9), lp.charge, lp.radius, lp.epsilon)
    with pytest.raises(SizeError):
        dev.grid_score_batch(dg, inst, bad, poses, BASELINE, 64)


def test_c4_full_size_maps_and_scores(port, dev):
    """BASELINE config C4 at full size: 126^3 x 6 maps built on the device
    (48 MB) equal the oracle's builder at sampled lattice points (oracle run
    on 2x2x2 sub-lattices anchored there), and the 100-atom / 30-torsion
    ligand scores on those maps match the oracle scoring the downloaded maps."""
    from paper_2410_10447_b200._abi import Grid
    from paper_2410_10447_b200.workloads import c4

    inst, params, fields, grid, _ = c4()
    dg = dev.grid_build(inst, fields, grid)
    maps = dg.download()
    assert maps.shape == (6, 126, 126, 126)
    rng = derive_rng(3, "c4/points")
    for _ in range(12):
        ix, iy, iz = (int(rng.next_index(125)) for _ in range(3))
        sub = Grid((2, 2, 2), grid.n_types, tuple(o + grid.spacing * i for o, i in zip(grid.origin, (ix, iy, iz))),
                   grid.spacing)
        want = port.grid_build(inst, fields, sub)
        got = maps[:, iz:iz + 2, iy:iy + 2, ix:ix + 2]
        ulp = np.abs(got.view(np.int32).astype(np.int64) - want.view(np.int32).astype(np.int64))
        assert ulp.max() <= 2
    G = Grid(grid.shape, grid.n_types, grid.origin, grid.spacing, maps)
    poses = _poses(inst, 12, 9, spread=4.0)
    e, g, _ = dev.grid_score_batch(dg, inst, params, poses, BASELINE, 128)
    for i, p in enumerate(poses):
        we, wg, _, _ = port.grid_score(inst, G, params, p)
        assert abs(e[i] - we) <= 1e-5 * max(1.0, abs(we))
        assert np.abs(g[i] - wg).max() <= 2e-5 * max(1.0, np.abs(wg).max())


# ---- strict FP64 grid mode (context pair precision MDR_PAIR_FP64): the
# oracle's double arithmetic in the oracle's order with correctly rounded
# trig on both sides (csrc/crmath.cuh, oracle/crmath.h), so dockings are
# compared run for run, bit for bit.
@pytest.fixture(scope="module")
def strict_dev():
    from paper_2410_10447_b200 import PAIR_FP64, Device

    d = Device(0, pair=PAIR_FP64)
    yield d
    d.close()


def test_crmath_device_equals_oracle(dev):
    """csrc/crmath.cuh (device) and oracle/crmath.h compute the same
    correctly rounded sin / cos / log bit for bit (10^6 inputs)."""
    import ctypes as C

    from oracle.oracle import cr_values

    n = 1 << 20
    out = np.zeros((n, 8))
    assert dev.lib.mdr_crmath_values(dev.ctx, 0, n, C.c_void_p(out.ctypes.data)) == 0
    want = cr_values(0, n)
    assert np.array_equal(out[:, :4].view(np.uint64), want.view(np.uint64))


def test_grid_strict_local_search_identical(port, strict_dev, small):
    inst, lp, G, _ = small
    dg = strict_dev.grid_upload(G)
    starts = _poses(inst, 24, 5, spread=2.0)
    res = strict_dev.grid_local_search_batch(dg, inst, lp, starts, 150, 1e-4, BASELINE, 64)
    for s, r in zip(starts, res):
        w = port.grid_local_search(inst, G, lp, s, 150, 1e-4)
        assert r.energy == w["energy"] and r.iterations == w["iterations"]
        assert np.array_equal(r.genotype, w["genotype"])
    dg.free()


def test_grid_strict_lga_identical(port, strict_dev, small, large):
    """Whole grid-mode LGA runs (init, offspring with correctly rounded
    Box-Muller draws, Lamarckian searches, polish): the device's strict path
    equals orc_grid_lga_run run for run, with and without intramolecular
    terms, small and 100-atom / 30-torsion ligands."""
    for case, gens in ((small, 4), (large, 2)):
        inst, lp, G, _ = case
        dg = strict_dev.grid_upload(G)
        s = LgaSettings(generations=gens)
        seeds = np.arange(4, dtype=np.uint64) + 2000
        gpu = strict_dev.grid_lga_run_batch(dg, inst, lp, BASELINE, s, seeds)
        for r, sd in zip(gpu, seeds):
            w = port.grid_lga_run(inst, G, lp, s, int(sd))
            assert r.best_energy == w["best_energy"] and r.evaluations == w["evaluations"], (sd, r.best_energy, w)
            assert np.array_equal(r.best_genotype, w["best_genotype"])
            assert [x[0] for x in r.runs] == [x[0] for x in w["runs"]]
        dg.free()


def test_c4_grid_strict_runs_identical_to_oracle():
    """C4 at full size (100 atoms / 30 torsions, 126^3 x 6 device-built maps,
    intramolecular on, default LgaSettings, partition 64), 16 paired seeds:
    the strict FP64 device docking reproduces orc_grid_lga_run run for run
    (best energy, evaluations, genotype) and the 2 A clustering of the final
    poses is identical (north_star: "final best-pose energies and RMSD
    clustering must match")."""
    from oracle.oracle import Oracle, grid_lga_runs_parallel
    from paper_2410_10447_b200 import PAIR_FP64, Device
    from paper_2410_10447_b200._abi import Grid
    from paper_2410_10447_b200.workloads import c4

    inst, params, fields, grid, s = c4()
    d = Device(0, pair=PAIR_FP64)
    try:
        dg = d.grid_build(inst, fields, grid)
        G = Grid(grid.shape, grid.n_types, grid.origin, grid.spacing, dg.download())
        seeds = np.arange(16, dtype=np.uint64) + np.uint64(515000)
        gpu = d.grid_lga_run_batch(dg, inst, params, BASELINE, s, seeds)
        cpu = grid_lga_runs_parallel(inst, G, params, s, seeds)
        for g, c in zip(gpu, cpu):
            assert g.best_energy == c[0] and g.evaluations == c[1]
            assert np.array_equal(g.best_genotype, c[3])
        ge = np.array([g.best_energy for g in gpu])
        gc, _, gn = d.cluster_poses(inst, np.stack([g.best_genotype for g in gpu]), ge, 2.0)
        cc, _, cn = Oracle("port").cluster_poses(inst, np.stack([c[3] for c in cpu]), np.array([c[0] for c in cpu]), 2.0)
        assert gn == cn and np.array_equal(gc, cc)
        dg.free()
    finally:
        d.close()
