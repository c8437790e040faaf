"""GPU parity of scoring, ADADELTA, local search and LGA (C-ABI) against the
CPU oracle and the fixtures recorded from the reference itself.

Tolerances (written here):
  * Baseline method with FP64 pair terms (the default): per-evaluation float
    outputs bit-identical to the reference for >= 99 % of poses; the rest
    (a CUDA sin/cos differing from glibc by an ulp) within 1e-6 relative.
  * Tcu method (paper's f16 MMA): per-component within 2 half-ulps of the
    reference's emulated result (hardware fp32 accumulation order).
  * TcuSplit and the FP32 fast pair mode: energy within 1e-4 * max(|E|, 1) and
    gradient within 1e-4 * max(max|g|, 1) of the fp32 reference (Baseline).
  * Full LGA runs: statistical parity (paired seeds, relative difference of
    mean best energies < 0.2 %, the reference's acceptance.cpp:128-145 gate);
    plus exact equality of runs whose trajectories do not diverge.
"""
import numpy as np
import pytest

from paper_2410_10447_b200 import (
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
    NumericDomainError,
    SizeError,
    UnsupportedBlockSizeError,
    validate_pair,
)
from paper_2410_10447_b200._abi import Instance, derive_rng, random_instance, random_pose

pytestmark = pytest.mark.gpu


def bits(x):
    return np.asarray(x, np.float32).view(np.uint32)


def half_ulp(v):
    a = np.maximum(np.abs(np.asarray(v, np.float64)), 2.0**-14)
    return 2.0 ** (np.floor(np.log2(a)) - 10)


def random_cases(seed, count, natoms_max=40, nsites_max=40):
    rng = derive_rng(seed, "gpu/score")
    out = []
    for rep in range(count):
        inst = random_instance(rng, rep % 9, 1 + rng.next_index(natoms_max), 1 + rng.next_index(nsites_max))
        poses = np.stack([random_pose(rng, inst.n_rot, 1.0 if k % 2 else 0.4) for k in range(16)])
        out.append((inst, poses))
    return out


def test_score_golden_fixtures(dev, instances, ref_vectors):
    mism = 0
    total = 0
    for c in ref_vectors["score"]:
        if c["method"] == "reference":
            continue
        inst = instances[c["inst"]]
        r = dev.score(inst, np.array(c["g"]), c["method"], c["accum"], c["partition"])
        assert list(r.reduce_stats.as_tuple()) == c["stats"]
        want_e, want_g = np.float32(c["energy"]), np.array(c["grad"], np.float32)
        if c["method"] == BASELINE:
            total += 1
            same = bits(r.energy) == bits(want_e) and np.array_equal(bits(r.gradient), bits(want_g))
            mism += not same
            assert abs(float(r.energy) - float(want_e)) <= 1e-6 * max(abs(float(want_e)), 1.0)
        else:
            assert abs(float(r.energy) - float(want_e)) <= 2 * half_ulp(want_e)
    assert mism <= 0.01 * total + 1


def test_score_stationary_single_well(dev):
    inst = Instance(np.array([[1.5, 0, 0, 1.0]]), np.array([-1]), np.array([[0, 0, 0, 1.25, 1.5]]), 0)
    for m, a in ((BASELINE, SINGLE), (TCU, SINGLE), (TCU, HALF), (TCU_SPLIT, SINGLE)):
        r = dev.score(inst, np.zeros(6), m, a, 64)
        assert r.energy == np.float32(-1.25) and not r.gradient.any() and not r.torque.any()


def test_score_validation(dev, instances):
    inst = instances["s1"]
    with pytest.raises(UnsupportedBlockSizeError):
        dev.score(inst, np.zeros(6), TCU, HALF, 32)
    with pytest.raises(UnsupportedBlockSizeError):
        dev.score(inst, np.zeros(6), BASELINE, HALF, 48)
    with pytest.raises(SizeError):
        dev.score(inst, np.zeros(8), BASELINE, HALF, 64)
    dev.score(inst, np.zeros(6), BASELINE, SINGLE, 32)


@pytest.mark.parametrize("partition", [32, 64, 128])
def test_score_baseline_bit_exact_random(dev, port, partition):
    exact = total = 0
    for inst, poses in random_cases(100 + partition, 25, natoms_max=140):
        e, g, t, _ = dev.score_batch(inst, poses, BASELINE, SINGLE, partition)
        for i, p in enumerate(poses):
            we, wg, wt, _ = port.score(inst, p, BASELINE, SINGLE, partition)
            total += 1
            same = bits(e[i]) == bits(we) and np.array_equal(bits(g[i]), bits(wg)) and np.array_equal(
                bits(t[i]), bits(wt))
            exact += same
            scale = max(float(np.abs(wg).max()), 1.0)
            assert abs(float(e[i]) - float(we)) <= 1e-6 * max(abs(float(we)), 1.0)
            assert np.abs(g[i] - wg).max() <= 1e-6 * scale
    assert exact >= 0.99 * total, (exact, total)


def test_score_tcu_reference_compatible(dev, port):
    for inst, poses in random_cases(7, 10):
        for mode in (HALF, SINGLE):
            e, g, t, st = dev.score_batch(inst, poses, TCU, mode, 64)
            for i, p in enumerate(poses):
                we, wg, wt, wst = port.score(inst, p, TCU, mode, 64)
                assert st == wst
                assert abs(float(e[i]) - float(we)) <= 2 * half_ulp(we)
                assert np.all(np.abs(t[i] - wt) <= 2 * half_ulp(wt))


@pytest.mark.parametrize("method,pair", [(TCU_SPLIT, PAIR_FP64), (BASELINE, PAIR_FP32), (TCU_SPLIT, PAIR_FP32),
                                         (BASELINE, PAIR_FP64_FAST), (TCU_SPLIT, PAIR_FP64_FAST)])
def test_score_within_1e4_of_fp32_reference(method, pair, port, dev):
    dev = Device(0, pair=pair)
    worst_e = worst_g = 0.0
    for inst, poses in random_cases(31, 20, natoms_max=100, nsites_max=64):
        e, g, _, _ = dev.score_batch(inst, poses, method, SINGLE, 128)
        for i, p in enumerate(poses):
            we, wg, _, _ = port.score(inst, p, BASELINE, SINGLE, 128)
            worst_e = max(worst_e, abs(float(e[i]) - float(we)) / max(abs(float(we)), 1.0))
            worst_g = max(worst_g, float(np.abs(g[i] - wg).max()) / max(float(np.abs(wg).max()), 1.0))
    dev.close()
    assert worst_e <= 1e-4 and worst_g <= 1e-4, (worst_e, worst_g)


def test_score_reference_and_fd(dev, port):
    for inst, poses in random_cases(55, 10):
        e, g, t = dev.score_reference_batch(inst, poses)
        for i, p in enumerate(poses):
            we, wg, wt = port.score_reference(inst, p)
            assert abs(e[i] - we) <= 1e-12 * max(abs(we), 1.0)
            assert np.abs(g[i] - wg).max() <= 1e-12 * max(np.abs(wg).max(), 1.0)


def test_adadelta_step_bit_exact(dev, port):
    rng = np.random.default_rng(5)
    n, dim = 64, 14
    a = [rng.uniform(0, 1, (n, dim)), rng.uniform(0, 1e-3, (n, dim)), rng.uniform(-4, 4, (n, dim)),
         rng.normal(size=(n, dim))]
    got = dev.adadelta_step_batch(*a)
    for i in range(n):
        want = port.adadelta_step(a[0][i], a[1][i], a[2][i], a[3][i])
        for u, v in zip(got, want):
            assert np.array_equal(u[i], v)
    sg, su, g = dev.adadelta_step(np.zeros(6), np.zeros(6), np.zeros(6), [1, 0, 0, 0, 0, 0])
    assert abs(g[0] - -0.004472091234310839) <= 1e-12 * 0.0045
    bad = np.zeros(6)
    bad[3] = np.nan
    with pytest.raises(NumericDomainError):
        dev.adadelta_step(np.zeros(6), np.zeros(6), np.zeros(6), bad)


def test_local_search_golden(dev, instances, ref_vectors):
    exact = total = 0
    for c in ref_vectors["local_search"]:
        r = dev.local_search(instances[c["inst"]], np.array(c["start"]), c["max_iters"], c["tol"], c["method"],
                             c["accum"], 64)
        if c["method"] == BASELINE:
            total += 1
            same = (r.energy == c["energy"] and r.iterations == c["iterations"] and r.converged == c["converged"]
                    and np.array_equal(r.genotype, np.array(c["genotype"])))
            exact += same
            assert abs(r.energy - c["energy"]) <= 1e-5 * max(abs(c["energy"]), 1.0)
        assert r.stats.block_syncs == (r.iterations + 1) * (21 if c["method"] == BASELINE else 4)
    assert exact >= total - 1, (exact, total)


def test_local_search_single_well(dev):
    inst = Instance(np.array([[1.5, 0, 0, 1.0]]), np.array([-1]), np.array([[0, 0, 0, 1.25, 1.5]]), 0)
    ls = dev.local_search(inst, np.zeros(6), 100, 1e-6, TCU, HALF, 64)
    assert ls.converged and ls.iterations <= 17 and ls.energy == -1.25 and not ls.genotype.any()
    ls = dev.local_search(inst, np.array([0.9, -0.4, 0.3, 0, 0, 0]), 600, 1e-7, BASELINE, SINGLE, 64)
    assert abs(ls.energy - -1.25) <= 1.25e-3 and ls.iterations >= 16


def test_local_search_batch_vs_oracle(dev, port, instances):
    inst = instances["s3"]
    rng = derive_rng(6005, "dock-det")
    starts = np.stack([random_pose(rng, inst.n_rot, 0.6) for _ in range(64)])
    res = dev.local_search_batch(inst, starts, 150, 1e-4, BASELINE, SINGLE, 64)
    same = 0
    for s, r in zip(starts, res):
        w = port.local_search(inst, s, 150, 1e-4, BASELINE, SINGLE, 64)
        same += r.energy == w["energy"] and r.iterations == w["iterations"]
    assert same >= 60, same


def test_lga_golden_and_determinism(dev, instances, ref_vectors):
    exact = 0
    for c in ref_vectors["lga_run"]:
        s = LgaSettings(**c["settings"])
        r = dev.lga_run(instances[c["inst"]], c["method"], c["accum"], s, c["seed"])
        assert r.evaluations <= s.max_evaluations
        assert r.best_energy == min(x[0] for x in r.runs) or r.best_energy <= min(x[0] for x in r.runs)
        assert list(r.total_stats.as_tuple()) == [r.evaluations * x for x in
                                                  dev.score(instances[c["inst"]], np.zeros(instances[c["inst"]].dim),
                                                            c["method"], c["accum"], s.partition).reduce_stats.as_tuple()]
        if c["method"] == BASELINE:
            same = (r.best_energy == c["best_energy"] and r.evaluations == c["evaluations"]
                    and [list(x) for x in r.runs] == [[x[0], x[1], bool(x[2])] for x in c["runs"]])
            exact += same
    assert exact >= 3, exact
    s = LgaSettings()
    a = dev.lga_run_batch(instances["s2"], TCU, HALF, s, [20260816, 20260816])
    assert a[0].best_energy == a[1].best_energy and np.array_equal(a[0].best_genotype, a[1].best_genotype)
    assert a[0].runs == a[1].runs and a[0].evaluations == a[1].evaluations


def test_lga_budget_and_degenerate(dev, instances):
    inst = instances["s1"]
    r = dev.lga_run(inst, BASELINE, SINGLE, LgaSettings(population_size=6, generations=50, max_evaluations=200,
                                                         ls_max_iters=40), 7)
    assert r.evaluations <= 200
    r = dev.lga_run(inst, BASELINE, SINGLE, LgaSettings(population_size=2, generations=1, mutation_sigma=0.0,
                                                         ls_fraction=1.0, ls_max_iters=60), 99)
    assert len(r.runs) == 2 and r.best_energy == min(x[0] for x in r.runs)
    with pytest.raises(SizeError):
        dev.lga_run(inst, BASELINE, SINGLE, LgaSettings(population_size=1), 1)


@pytest.mark.parametrize("name", ["s1", "s2", "s3"])
def test_lga_paired_statistical_parity(dev, port, instances, name):
    """GPU Baseline vs the CPU reference path, 100 paired seeds (acceptance
    check 3 methodology): relative difference of mean best energies < 0.2 %."""
    inst = instances[name]
    s = LgaSettings()
    seeds = np.arange(100, dtype=np.uint64) + np.uint64(12345)
    gpu = dev.lga_run_batch(inst, BASELINE, SINGLE, s, seeds)
    cpu = [port.lga_run(inst, BASELINE, SINGLE, s, int(x)) for x in seeds]
    mg = np.mean([r.best_energy for r in gpu])
    mc = np.mean([r["best_energy"] for r in cpu])
    assert abs(mg - mc) / abs(mc) < 0.002
    same = sum(g.best_energy == c["best_energy"] and g.evaluations == c["evaluations"] for g, c in zip(gpu, cpu))
    assert same >= 50, same  # most trajectories are reproduced exactly


def test_validate_pair_tcu_vs_baseline(dev, instances):
    rep = validate_pair(dev, instances["s2"], BASELINE, TCU, HALF, 100, 12345, LgaSettings())
    assert rep["relative_error"] < 0.002
    rep = validate_pair(dev, instances["s2"], BASELINE, TCU_SPLIT, SINGLE, 100, 12345, LgaSettings())
    assert rep["relative_error"] < 0.002


@pytest.mark.parametrize("pair", [PAIR_FP64_FAST, PAIR_FP32])
def test_fast_modes_cta_local_search_and_lga(pair, port, instances, dev):
    """Fast pair modes run the CTA-per-pose local search (sites split over 4
    warps).  Per-evaluation tolerance 1e-4 is covered above; here the search
    trajectories: final energies within 1e-3 of the CPU reference for >= 90 %
    of the starts, and LGA paired-seed mean best energy within 0.2 %."""
    fast = Device(0, pair=pair)
    inst = instances["synth20"]
    rng = derive_rng(99, "fast/ls")
    starts = np.stack([random_pose(rng, inst.n_rot, 0.6) for _ in range(48)])
    res = fast.local_search_batch(inst, starts, 150, 1e-4, BASELINE, SINGLE, 64)
    close = 0
    for s, r in zip(starts, res):
        w = port.local_search(inst, s, 150, 1e-4, BASELINE, SINGLE, 64)
        close += abs(r.energy - w["energy"]) <= 1e-3 * max(abs(w["energy"]), 1.0)
    assert close >= 0.9 * len(starts), close
    s = LgaSettings()
    seeds = np.arange(64, dtype=np.uint64) + np.uint64(777)
    gpu = fast.lga_run_batch(instances["s2"], BASELINE, SINGLE, s, seeds)
    cpu = [port.lga_run(instances["s2"], BASELINE, SINGLE, s, int(x)) for x in seeds]
    mg = np.mean([r.best_energy for r in gpu])
    mc = np.mean([r["best_energy"] for r in cpu])
    assert abs(mg - mc) / abs(mc) < 0.002
    fast.close()


def test_chunked_site_mapping_matches_lane_per_atom(port, instances, monkeypatch):
    """FP64-fast small ligands run the chunked site mapping (atoms x site
    chunks over all 32 lanes, capi.cpp pick_chunks); MDR_CHUNKING=0 keeps
    lane per atom.  The two differ only in FP64 summation order (chunk
    partial sums), so: float outputs bit-identical for >= 99 % of
    evaluations and within 1e-6 relative for all; every local search within
    1e-5 relative; both against the CPU reference as in the tests above."""
    chunked = Device(0, pair=PAIR_FP64_FAST)
    monkeypatch.setenv("MDR_CHUNKING", "0")
    lane = Device(0, pair=PAIR_FP64_FAST)
    same = total = 0
    rng = derive_rng(92, "chunk/many-torsions")
    wide = random_instance(rng, 40, 16, 64)  # 43 angles: the lane-trig table's second round
    wide_poses = np.stack([random_pose(rng, wide.n_rot, 0.8) for _ in range(16)])
    for inst, poses in random_cases(91, 12, natoms_max=60, nsites_max=80) + [(wide, wide_poses)]:
        ec, gc, _, _ = chunked.score_batch(inst, poses)
        el, gl, _, _ = lane.score_batch(inst, poses)
        total += len(poses)
        same += int(np.sum((bits(ec) == bits(el)) & np.all(bits(gc) == bits(gl), axis=1)))
        assert np.all(np.abs(ec - el) <= 1e-6 * np.maximum(np.abs(el), 1.0))
        scale = np.maximum(np.abs(gl).max(axis=1, keepdims=True), 1.0)
        assert np.all(np.abs(gc - gl) <= 1e-6 * scale)
    assert same >= 0.99 * total, (same, total)
    inst = instances["synth20"]
    rng = derive_rng(17, "chunk/ls")
    starts = np.stack([random_pose(rng, inst.n_rot, 0.6) for _ in range(32)])
    rc = chunked.local_search_batch(inst, starts, 150, 1e-4, BASELINE, SINGLE, 64)
    rl = lane.local_search_batch(inst, starts, 150, 1e-4, BASELINE, SINGLE, 64)
    for a, b in zip(rc, rl):
        assert abs(a.energy - b.energy) <= 1e-5 * max(abs(b.energy), 1.0)
    chunked.close()
    lane.close()


@pytest.mark.parametrize("warps,group", [(0, 0), (2, 1), (2, 3), (3, 0), (3, 1)])
def test_multi_warp_search_bit_identical(instances, monkeypatch, warps, group):
    """FP64-fast chunked ligands run each Lamarckian search of the LGA on
    several warps (ls_multi.cu: warps = 3, a leader per search and a pool of
    item warps shared by the CTA's searches; warps = 2, a leader and a
    helper; 0 = the legacy warp-pair kernel): the pool or the helper takes
    chunk items of every evaluation, the leader keeps the
    genotype in registers; an item is one chunk of sites against 1 or 3
    atoms; ligands past 32 atoms or 32 dimensions run the kernel's BIG form
    (C4 analytic, a 40-torsion ligand).  Same items, same arithmetic, same
    combine order as the one-warp kernel, so with the same site chunking
    (pinned here: MDR_CHUNK_LEN = MDR_LS_CHUNK_LEN = 8) whole LGA runs are
    bit-identical.  Covers a 40-torsion ligand (dim 46 > 32: the multi-warp
    kernel falls back to the legacy pair kernel)."""
    from paper_2410_10447_b200.workloads import c3

    monkeypatch.setenv("MDR_CHUNK_LEN", "8")
    monkeypatch.setenv("MDR_LS_CHUNK_LEN", "8")
    if group:
        monkeypatch.setenv("MDR_LS_GROUP", str(group))  # atoms per chunk item (register blocking)
    multi = Device(0, pair=PAIR_FP64_FAST)
    assert multi.lib.mdr_ctx_set_ls_warps(multi.ctx, warps) == 0
    single = Device(0, pair=PAIR_FP64_FAST)
    assert single.lib.mdr_ctx_set_ls_warps(single.ctx, 1) == 0
    from paper_2410_10447_b200.workloads import c4_analytic

    rng = derive_rng(93, "pair/identity")
    c4a, c4s = c4_analytic()
    cases = [(c3(), LgaSettings(), 16), (random_instance(rng, 3, 28, 64), LgaSettings(), 16),
             (random_instance(rng, 40, 16, 64), LgaSettings(), 16),  # dim 46: two dimensions per lane
             (c4a, c4s, 4)]  # 100 atoms: atoms in blocks of 32
    for inst, st, n_seeds in cases:
        seeds = np.arange(n_seeds, dtype=np.uint64) + np.uint64(4321)
        for method in (BASELINE, TCU_SPLIT, TCU):
            a = multi.lga_run_batch(inst, method, SINGLE, st, seeds)
            b = single.lga_run_batch(inst, method, SINGLE, st, seeds)
            for x, y in zip(a, b):
                assert x.best_energy == y.best_energy and x.evaluations == y.evaluations
                assert np.array_equal(x.best_genotype, y.best_genotype)
    multi.close()
    single.close()


def test_branch_free_sqrt_is_ieee(dev):
    """The multi-warp search's dsqrt_rn must equal IEEE sqrt bit for bit."""
    import ctypes as C

    bad = C.c_uint64()
    assert dev.lib.mdr_selftest_dsqrt(dev.ctx, 12345, 200_000_000, C.byref(bad)) == 0
    assert bad.value == 0


def test_branch_free_sincos_is_libdevice(dev):
    """The multi-warp search's sincos_fast must equal libdevice sincos bit
    for bit (angles in [-pi, pi) and magnitudes 2^-30 .. 2^30)."""
    import ctypes as C

    bad = C.c_uint64()
    assert dev.lib.mdr_selftest_sincos(dev.ctx, 777, 200_000_000, C.byref(bad)) == 0
    assert bad.value == 0
