"""Pin the CPU oracle (plain-C restatement, oracle/mdr_oracle.c) before it is
trusted as the parity checker: against the golden vectors of the reference's
own tests, against fixtures recorded from the reference itself
(tests/golden/ref_vectors.json, made by tests/golden/make_golden.py), and
bit-for-bit against the reference library compiled in place (oracle/_ref)."""
import math

import numpy as np
import pytest

from paper_2410_10447_b200._abi import (
    BASELINE,
    HALF,
    SINGLE,
    TCU,
    Instance,
    LgaSettings,
    NumericDomainError,
    SizeError,
    UnsupportedBlockSizeError,
    derive_rng,
    random_instance,
    random_pose,
)


def bits32(x):
    return np.asarray(x, np.float32).view(np.uint32)


# ---------------------------------------------------------------- RNG
def test_rng_golden_sequence(port):
    # reference tests/test_rng_io.cpp:16-28
    want = [0x1521A18246366D92, 0x9D07F170119DDEAC, 0x4F24E237C4AA8F1C, 0xD99886563AFA1125,
            0xB3F4A8059AE62D41, 0xCAFB9F189122EFF6, 0x69531C330023818D, 0x78A03C2B866C4730,
            0xAEA39534C98C5EFD, 0xCCFC0166FCF2CB6A]
    assert [int(x) for x in port.rng_draws(42, "golden", 10)] == want
    r = derive_rng(42, "golden")  # host-side mirror used for synthetic inputs
    assert [r.next_u64() for _ in range(10)] == want


def test_rng_normals_match_reference(port, ref_vectors):
    assert port.rng_normals(12345, "lga", 16).tolist() == ref_vectors["normals_12345_lga"]


# ---------------------------------------------------------------- half
def test_half_frozen_conversions(port):
    # reference tests/test_half.cpp:88-101, 161-166
    cases = {1.0: 0x3C00, 0.1: 0x2E66, 65520.0: 0x7C00, 65504.0: 0x7BFF, 65519.9: 0x7BFF,
             2.0**-24: 0x0001, 2.0**-25: 0x0000, -1.0: 0xBC00, -65520.0: 0xFC00}
    got = port.f32_to_half(np.array(list(cases), np.float32))
    assert got.tolist() == list(cases.values())
    assert port.f32_to_half(np.array([np.nan], np.float32))[0] == 0x7E00


def test_half_exhaustive_roundtrip(port):
    # reference tests/test_half.cpp:117-129, acceptance.cpp:308-343
    h = np.arange(65536, dtype=np.uint32).astype(np.uint16)
    finite = h[(h & 0x7C00) != 0x7C00]
    assert finite.size == 63488
    assert np.array_equal(port.f32_to_half(port.half_to_f32(finite)), finite)


def test_half_matches_reference_bitwise(port, ref):
    rng = np.random.default_rng(1)
    x = np.concatenate([
        rng.uniform(-70000, 70000, 200000),
        rng.uniform(-1e-4, 1e-4, 200000),
        rng.uniform(-1e-7, 1e-7, 50000),
        np.ldexp(rng.uniform(1, 2, 50000), rng.integers(-30, 17, 50000)),
    ]).astype(np.float32)
    # exact midpoints between consecutive halves exercise the ties-to-even rule
    h = np.arange(0, 0x7BFF, dtype=np.uint16)
    lo, hi = port.half_to_f32(h), port.half_to_f32(h + 1)
    mid = ((lo.astype(np.float64) + hi) / 2).astype(np.float32)
    x = np.concatenate([x, mid, -mid, np.array([np.inf, -np.inf, 0.0, -0.0], np.float32)])
    assert np.array_equal(port.f32_to_half(x), ref.f32_to_half(x))


# ---------------------------------------------------------------- MMA
def test_mma_frozen(port):
    one, two = 0x3C00, 0x4000
    eye = np.zeros((16, 16), np.uint16)
    np.fill_diagonal(eye, one)
    iota = port.f32_to_half(np.arange(256, dtype=np.float32)).reshape(16, 16)
    z = np.zeros((16, 16), np.float32)
    # identity * B = B (reference tests/test_mma.cpp:121-152)
    d = port.mma(eye, iota, z, SINGLE)
    assert np.array_equal(d, port.half_to_f32(iota.reshape(-1)).reshape(16, 16))
    ones = np.full((16, 16), one, np.uint16)
    assert np.all(port.mma(ones, ones, z, HALF) == 16.0)
    diag2 = np.zeros((16, 16), np.uint16)
    np.fill_diagonal(diag2, two)
    d = port.mma(diag2, diag2, np.ones((16, 16), np.float32), HALF)  # diag(2)^2 + 1
    assert np.all(np.diag(d) == 5.0) and d[0, 1] == 1.0


def test_mma_matches_reference(port, ref):
    rng = derive_rng(300, "acceptance/mma")
    for t in range(40):
        a = port.f32_to_half(np.array([rng.uniform(-1, 1) for _ in range(256)], np.float32))
        b = port.f32_to_half(np.array([rng.uniform(-1, 1) for _ in range(256)], np.float32))
        c = np.array([rng.uniform(-1, 1) for _ in range(256)], np.float32)
        for mode in (HALF, SINGLE):
            assert np.array_equal(bits32(port.mma(a, b, c, mode)), bits32(ref.mma(a, b, c, mode)))


# ---------------------------------------------------------------- reductions
def test_reduce4_frozen(port):
    # reference tests/test_reduce.cpp:105-140
    for mode in (HALF, SINGLE):
        r, st = port.reduce4(np.tile([1, 0, 0, 0], (64, 1)), mode)
        assert r.tolist() == [64, 0, 0, 0] and st.block_syncs == 2 and st.mma_ops == 2
        assert st.atomic_adds == 0 and st.memory_fences == 0
    b = np.array([[i % 2, 0, 0, 1] for i in range(128)])
    r, st = port.reduce4(b, HALF)
    assert r.tolist() == [64, 0, 0, 128] and st.mma_ops == 3
    r, st = port.reduce4(np.array([[1.5, -2.0, 0.25, 3.0]]), HALF)
    assert r.tolist() == [1.5, -2.0, 0.25, 3.0] and st.block_syncs == 2
    with pytest.raises(SizeError):
        port.reduce4(np.zeros((0, 4)), HALF)


def test_reduce4_integer_exact_and_vs_reference(port, ref):
    rng = derive_rng(4001, "reduce4-int")
    for trial in range(30):
        n = 1 + rng.next_index(1024)
        v = np.array([[rng.next_index(5) - 2.0 for _ in range(4)] for _ in range(n)], np.float32)
        for mode in (HALF, SINGLE):
            r, st = port.reduce4(v, mode)
            assert r.tolist() == v.astype(np.float64).sum(0).tolist()
            r2, st2 = ref.reduce4(v, mode)
            assert np.array_equal(bits32(r), bits32(r2)) and st == st2


def test_reduce4_random_vs_reference(port, ref):
    rng = np.random.default_rng(7)
    for trial in range(60):
        n = int(rng.integers(1, 1025))
        v = (rng.uniform(-1, 1, (n, 4)) * (10.0 ** rng.integers(-3, 3))).astype(np.float32)
        for mode in (HALF, SINGLE):
            r, st = port.reduce4(v, mode)
            r2, st2 = ref.reduce4(v, mode)
            assert np.array_equal(bits32(r), bits32(r2)) and st == st2


def test_warp_and_block_reduce_frozen(port, ref):
    # reference tests/test_reduce.cpp:228-299
    s, st = port.warp_reduce(np.arange(32, dtype=np.float32))
    assert s == 496.0 and st.warp_shuffles == 160 and st.block_syncs == 0
    s, st = port.block_reduce(np.ones(64, np.float32), 64)
    assert s == 64 and st.block_syncs == 3 and st.atomic_adds == 2 and st.memory_fences == 2
    s, st = port.block_reduce(np.arange(1024, dtype=np.float32), 1024)
    assert s == 523776.0 and st.atomic_adds == 32
    with pytest.raises(UnsupportedBlockSizeError):
        port.block_reduce(np.ones(33, np.float32), 33)
    with pytest.raises(SizeError):
        port.block_reduce(np.ones(64, np.float32), 96)
    rng = np.random.default_rng(3)
    for threads in range(32, 1025, 32):
        x = rng.uniform(-1, 1, threads).astype(np.float32)
        a, sa = port.block_reduce(x, threads)
        b, sb = ref.block_reduce(x, threads)
        assert bits32(a) == bits32(b) and sa == sb


def test_reduce7_frozen_and_vs_reference(port, ref):
    # reference tests/test_reduce.cpp:301-342
    recs = np.tile(np.arange(1, 8, dtype=np.float32), (64, 1))
    for m in (BASELINE, TCU):
        s, _ = port.reduce7(recs, m, HALF)
        assert s.tolist() == [64, 128, 192, 256, 320, 384, 448]
    _, st = port.reduce7(recs, BASELINE, HALF)
    assert st.block_syncs == 21 and st.atomic_adds == 14
    _, st = port.reduce7(recs, TCU, HALF)
    assert st.block_syncs == 4 and st.atomic_adds == 0 and st.mma_ops == 4
    with pytest.raises(UnsupportedBlockSizeError):
        port.reduce7(np.zeros((63, 7)), TCU, HALF)
    s, _ = port.reduce7(np.tile([1, 0, 0, 0, 0, 0, 1], (100, 1)), TCU, HALF)
    assert s[0] == 100 and s[6] == 100
    rng = np.random.default_rng(11)
    for trial in range(40):
        n = 32 * int(rng.integers(2, 33))
        r = rng.uniform(-1, 1, (n, 7)).astype(np.float32)
        for m, a in ((BASELINE, HALF), (TCU, HALF), (TCU, SINGLE)):
            x, sx = port.reduce7(r, m, a)
            y, sy = ref.reduce7(r, m, a)
            assert np.array_equal(bits32(x), bits32(y)) and sx == sy


# ---------------------------------------------------------------- scoring
def single_well():
    return Instance(np.array([[1.5, 0, 0, 1.0]]), np.array([-1]), np.array([[0, 0, 0, 1.25, 1.5]]), 0)


def test_score_stationary_single_well(port):
    # reference tests/test_docking.cpp:92-118
    inst = single_well()
    for m, a in ((BASELINE, SINGLE), (TCU, SINGLE), (TCU, HALF)):
        e, g, t, _ = port.score(inst, np.zeros(6), m, a, 64)
        assert e == np.float32(-1.25) and not g.any() and not t.any()
    e, g, t = port.score_reference(inst, np.zeros(6))
    assert e == -1.25 and not g.any()


def test_score_matches_golden(port, instances, ref_vectors):
    for c in ref_vectors["score"]:
        inst = instances[c["inst"]]
        g = np.array(c["g"])
        if c["method"] == "reference":
            e, gr, tq = port.score_reference(inst, g)
            assert e == c["energy"] and gr.tolist() == c["grad"] and tq.tolist() == c["torque"]
            continue
        e, gr, tq, st = port.score(inst, g, c["method"], c["accum"], c["partition"])
        assert float(e) == c["energy"], c
        assert gr.astype(float).tolist() == c["grad"]
        assert tq.astype(float).tolist() == c["torque"]
        assert list(st.as_tuple()) == c["stats"]


def test_score_random_vs_reference(port, ref):
    rng = derive_rng(9001, "oracle/score")
    for rep in range(30):
        inst = random_instance(rng, rep % 9, 4 + rng.next_index(40), 2 + rng.next_index(30))
        g = random_pose(rng, inst.n_rot, 1.0)
        for part in (32, 64, 128):
            for m, a in ((BASELINE, SINGLE), (TCU, HALF), (TCU, SINGLE)):
                if m == TCU and part < 64:
                    with pytest.raises(UnsupportedBlockSizeError):
                        port.score(inst, g, m, a, part)
                    continue
                x = port.score(inst, g, m, a, part)
                y = ref.score(inst, g, m, a, part)
                assert bits32(x[0]) == bits32(y[0])
                assert np.array_equal(bits32(x[1]), bits32(y[1]))
                assert np.array_equal(bits32(x[2]), bits32(y[2])) and x[3] == y[3]
        x, y = port.score_reference(inst, g), ref.score_reference(inst, g)
        assert x[0] == y[0] and np.array_equal(x[1], y[1]) and np.array_equal(x[2], y[2])


def test_score_reference_finite_differences(port):
    # reference tests/test_docking.cpp:151-164 / acceptance.cpp:149-208
    rng = derive_rng(6002, "dock-fd")
    inst = random_instance(rng, 3, 7, 4)
    h = 1e-4
    for rep in range(5):
        g = random_pose(rng, inst.n_rot, 1.0)
        _, grad, _ = port.score_reference(inst, g)
        for d in range(inst.dim):
            lo, hi = g.copy(), g.copy()
            lo[d] -= h
            hi[d] += h
            fd = (port.score_reference(inst, hi)[0] - port.score_reference(inst, lo)[0]) / (2 * h)
            assert abs(grad[d] - fd) / max(abs(fd), 1.0) < 1e-4


# ---------------------------------------------------------------- search
def test_adadelta_first_step(port, ref):
    # reference tests/test_docking.cpp:211-243
    grad = np.zeros(6)
    grad[0] = 1.0
    sg, su, g = port.adadelta_step(np.zeros(6), np.zeros(6), np.zeros(6), grad)
    assert math.isclose(g[0], -0.004472091234310839, rel_tol=1e-12)
    assert math.isclose(sg[0], 0.05, rel_tol=1e-12) and g[1] == 0.0
    bad = np.zeros(6)
    bad[3] = np.inf
    with pytest.raises(NumericDomainError):
        port.adadelta_step(np.zeros(6), np.zeros(6), np.zeros(6), bad)
    rng = np.random.default_rng(5)
    for _ in range(50):
        a = [rng.uniform(0, 1, 9), rng.uniform(0, 1e-3, 9), rng.uniform(-4, 4, 9), rng.normal(size=9)]
        x, y = port.adadelta_step(*a), ref.adadelta_step(*a)
        for u, v in zip(x, y):
            assert np.array_equal(u, v)


def test_local_search_matches_golden(port, instances, ref_vectors):
    for c in ref_vectors["local_search"]:
        r = port.local_search(instances[c["inst"]], np.array(c["start"]), c["max_iters"], c["tol"],
                              c["method"], c["accum"], 64)
        assert r["energy"] == c["energy"] and r["iterations"] == c["iterations"]
        assert r["converged"] == c["converged"] and r["genotype"].tolist() == c["genotype"]


def test_lga_run_matches_golden(port, instances, ref_vectors):
    for c in ref_vectors["lga_run"]:
        s = LgaSettings(**c["settings"])
        r = port.lga_run(instances[c["inst"]], c["method"], c["accum"], s, c["seed"])
        assert r["best_energy"] == c["best_energy"] and r["evaluations"] == c["evaluations"]
        assert r["best_genotype"].tolist() == c["best_genotype"]
        assert [list(x) for x in r["runs"]] == c["runs"] and r["converged"] == c["converged"]
        assert list(r["total_stats"].as_tuple()) == c["total_stats"]


def test_lga_determinism_pin(ref_vectors):
    # reference acceptance.cpp:283-304 (energy -10.296875, 25 549 evaluations)
    c = [c for c in ref_vectors["lga_run"] if c["seed"] == 20260816][0]
    assert c["best_energy"] == -10.296875 and c["evaluations"] == 25549 and len(c["runs"]) == 181


def test_lga_random_vs_reference(port, ref, instances):
    s = LgaSettings(population_size=10, generations=3, ls_max_iters=40)
    for seed in range(5):
        for m, a in ((BASELINE, SINGLE), (TCU, HALF)):
            x = port.lga_run(instances["s3"], m, a, s, 1000 + seed)
            y = ref.lga_run(instances["s3"], m, a, s, 1000 + seed)
            assert x["best_energy"] == y["best_energy"] and x["evaluations"] == y["evaluations"]
            assert np.array_equal(x["best_genotype"], y["best_genotype"]) and x["runs"] == y["runs"]


def test_c2_bench_inputs_are_the_reference_stream(ref):
    """The C2 microbench inputs: ref_fill_uniform (the
    reference's RngStream::uniform(-1, 1), rng.cpp:43-45) equals the Python
    mirror draw for draw; the device generator is pinned to the same shim in
    tests/test_gpu_units.py."""
    import ctypes as C

    from paper_2410_10447_b200._abi import derive_rng

    n = 257
    x = np.empty(n, np.float32)
    ref.lib.ref_fill_uniform.argtypes = [C.c_uint64, C.c_char_p, C.c_int64, C.c_void_p]
    assert ref.lib.ref_fill_uniform(12345, b"bench/64/float4", n, x.ctypes.data) == 0
    rng = derive_rng(12345, "bench/64/float4")
    want = np.array([rng.uniform(-1.0, 1.0) for _ in range(n)], np.float32)
    assert np.array_equal(x.view(np.uint32), want.view(np.uint32))


def test_c2_cpu_leg_times_the_reference(ref):
    """The CPU leg of the C2 microbench runs the reference's own reduce4 /
    simulate_block / reduce7 / baseline_block_reduce (ref_time_reduce)."""
    from paper_2410_10447_b200.microbench import cpu_leg

    out = cpu_leg(blocks=(64,), n_sample=8, budget_s=0.05, procs=2)
    row = out["results"]["64"]
    assert len(row) == 5 and all(v["ns_per_call_1core"] > 0 and v["calls_all_cores"] > 0 for v in row.values())
    assert out["kind"] == "reference" and out["cores"] == 2
