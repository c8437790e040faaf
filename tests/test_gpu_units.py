"""GPU parity of the L0/L1 units (binary16, MMA unit, reductions) through the
C-ABI against the CPU oracle (oracle/mdr_oracle.c, pinned in test_oracle.py).

Tolerances (written here):
  * Baseline reductions: bit-exact (same shuffle-tree order as reduce.cpp).
  * Tcu (paper's f16 MMA, reference-compatible): hardware fp32 accumulation
    order differs from the emulator's ascending-k loop, so each reduced
    component must be within 1 half-ulp of the emulator (exact for integers).
  * TcuSplit: |err| <= 1e-6 * sum|x| against a float64 oracle (fp32-accurate).
"""
import numpy as np
import pytest

from paper_2410_10447_b200 import BASELINE, HALF, SINGLE, TCU, TCU_SPLIT, SizeError, UnsupportedBlockSizeError
from paper_2410_10447_b200._abi import derive_rng

pytestmark = pytest.mark.gpu


def bits(x):
    return np.asarray(x, np.float32).view(np.uint32)


def half_ulp(v):
    """spacing of binary16 at |v| (subnormal spacing below 2^-14)."""
    a = np.maximum(np.abs(np.asarray(v, np.float64)), 2.0**-14)
    return 2.0 ** (np.floor(np.log2(a)) - 10)


def test_f32_to_half_exhaustive_and_random(dev, port):
    h = np.arange(65536, dtype=np.uint32).astype(np.uint16)
    finite = h[(h & 0x7C00) != 0x7C00]
    f = dev.half_to_f32(finite)
    assert np.array_equal(bits(f), bits(port.half_to_f32(finite)))
    assert np.array_equal(dev.f32_to_half(f), finite)
    rng = np.random.default_rng(2)
    x = np.concatenate([rng.uniform(-70000, 70000, 300000), rng.uniform(-1e-4, 1e-4, 300000),
                        np.ldexp(rng.uniform(1, 2, 100000), rng.integers(-30, 17, 100000)),
                        [np.inf, -np.inf, 0.0, -0.0, np.nan, 65520.0, 65519.99, 2.0**-25]]).astype(np.float32)
    assert np.array_equal(dev.f32_to_half(x), port.f32_to_half(x))


def test_mma_unit(dev, port):
    # frozen examples (reference tests/test_mma.cpp:121-173)
    one = 0x3C00
    eye = np.zeros((16, 16), np.uint16)
    np.fill_diagonal(eye, one)
    iota = port.f32_to_half(np.arange(256, dtype=np.float32)).reshape(16, 16)
    z = np.zeros((16, 16), np.float32)
    assert np.array_equal(dev.mma(eye, iota, z, SINGLE), port.half_to_f32(iota.reshape(-1)).reshape(16, 16))
    ones = np.full((16, 16), one, np.uint16)
    assert np.all(dev.mma(ones, ones, z, HALF) == 16.0)
    # fidelity vs double oracle (reference acceptance.cpp:213-263): single
    # within 16 ulp of the accumulated mass, half within one half-ulp
    rng = np.random.default_rng(300)
    n = 500
    a = port.f32_to_half(rng.uniform(-1, 1, n * 256).astype(np.float32)).reshape(n, 16, 16)
    b = port.f32_to_half(rng.uniform(-1, 1, n * 256).astype(np.float32)).reshape(n, 16, 16)
    c = rng.uniform(-1, 1, (n, 16, 16)).astype(np.float32)
    af = port.half_to_f32(a.reshape(-1)).reshape(a.shape).astype(np.float64)
    bf = port.half_to_f32(b.reshape(-1)).reshape(b.shape).astype(np.float64)
    prod = np.einsum("nik,nkj->nij", af, bf)
    mass = np.einsum("nik,nkj->nij", np.abs(af), np.abs(bf)) + np.abs(c)
    ds = dev.mma_batch(a, b, c, SINGLE)
    ulp = np.spacing(mass.astype(np.float32)).astype(np.float64)
    assert np.max(np.abs(ds - (prod + c)) / ulp) <= 16.0
    ch = port.half_to_f32(port.f32_to_half(c.reshape(-1))).reshape(c.shape)
    dh = dev.mma_batch(a, b, ch, HALF)
    want = port.f32_to_half((prod + ch).astype(np.float32).reshape(-1)).astype(np.int32)
    got = port.f32_to_half(dh.reshape(-1)).astype(np.int32)
    rank = lambda h: np.where(h & 0x8000, -(h & 0x7FFF), h & 0x7FFF)  # noqa: E731
    assert np.max(np.abs(rank(got) - rank(want))) <= 1


def test_warp_and_block_reduce_bit_exact(dev, port):
    s, st = dev.warp_reduce(np.arange(32, dtype=np.float32))
    assert s == 496.0 and st.warp_shuffles == 160
    rng = np.random.default_rng(4)
    lanes = rng.uniform(-10, 10, (2000, 32)).astype(np.float32)
    got, _ = dev.warp_reduce_batch(lanes)
    want = np.array([port.warp_reduce(l)[0] for l in lanes[:300]], np.float32)
    assert np.array_equal(bits(got[:300]), bits(want))
    for threads in range(32, 1025, 32):
        x = rng.uniform(-1, 1, (8, threads)).astype(np.float32)
        got, st = dev.block_reduce_batch(x, threads)
        want = [port.block_reduce(r, threads) for r in x]
        assert np.array_equal(bits(got), bits([w[0] for w in want])) and st == want[0][1]
    s, st = dev.block_reduce(np.arange(1024, dtype=np.float32), 1024)
    assert s == 523776.0 and st.atomic_adds == 32 and st.block_syncs == 3
    with pytest.raises(UnsupportedBlockSizeError):
        dev.block_reduce(np.ones(33, np.float32), 33)
    with pytest.raises(SizeError):
        dev.block_reduce(np.ones(64, np.float32), 96)


def test_reduce4_frozen_and_integer_exact(dev, port):
    # reference tests/test_reduce.cpp:105-140 and acceptance.cpp:75-106
    for mode in (HALF, SINGLE):
        r, st = dev.reduce4(np.tile([1, 0, 0, 0], (64, 1)), mode)
        assert r.tolist() == [64, 0, 0, 0] and st.block_syncs == 2 and st.mma_ops == 2
    r, st = dev.reduce4(np.array([[i % 2, 0, 0, 1] for i in range(128)]), HALF)
    assert r.tolist() == [64, 0, 0, 128] and st.mma_ops == 3
    r, _ = dev.reduce4(np.array([[1.5, -2.0, 0.25, 3.0]]), HALF)
    assert r.tolist() == [1.5, -2.0, 0.25, 3.0]
    with pytest.raises(SizeError):
        dev.reduce4(np.zeros((0, 4)), HALF)
    rng = derive_rng(20001, "acceptance/integers")
    v = np.array([rng.next_index(2) for _ in range(200 * 1024 * 4)], np.float32).reshape(200, 1024, 4)
    for mode in (HALF, SINGLE):
        got, _ = dev.reduce4_batch(v, mode, TCU)
        assert np.array_equal(got, v.sum(1))
    got, _ = dev.reduce4_batch(v, HALF, TCU_SPLIT)
    assert np.array_equal(got, v.sum(1))


@pytest.mark.parametrize("mode", [HALF, SINGLE])
def test_reduce4_tcu_within_half_ulp_of_emulator(dev, port, mode):
    rng = np.random.default_rng(17 + mode)
    worst = 0.0
    for n in (1, 37, 64, 100, 256, 1000, 1024):
        v = rng.uniform(-1, 1, (40, n, 4)).astype(np.float32)
        got, st = dev.reduce4_batch(v, mode, TCU)
        for i in range(40):
            want, wst = port.reduce4(v[i], mode)
            err = np.abs(got[i].astype(np.float64) - want) / half_ulp(want)
            worst = max(worst, float(err.max()))
        assert st == wst
    assert worst <= 1.0, worst


def test_reduce4_split_and_baseline(dev, port):
    rng = np.random.default_rng(23)
    for n in (32, 64, 96, 256, 1024):
        v = (rng.uniform(-1, 1, (50, n, 4)) * 10.0 ** rng.integers(-6, 4, (50, 1, 4))).astype(np.float32)
        got, _ = dev.reduce4_batch(v, HALF, TCU_SPLIT)
        exact = v.astype(np.float64).sum(1)
        mass = np.abs(v.astype(np.float64)).sum(1)
        assert np.all(np.abs(got - exact) <= 1e-6 * mass + 1e-30)
        got, st = dev.reduce4_batch(v, HALF, BASELINE)
        for i in range(5):
            want, wst = port.simulate_block4(v[i], BASELINE, HALF)
            assert np.array_equal(bits(got[i]), bits(want)) and st == wst


def test_reduce7_all_methods(dev, port):
    recs = np.tile(np.arange(1, 8, dtype=np.float32), (64, 1))
    for m in (BASELINE, TCU, TCU_SPLIT):
        s, _ = dev.reduce7(recs, m, HALF)
        assert s.tolist() == [64, 128, 192, 256, 320, 384, 448]
    _, st = dev.reduce7(recs, BASELINE, HALF)
    assert st.block_syncs == 21 and st.atomic_adds == 14
    _, st = dev.reduce7(recs, TCU, HALF)
    assert st.block_syncs == 4 and st.mma_ops == 4 and st.atomic_adds == 0
    with pytest.raises(UnsupportedBlockSizeError):
        dev.reduce7(np.zeros((63, 7)), TCU, HALF)
    with pytest.raises(UnsupportedBlockSizeError):
        dev.reduce7(np.zeros((63, 7)), BASELINE, HALF)
    s, _ = dev.reduce7(np.tile([1, 0, 0, 0, 0, 0, 1], (100, 1)), TCU, HALF)
    assert s[0] == 100 and s[6] == 100
    rng = np.random.default_rng(29)
    for n in (64, 128, 320, 1024):
        r = rng.uniform(-1, 1, (30, n, 7)).astype(np.float32)
        b, _ = dev.reduce7_batch(r, BASELINE, HALF)
        for i in range(30):
            want, _ = port.reduce7(r[i], BASELINE, HALF)
            assert np.array_equal(bits(b[i]), bits(want))
        for mode in (HALF, SINGLE):
            t, _ = dev.reduce7_batch(r, TCU, mode)
            for i in range(10):
                want, _ = port.reduce7(r[i], TCU, mode)
                assert np.all(np.abs(t[i] - want) <= half_ulp(want))
        s, _ = dev.reduce7_batch(r, TCU_SPLIT, HALF)
        mass = np.abs(r.astype(np.float64)).sum(1)
        assert np.all(np.abs(s - r.astype(np.float64).sum(1)) <= 1e-6 * mass)


def test_branch_free_division_is_ieee(dev):
    """The strict pair loop's ddiv_rn must equal IEEE a / b bit for bit."""
    import ctypes as C

    bad = C.c_uint64()
    rc = dev.lib.mdr_selftest_ddiv(dev.ctx, 2024, 200_000_000, C.byref(bad))
    assert rc == 0 and bad.value == 0, bad.value


# ---- TcuSplit batches routed to the tcgen05 contraction (tc05_reduce.cu)
@pytest.mark.parametrize("n", [32, 64, 128, 256])
def test_reduce4_split_tcgen05_route(dev, n):
    """A TcuSplit batch of >= 148*32 reductions of a multiple of 32 records
    runs as one batched tcgen05 contraction (reduce.cpp:80-111 semantics,
    fp32-accurate: |err| <= 1e-6 * sum|x| against float64), with a ragged
    last tile; the warp-per-reduction mma.sync kernel (route off) obeys the
    same bound."""
    n_red = 148 * 32 + 37
    assert dev.lib.mdr_reduce_uses_tc05(dev.ctx, TCU_SPLIT, n, n_red) == 1
    assert dev.lib.mdr_reduce_uses_tc05(dev.ctx, TCU_SPLIT, n + 16, n_red) == 0
    assert dev.lib.mdr_reduce_uses_tc05(dev.ctx, TCU_SPLIT, n, 100) == 0
    assert dev.lib.mdr_reduce_uses_tc05(dev.ctx, BASELINE, n, n_red) == 0
    rng = np.random.default_rng(n)
    v = (rng.uniform(-1, 1, (n_red, n, 4)) * 10.0 ** rng.integers(-6, 4, (n_red, 1, 4))).astype(np.float32)
    exact = v.astype(np.float64).sum(1)
    mass = np.abs(v.astype(np.float64)).sum(1)
    got, st = dev.reduce4_batch(v, SINGLE, TCU_SPLIT)
    assert np.all(np.abs(got - exact) <= 1e-6 * mass + 1e-30)
    dev.lib.mdr_ctx_set_tc05(dev.ctx, 0)
    try:
        warp, st2 = dev.reduce4_batch(v, SINGLE, TCU_SPLIT)
    finally:
        dev.lib.mdr_ctx_set_tc05(dev.ctx, 1)
    assert np.all(np.abs(warp - exact) <= 1e-6 * mass + 1e-30)
    assert st == st2  # the reference-model counters do not depend on the route


@pytest.mark.parametrize("n", [32, 64, 128])
def test_reduce7_split_tcgen05_route(dev, n):
    """Partial7 records (reduce7 reduce.cpp:165-209) through the tcgen05
    contraction: 16 reductions x 8 rows per tile, ragged tail."""
    n_red = 148 * 32 + 21
    assert dev.lib.mdr_reduce_uses_tc05(dev.ctx, TCU_SPLIT, n, n_red) == 1
    rng = np.random.default_rng(100 + n)
    r = (rng.uniform(-1, 1, (n_red, n, 7)) * 10.0 ** rng.integers(-5, 3, (n_red, 1, 7))).astype(np.float32)
    got, _ = dev.reduce7_batch(r, TCU_SPLIT, SINGLE)
    exact = r.astype(np.float64).sum(1)
    mass = np.abs(r.astype(np.float64)).sum(1)
    assert np.all(np.abs(got - exact) <= 1e-6 * mass + 1e-30)
    # integer records: exact
    ri = rng.integers(0, 2, (n_red, n, 7)).astype(np.float32)
    got, _ = dev.reduce7_batch(ri, TCU_SPLIT, SINGLE)
    assert np.array_equal(got, ri.sum(1))


def test_c2_device_inputs_equal_reference_stream(dev, ref):
    """mdr_fill_uniform_dev (the C2 microbench's device-generated inputs)
    equals the reference's RngStream::uniform(-1, 1) draw for draw."""
    import ctypes as C

    import torch

    n = 100_003
    x = torch.empty(n, dtype=torch.float32, device="cuda")
    assert dev.lib.mdr_fill_uniform_dev(dev.ctx, 12345, b"bench/128/float4", n, C.c_void_p(x.data_ptr())) == 0
    torch.cuda.synchronize()
    want = np.empty(n, np.float32)
    ref.lib.ref_fill_uniform.argtypes = [C.c_uint64, C.c_char_p, C.c_int64, C.c_void_p]
    assert ref.lib.ref_fill_uniform(12345, b"bench/128/float4", n, want.ctypes.data) == 0
    assert np.array_equal(x.cpu().numpy().view(np.uint32), want.view(np.uint32))
