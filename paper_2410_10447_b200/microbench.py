"""C2 microbench driver: block float4 sum-reduction, MMA vs warp-shuffle vs
CPU (BASELINE.json configs[1]: block 64/128/256, 10^6 reductions).

Inputs: component c of thread t of reduction r is
(float) uniform(-1, 1) of draw (r B + t) 4 + c + 1 of
derive_rng(12345, "bench/<B>/float4") (rng.hpp:41-43) -- generated on the
device by mdr_fill_uniform_dev (offset-addressable counter RNG, resident in
HBM before timing) and by the reference's own RngStream on the host for the
CPU leg, so both sides reduce identical values.  Partial7 records (reduce7)
use "bench/<B>/partial7", single floats (baseline_block_reduce)
"bench/<B>/float".

Per kernel and block size:
  chain_ns   on-chip: 10^6 reduce-and-broadcasts as dependent chains of 100
             steps per block (the paper's test-kernel shape), ns per
             reduction of the whole GPU;
  latency    clock64 cycles per dependent step of one block's chain (median
             over blocks), and ns at the run's SM clock;
  stream_ns  10^6 distinct input sets read from HBM, ns per reduction;
  roofline   chain: 16 B bytes per reduction over the shared-memory
             bandwidth 148 SMs x 128 B/clk x f_SM; stream: the
             same bytes over the measured HBM bandwidth (MEASURED_PEAKS.json).
Product entry points (mdr_reduce4_dev / mdr_reduce7_dev: TcuSplit on the
tcgen05 contraction, and its warp mma.sync fallback, Baseline trees, the
paper's Tcu) are timed in streaming mode on the same inputs.  CPU leg
(`cpu_leg`): the reference library's reduce4 / simulate_block / reduce7 /
baseline_block_reduce (oracle/_ref, cli.cpp:195-266's loop) ns per call on
one core and aggregated over all cores (one process per core).

  python -m paper_2410_10447_b200.microbench [--blocks 64 128 256] [--cpu]
"""
from __future__ import annotations

import ctypes as C
import json
import os
import statistics
import time

import numpy as np

N_RED = 1_000_000
CHAIN = 100  # dependent reduce-and-broadcast steps per block (on-chip mode)
SEED = 12345  # cli.cpp:25
SMEM_BYTES_PER_CLK = 128  # per SM
N_SM = 148


def kernel_names(lib):
    return [lib.mdr_reduce_bench_kernel_name(k).decode() for k in range(lib.mdr_reduce_bench_kernels())]


def _peaks():
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    try:
        with open(os.path.join(root, "MEASURED_PEAKS.json")) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "MEASURED_PEAKS.json hbm_gbs"
    except (OSError, KeyError, ValueError):
        return 7700.0, "B200 nominal (MEASURED_PEAKS.json absent)"


def _sm_mhz():
    """SM clock now (nvidia-smi), for the cycle-based roofline and latency."""
    import subprocess

    try:
        out = subprocess.run(["nvidia-smi", "--query-gpu=clocks.sm", "--format=csv,noheader,nounits", "-i", "0"],
                             capture_output=True, text=True, timeout=10).stdout.strip().splitlines()
        return float(out[0])
    except (OSError, ValueError, IndexError, subprocess.TimeoutExpired):
        return 1965.0


def fill(dev, lib, x, label):
    rc = lib.mdr_fill_uniform_dev(dev.ctx, SEED, label.encode(), x.numel(), C.c_void_p(x.data_ptr()))
    assert rc == 0, lib.mdr_last_error(dev.ctx)


def reduce_microbench(dev, lib, torch, blocks=(64, 128, 256), n_red=N_RED, chain=CHAIN, reps=3):
    """Every bench kernel and the product entry points, per block size."""
    dev_idx = torch.cuda.current_device()
    stream = torch.cuda.current_stream()
    dev.set_stream(stream.cuda_stream)
    names = kernel_names(lib)
    hbm, hbm_src = _peaks()
    out = {"n_reductions": n_red, "chain_steps": chain, "kernels": names, "unit": "ns/reduction",
           "inputs": "uniform(-1,1) of derive_rng(12345, 'bench/<B>/float4'), draw (r B + t) 4 + c + 1 "
                     "(device-generated, identical to the reference RngStream)",
           "hbm_peak_GBps": hbm, "hbm_peak_source": hbm_src, "results": {}, "product": {}}

    def timed(go):
        go()
        torch.cuda.synchronize()
        best = float("inf")
        for _ in range(reps):
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(stream)
            go()
            b.record(stream)
            b.synchronize()
            best = min(best, a.elapsed_time(b))
        return best

    for B in blocks:
        res = {}
        n_stream = min(n_red, (4 << 30) // (16 * B))  # <= 4 GB of float4
        n_blocks = n_red // chain
        x = torch.empty((n_stream, B, 4), device=f"cuda:{dev_idx}")
        fill(dev, lib, x, f"bench/{B}/float4")  # the chain blocks use the stream's first n_blocks sets
        y = torch.empty((max(n_stream, n_blocks), 4), device=f"cuda:{dev_idx}")
        cyc = torch.zeros(n_blocks, dtype=torch.int64, device=f"cuda:{dev_idx}")
        ref = x[:2048].double().sum(1)
        mass = x[:2048].double().abs().sum(1)
        mhz = _sm_mhz()
        smem_peak = N_SM * SMEM_BYTES_PER_CLK * mhz * 1e6 / 1e9  # GB/s
        for k, name in enumerate(names):
            row = {}
            batched = "tcgen05" in name  # batched contraction: streaming only
            if not batched:
                ms = timed(lambda: lib.mdr_reduce_bench_dev(dev.ctx, k, B, C.c_void_p(x.data_ptr()), n_blocks * chain,
                                                            chain, C.c_void_p(y.data_ptr())))
                row["chain_ns"] = ms * 1e6 / (n_blocks * chain)
                rc = lib.mdr_reduce_bench_chain_cycles_dev(dev.ctx, k, B, C.c_void_p(x.data_ptr()), n_blocks * chain,
                                                           chain, C.c_void_p(y.data_ptr()), C.c_void_p(cyc.data_ptr()))
                assert rc == 0, lib.mdr_last_error(dev.ctx)
                torch.cuda.synchronize()
                cps = float(cyc.double().median().item()) / chain
                row["latency"] = {"cycles_per_step": cps, "ns_per_step": cps / mhz * 1e3, "sm_mhz": mhz}
                gbs = 16.0 * B / (row["chain_ns"] * 1e-9) / 1e9
                row["chain_roofline"] = {"bound": "smem", "achieved": gbs, "peak": smem_peak, "unit": "GB/s",
                                         "frac": gbs / smem_peak,
                                         "peak_source": f"148 SMs x 128 B/clk x {mhz:.0f} MHz (sampled)"}
            else:
                row["chain_ns"] = None
            ms = timed(lambda: lib.mdr_reduce_bench_dev(dev.ctx, k, B, C.c_void_p(x.data_ptr()), n_stream, 0,
                                                        C.c_void_p(y.data_ptr())))
            row["stream_ns"] = ms * 1e6 / n_stream
            gbs = 16.0 * B * n_stream / (ms * 1e-3) / 1e9
            row["stream_roofline"] = {"bound": "hbm", "achieved": gbs, "peak": hbm, "unit": "GB/s", "frac": gbs / hbm}
            err = ((y[:2048].double() - ref).abs() / mass.clamp_min(1e-30)).max().item()
            row["max_rel_err_vs_mass"] = err
            res[name] = row
        out["results"][str(B)] = res
        out["product"][str(B)] = product_entry_points(dev, lib, torch, x, B, n_stream, timed)
        del x, y, cyc
        torch.cuda.empty_cache()
    return out


def product_entry_points(dev, lib, torch, x, B, n, timed):
    """mdr_reduce4_dev / mdr_reduce7_dev (the library's reduce4 / reduce7,
    reduce.cpp:80-111 / 165-209) on the bench inputs, streaming mode."""
    from . import BASELINE, HALF, SINGLE, TCU, TCU_SPLIT

    y = torch.empty((n, 4), device=x.device)
    out = {}
    for name, method, accum, tc05 in (("reduce4 TcuSplit (tcgen05 route)", TCU_SPLIT, SINGLE, 1),
                                      ("reduce4 TcuSplit (warp mma.sync)", TCU_SPLIT, SINGLE, 0),
                                      ("reduce4 Tcu f16 (paper, Half)", TCU, HALF, 1),
                                      ("reduce4 Baseline (4 block trees)", BASELINE, SINGLE, 1)):
        lib.mdr_ctx_set_tc05(dev.ctx, tc05)
        routed = lib.mdr_reduce_uses_tc05(dev.ctx, method, B, n)

        def go():
            rc = lib.mdr_reduce4_dev(dev.ctx, C.c_void_p(x.data_ptr()), B, n, method, accum, C.c_void_p(y.data_ptr()))
            assert rc == 0, lib.mdr_last_error(dev.ctx)

        ms = timed(go)
        out[name] = {"stream_ns": ms * 1e6 / n, "GBps": 16.0 * B * n / (ms * 1e-3) / 1e9, "tcgen05": bool(routed)}
    lib.mdr_ctx_set_tc05(dev.ctx, 1)
    n7 = min(n, (2 << 30) // (28 * B))
    r7 = torch.empty((n7, B, 7), device=x.device)
    fill(dev, lib, r7, f"bench/{B}/partial7")
    y7 = torch.empty((n7, 7), device=x.device)
    for name, method, accum in (("reduce7 TcuSplit", TCU_SPLIT, SINGLE), ("reduce7 Tcu f16 (Half)", TCU, HALF),
                                ("reduce7 Baseline", BASELINE, SINGLE)):
        def go7():
            rc = lib.mdr_reduce7_dev(dev.ctx, C.c_void_p(r7.data_ptr()), B, n7, method, accum,
                                     C.c_void_p(y7.data_ptr()))
            assert rc == 0, lib.mdr_last_error(dev.ctx)

        ms = timed(go7)
        out[name] = {"stream_ns": ms * 1e6 / n7, "GBps": 28.0 * B * n7 / (ms * 1e-3) / 1e9,
                     "tcgen05": bool(lib.mdr_reduce_uses_tc05(dev.ctx, method, B, n7)), "n_reductions": n7}
    del r7, y7, y
    return out


# ------------------------------------------------------------- CPU leg
CPU_CASES = (  # (name, kind, method, accum, label suffix, components)
    ("reduce4 Tcu f16 (Half)", 0, 1, 0, "float4", 4),
    ("simulate_block Baseline (4 block trees)", 0, 0, 0, "float4", 4),
    ("reduce7 Baseline", 1, 0, 0, "partial7", 7),
    ("reduce7 Tcu f16 (Half)", 1, 1, 0, "partial7", 7),
    ("baseline_block_reduce (1 component)", 2, 0, 0, "float", 1),
)


def _cpu_case(args):
    """One process: the reference's call on n_sample input sets, looped for
    budget_s (ref_time_reduce in oracle/ref_shim.cpp)."""
    B, kind, method, accum, label, comps, n_sample, budget_s = args
    from oracle.oracle import Oracle

    lib = Oracle("reference").lib
    x = np.empty(n_sample * B * comps, np.float32)
    lib.ref_fill_uniform.argtypes = [C.c_uint64, C.c_char_p, C.c_int64, C.c_void_p]
    assert lib.ref_fill_uniform(SEED, label.encode(), x.size, x.ctypes.data) == 0
    ns, chk, calls = C.c_double(), C.c_double(), C.c_int64()
    lib.ref_time_reduce.argtypes = [C.c_int, C.c_int, C.c_int, C.c_int, C.c_void_p, C.c_int, C.c_double, C.c_void_p,
                                    C.c_void_p, C.c_void_p]
    assert lib.ref_time_reduce(kind, method, accum, B, x.ctypes.data, n_sample, budget_s, C.byref(ns), C.byref(chk),
                               C.byref(calls)) == 0
    return ns.value, calls.value


def cpu_leg(blocks=(64, 128, 256), n_sample=256, budget_s=1.0, procs=None):
    """The reference library's reductions on this host: ns per call on one
    core, and the aggregate rate with one process per core (CPU model and
    core count reported)."""
    import multiprocessing as mp

    from oracle.oracle import available

    if not available("reference"):
        return {"unavailable": "oracle/_ref not built (the reference sources are needed to build it)"}
    procs = procs or os.cpu_count() or 1
    model = "unknown"
    try:
        with open("/proc/cpuinfo") as f:
            model = next(line.split(":", 1)[1].strip() for line in f if line.startswith("model name"))
    except (OSError, StopIteration):
        pass
    out = {"cores": procs, "cpu_model": model, "kind": "reference", "unit": "ns/call",
           "sample": f"{n_sample} input sets per (case, B) from derive_rng(12345, 'bench/<B>/<float4|partial7|float>') "
                     f"(the GPU's inputs), each call looped for ~{budget_s:.1f} s", "results": {}}
    ctx = mp.get_context("fork")
    for B in blocks:
        row = {}
        for name, kind, method, accum, suffix, comps in CPU_CASES:
            label = f"bench/{B}/{suffix}"
            one = _cpu_case((B, kind, method, accum, label, comps, n_sample, budget_s))
            t0 = time.perf_counter()
            with ctx.Pool(procs) as pool:
                res = pool.map(_cpu_case, [(B, kind, method, accum, label, comps, n_sample, budget_s)] * procs)
            wall = time.perf_counter() - t0
            calls = sum(r[1] for r in res)
            row[name] = {"ns_per_call_1core": one[0], "ns_per_call_all_cores": statistics.mean(r[0] for r in res) / procs,
                         "calls_all_cores": calls, "wall_s": wall}
        out["results"][str(B)] = row
    return out


def main():
    import argparse

    import torch

    from . import Device
    from ._lib import load

    ap = argparse.ArgumentParser()
    ap.add_argument("--blocks", type=int, nargs="+", default=[64, 128, 256])
    ap.add_argument("--n", type=int, default=N_RED)
    ap.add_argument("--chain", type=int, default=CHAIN)
    ap.add_argument("--cpu", action="store_true", help="also run the CPU leg (reference library)")
    ap.add_argument("--kernel", type=int, default=-1, help="run only this kernel id once per mode (for ncu)")
    args = ap.parse_args()
    lib = load()
    dev = Device(0)
    s = torch.cuda.Stream()
    torch.cuda.set_stream(s)
    dev.set_stream(s.cuda_stream)
    if args.kernel >= 0:
        for B in args.blocks:
            stream_only = "tcgen05" in lib.mdr_reduce_bench_kernel_name(args.kernel).decode()
            n = min(args.n, (4 << 30) // (16 * B))
            x = torch.empty((n, B, 4), device="cuda")
            fill(dev, lib, x, f"bench/{B}/float4")
            y = torch.empty((n, 4), device="cuda")
            if not stream_only:
                lib.mdr_reduce_bench_dev(dev.ctx, args.kernel, B, C.c_void_p(x.data_ptr()),
                                         args.n // args.chain * args.chain, args.chain, C.c_void_p(y.data_ptr()))
            lib.mdr_reduce_bench_dev(dev.ctx, args.kernel, B, C.c_void_p(x.data_ptr()), n, 0, C.c_void_p(y.data_ptr()))
            torch.cuda.synchronize()
        return
    out = reduce_microbench(dev, lib, torch, tuple(args.blocks), args.n, args.chain)
    if args.cpu:
        out["cpu_leg"] = cpu_leg(tuple(args.blocks))
    print(json.dumps(out))


if __name__ == "__main__":
    main()
