"""C2 microbench driver: block float4 sum-reduction, MMA vs warp-shuffle
(BASELINE.json configs[1]: block 64/128/256, 10^6 reductions).

Inputs follow SURVEY §8d: component c of thread t of reduction r is
uniform(-1, 1) — generated here with a seeded numpy stream (the bench never
hashes in-kernel) and resident in HBM before timing.

  python -m paper_2410_10447_b200.microbench [--blocks 64 128 256] [--json]
"""
from __future__ import annotations

import ctypes as C
import json

import numpy as np

N_RED = 1_000_000
CHAIN = 100  # dependent reduce-and-broadcast steps per block (on-chip mode)


def kernel_names(lib):
    return [lib.mdr_reduce_bench_kernel_name(k).decode() for k in range(lib.mdr_reduce_bench_kernels())]


def reduce_microbench(dev, lib, torch, blocks=(64, 128, 256), n_red=N_RED, chain=CHAIN, reps=3):
    """ns per reduction for every kernel, on-chip chain mode and HBM streaming
    mode; plus each kernel's max relative error on one checked batch."""
    dev_idx = torch.cuda.current_device()
    stream = torch.cuda.current_stream()
    dev.set_stream(stream.cuda_stream)
    names = kernel_names(lib)
    out = {"n_reductions": n_red, "chain_steps": chain, "kernels": names, "unit": "ns/reduction", "results": {}}
    gen = torch.Generator(device=f"cuda:{dev_idx}").manual_seed(12345)
    for B in blocks:
        res = {}
        # streaming input: n_red x B float4 (16 B * B * n_red); cap at ~4 GB
        n_stream = min(n_red, (4 << 30) // (16 * B))
        x_stream = torch.rand((n_stream, B, 4), device=f"cuda:{dev_idx}", generator=gen) * 2 - 1
        n_blocks = n_red // chain
        x_chain = torch.rand((n_blocks, B, 4), device=f"cuda:{dev_idx}", generator=gen) * 2 - 1
        y = torch.empty((max(n_stream, n_blocks), 4), device=f"cuda:{dev_idx}")
        ref = x_stream[:2048].double().sum(1)
        mass = x_stream[:2048].double().abs().sum(1)
        for k, name in enumerate(names):
            row = {}
            modes = (("chain", x_chain, n_blocks * chain, chain), ("stream", x_stream, n_stream, 0))
            if "tcgen05" in name:  # batched kernel: streaming only
                modes = modes[1:]
                row["chain_ns"] = None
            for mode, x, n, steps in modes:
                def go():
                    rc = lib.mdr_reduce_bench_dev(dev.ctx, k, B, C.c_void_p(x.data_ptr()), n, steps,
                                                  C.c_void_p(y.data_ptr()))
                    assert rc == 0, lib.mdr_last_error(dev.ctx)

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
                row[mode + "_ns"] = best * 1e6 / n
                row[mode + "_ms"] = best
                if mode == "stream":
                    # streamed bytes / time against measured HBM
                    row["stream_GBps"] = 16.0 * B * n / (best * 1e-3) / 1e9
                    err = ((y[:2048].double() - ref).abs() / mass.clamp_min(1e-30)).max().item()
                    row["max_rel_err_vs_mass"] = err
            res[name] = row
        out["results"][str(B)] = res
        del x_stream, x_chain, y
        torch.cuda.empty_cache()
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
    ap.add_argument("--kernel", type=int, default=-1, help="run only this kernel id once per mode (for ncu)")
    args = ap.parse_args()
    lib = load()
    dev = Device(0)
    s = torch.cuda.Stream()
    torch.cuda.set_stream(s)
    if args.kernel >= 0:
        for B in args.blocks:
            if args.chain == 0 or args.kernel in (7, 8):  # streaming mode
                args.chain = 0
                args.n = min(args.n, (4 << 30) // (16 * B))
            x = torch.rand((args.n // max(args.chain, 1), B, 4), device="cuda") * 2 - 1
            y = torch.empty((args.n, 4), device="cuda")
            dev.set_stream(s.cuda_stream)
            lib.mdr_reduce_bench_dev(dev.ctx, args.kernel, B, C.c_void_p(x.data_ptr()), args.n, args.chain,
                                     C.c_void_p(y.data_ptr()))
            torch.cuda.synchronize()
        return
    print(json.dumps(reduce_microbench(dev, lib, torch, tuple(args.blocks), args.n, args.chain)))


if __name__ == "__main__":
    main()
