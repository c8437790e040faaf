#!/usr/bin/env python3
"""Streaming-mode C2 reductions under the libraries named on the command
line (MDR_LIB_PATH per subprocess): ns per reduction and HBM fraction for
every non-batched kernel at B = 64 / 128 / 256 (prefetch-depth A/B)."""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CHILD = r"""
import ctypes as C, json, sys
sys.path.insert(0, %r)
import torch
from paper_2410_10447_b200 import Device
from paper_2410_10447_b200._lib import load
from paper_2410_10447_b200.microbench import fill
lib = load(); dev = Device(0); s = torch.cuda.Stream(); torch.cuda.set_stream(s); dev.set_stream(s.cuda_stream)
out = {}
for B in (64, 128, 256):
    n = min(1_000_000, (4 << 30) // (16 * B))
    x = torch.empty((n, B, 4), device="cuda"); fill(dev, lib, x, f"bench/{B}/float4")
    y = torch.empty((n, 4), device="cuda")
    for k in (0, 1, 2, 5, 6):
        call = lambda: lib.mdr_reduce_bench_dev(dev.ctx, k, B, C.c_void_p(x.data_ptr()), n, 0, C.c_void_p(y.data_ptr()))
        call(); torch.cuda.synchronize(); ms = []
        for _ in range(5):
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(s); call(); b.record(s); b.synchronize(); ms.append(a.elapsed_time(b))
        t = sorted(ms)[2]
        out[f"{B}/{lib.mdr_reduce_bench_kernel_name(k).decode()}"] = {"ns": t * 1e6 / n, "GBps": 16.0 * B * n / (t * 1e-3) / 1e9}
print(json.dumps(out))
""" % ROOT

res = {}
for lib in sys.argv[1:]:
    env = dict(os.environ, MDR_LIB_PATH=lib)
    p = subprocess.run([sys.executable, "-c", CHILD], env=env, capture_output=True, text=True, cwd=ROOT)
    res[lib] = json.loads(p.stdout.strip().splitlines()[-1]) if p.returncode == 0 else {"error": p.stderr[-1500:]}
os.makedirs(os.path.join(ROOT, "gpurun_out"), exist_ok=True)
json.dump(res, open(os.path.join(ROOT, "gpurun_out", "stream_prefetch_ab.json"), "w"), indent=1)
keys = list(next(iter(res.values())).keys())
for k in keys:
    print(k.ljust(40), "  ".join(f"{res[l][k]['GBps']:8.0f}" if k in res[l] else "   n/a" for l in res))
