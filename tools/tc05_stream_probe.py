import ctypes as C, json, os, sys
sys.path.insert(0, os.getcwd())
import torch
from paper_2410_10447_b200 import Device, SINGLE, TCU_SPLIT
from paper_2410_10447_b200._lib import load
from paper_2410_10447_b200.microbench import fill
lib = load(); dev = Device(0)
s = torch.cuda.Stream(); torch.cuda.set_stream(s); dev.set_stream(s.cuda_stream)
out = {}
for B in (64, 128, 256):
    n = min(1000000, (4 << 30) // (16 * B))
    x = torch.empty((n, B, 4), device="cuda"); fill(dev, lib, x, f"bench/{B}/float4")
    y = torch.empty((n, 4), device="cuda")
    def go(): assert lib.mdr_reduce4_dev(dev.ctx, C.c_void_p(x.data_ptr()), B, n, TCU_SPLIT, SINGLE, C.c_void_p(y.data_ptr())) == 0
    go(); torch.cuda.synchronize()
    best = 1e9
    for _ in range(5):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(s); go(); b.record(s); b.synchronize(); best = min(best, a.elapsed_time(b))
    ref = x[:4096].double().sum(1); mass = x[:4096].double().abs().sum(1)
    err = ((y[:4096].double() - ref).abs() / mass).max().item()
    out[B] = {"ns": best * 1e6 / n, "GBps": 16 * B * n / (best * 1e-3) / 1e9, "err": err}
    print(B, out[B], flush=True)
    del x, y; torch.cuda.empty_cache()
