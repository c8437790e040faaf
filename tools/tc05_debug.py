"""Diagnose the tcgen05 batched reduction layout with structured inputs."""
import ctypes as C
import sys

import torch

sys.path.insert(0, ".")
from paper_2410_10447_b200 import Device  # noqa: E402

dev = Device(0)
lib = dev.lib
s = torch.cuda.Stream()
torch.cuda.set_stream(s)
dev.set_stream(s.cuda_stream)
B, n = 64, 32


def run(x):
    y = torch.zeros((n, 4), device="cuda")
    rc = lib.mdr_reduce_bench_dev(dev.ctx, 7, B, C.c_void_p(x.data_ptr()), n, 0, C.c_void_p(y.data_ptr()))
    assert rc == 0
    torch.cuda.synchronize()
    return y.cpu()


torch.set_printoptions(linewidth=200, precision=2, sci_mode=False)
x = torch.ones((n, B, 4), device="cuda")
print("ones ->", run(x)[:6].tolist())
x = torch.zeros((n, B, 4), device="cuda")
x[:, :, :] = torch.arange(4, device="cuda", dtype=torch.float32) + 1
print("c+1 ->", run(x)[:6].tolist())
x = torch.zeros((n, B, 4), device="cuda")
x[:, :, :] = (torch.arange(n, device="cuda", dtype=torch.float32) + 1)[:, None, None]
print("r+1 ->", run(x)[:8].tolist())
for t0 in (0, 1, 4, 8, 31, 32, 63):
    x = torch.zeros((n, B, 4), device="cuda")
    x[:, t0, :] = 1.0
    y = run(x)
    print("onehot t", t0, "->", y[:3].tolist(), "sum", float(y.sum()))
for r0, c0 in ((0, 0), (0, 1), (0, 3), (1, 0), (5, 2), (31, 3)):
    x = torch.zeros((n, B, 4), device="cuda")
    x[r0, :, c0] = 1.0
    y = run(x)
    nz = (y != 0).nonzero().tolist()
    print("onehot r,c", (r0, c0), "-> nonzero", nz[:8], [float(y[i][j]) for i, j in nz[:8]])
