"""Correctness of the C2 microbench kernels (bench_reduce.cu) on small inputs:
every kernel must return the block sums (reduce-and-broadcast), within f16
accuracy for the paper's f16 method and fp32 accuracy for the others."""
import ctypes as C

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

# max |err| / sum|x| per kernel (K2 = the paper's f16 accumulator)
TOL = {0: 1e-6, 1: 1e-6, 2: 2e-2, 3: 1e-6, 4: 1e-6, 5: 1e-6, 6: 1e-6, 7: 1e-6, 8: 1e-6}


@pytest.mark.parametrize("block", [64, 128, 256, 1024])
def test_microbench_kernels_sum_correctly(dev, block):
    import torch

    lib = dev.lib
    s = torch.cuda.Stream()
    torch.cuda.set_stream(s)
    dev.set_stream(s.cuda_stream)
    n = 512
    x = (torch.rand((n, block, 4), device="cuda", generator=torch.Generator("cuda").manual_seed(block)) * 2 - 1)
    y = torch.zeros((n, 4), device="cuda")
    want = x.double().sum(1)
    mass = x.double().abs().sum(1)
    for k in range(lib.mdr_reduce_bench_kernels()):
        for steps in ((0,) if k in (7, 8) else (0, 1)):  # streaming, and chain of length 1
            y.zero_()
            rc = lib.mdr_reduce_bench_dev(dev.ctx, k, block, C.c_void_p(x.data_ptr()), n, steps,
                                          C.c_void_p(y.data_ptr()))
            assert rc == 0
            torch.cuda.synchronize()
            err = ((y.double() - want).abs() / mass).max().item()
            assert err <= TOL[k], (k, steps, err)
    # chain of 4 steps: v += 2^-20 * sum each step; check against a numpy model
    steps = 4
    xc = x[: n // steps].contiguous()
    y.zero_()
    assert lib.mdr_reduce_bench_dev(dev.ctx, 1, block, C.c_void_p(xc.data_ptr()), n, steps,
                                    C.c_void_p(y.data_ptr())) == 0
    torch.cuda.synchronize()
    v = xc.double().cpu().numpy()
    for _ in range(steps):
        sm = v.sum(1, keepdims=True)
        v = v + 2.0**-20 * sm
    got = y[: n // steps].double().cpu().numpy()
    assert np.allclose(got, sm[:, 0, :], rtol=1e-5, atol=1e-4)
    torch.cuda.set_stream(torch.cuda.default_stream())
    dev.set_stream(None)
