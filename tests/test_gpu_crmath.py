"""Correctly rounded device sin / cos / log (csrc/crmath.cuh) against this
host's glibc (the reference's libm).  glibc agrees with an 80-bit reference
to within ~0.1 %, so a correctly rounded implementation must match it on at
least 99.7 % of calls, where CUDA libdevice matches on 83-89 % (sin / cos)."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def test_crmath_matches_glibc(dev):
    n = 1 << 21
    m = np.zeros(8, np.uint64)
    assert dev.lib.mdr_selftest_crmath(dev.ctx, n, m.ctypes.data) == 0
    cr, lib = m[:4] / n, m[4:] / n
    assert np.all(cr <= 3e-3), cr  # measured 1.4e-3 (sin/cos), 0.8e-3 (log) over 2^24
    assert np.all(cr[[0, 1, 3]] * 20 < lib[[0, 1, 3]]), (cr, lib)


def test_strict_mode_lga_bit_parity(dev_ref, port, instances):
    """Strict FP64 mode (reference operation order + correctly rounded trig
    and Box-Muller draws): paired-seed LGA runs equal the reference's."""
    from paper_2410_10447_b200 import BASELINE, SINGLE, LgaSettings

    inst = instances["s1"]
    s = LgaSettings()
    seeds = np.arange(30, dtype=np.uint64) + 777000
    gpu = dev_ref.lga_run_batch(inst, BASELINE, SINGLE, s, seeds)
    same = sum(g.best_energy == c["best_energy"] and g.evaluations == c["evaluations"]
               for g, c in zip(gpu, (port.lga_run(inst, BASELINE, SINGLE, s, int(x)) for x in seeds)))
    assert same >= 29, same  # 99/100 measured (profiles/r1_parity_scale.json); libdevice trig: 80/100
