"""Exact per-group torsion gradient of the analytic path
(mdr_ctx_set_exact_torsion).

score() projects the TOTAL torque on every torsion axis (reference
docking.cpp:228-231), a documented approximation; score_reference() gives
torsion k the torque of its own group (docking.cpp:244-268), which equals the
finite-difference gradient of the energy.  In exact mode the device stages
each atom's torque in warp scratch during the normal evaluation and the lane
owning entry 6+k sums group k.

Tolerances (written here):
  * energy and entries 0..5 (translation, orientation): bit-identical to the
    default mode — the exact option changes only the torsion entries;
  * entries 6.. vs score_reference (double): within 2e-6 * max(max|g|, 1) in
    the FP64 pair modes (float sums of float torques over <= 60 atoms), within
    1e-4 * max(max|g|, 1) in the FP32 pair mode;
  * entries 6.. vs central finite differences of the double oracle's energy:
    within 1e-4 * max(max|g|, 1) (the reference's FD gate, acceptance.cpp:149-208).
"""
import numpy as np
import pytest

from paper_2410_10447_b200 import (
    BASELINE,
    PAIR_FP32,
    PAIR_FP64,
    PAIR_FP64_FAST,
    SINGLE,
    TCU_SPLIT,
    Device,
    LgaSettings,
    SizeError,
)
from paper_2410_10447_b200._abi import derive_rng, random_instance, random_pose

pytestmark = pytest.mark.gpu


def bits(x):
    return np.asarray(x, np.float32).view(np.uint32)


def cases(seed, count):
    rng = derive_rng(seed, "gpu/exact")
    out = []
    for rep in range(count):
        inst = random_instance(rng, 1 + rep % 9, 3 + rng.next_index(58), 4 + rng.next_index(60))
        poses = np.stack([random_pose(rng, inst.n_rot, 1.0 if k % 2 else 0.4) for k in range(12)])
        out.append((inst, poses))
    return out


@pytest.mark.parametrize("pair", [PAIR_FP64, PAIR_FP64_FAST, PAIR_FP32])
@pytest.mark.parametrize("method", [BASELINE, TCU_SPLIT])
def test_exact_torsion_matches_score_reference(pair, method, port):
    approx = Device(0, pair=pair)
    exact = Device(0, pair=pair)
    exact.set_exact_torsion(True)
    tol = 1e-4 if pair == PAIR_FP32 else 2e-6
    changed = 0
    for inst, poses in cases(11 + pair, 8):
        ea, ga, ta, _ = approx.score_batch(inst, poses, method, SINGLE, 64)
        ex, gx, tx, _ = exact.score_batch(inst, poses, method, SINGLE, 64)
        assert np.array_equal(bits(ex), bits(ea))
        assert np.array_equal(bits(gx[:, :6]), bits(ga[:, :6]))
        assert np.array_equal(bits(tx), bits(ta))
        for i, p in enumerate(poses):
            _, wg, _ = port.score_reference(inst, p)
            scale = max(np.abs(wg).max(), 1.0)
            assert np.abs(gx[i, 6:] - wg[6:]).max(initial=0.0) <= tol * scale
            changed += inst.n_rot > 0 and not np.array_equal(bits(gx[i, 6:]), bits(ga[i, 6:]))
    assert changed > 0
    approx.close()
    exact.close()


def test_exact_torsion_finite_differences(port):
    dev = Device(0)
    dev.set_exact_torsion(True)
    h = 1e-6
    for inst, poses in cases(23, 6):
        _, grads, _, _ = dev.score_batch(inst, poses[:4], BASELINE, SINGLE, 64)
        for p, gr in zip(poses[:4], grads):
            fd = np.zeros(inst.n_rot)
            for k in range(inst.n_rot):
                a, b = p.copy(), p.copy()
                a[6 + k] += h
                b[6 + k] -= h
                fd[k] = (port.score_reference(inst, a)[0] - port.score_reference(inst, b)[0]) / (2 * h)
            scale = max(np.abs(gr).max(), 1.0)
            assert np.abs(gr[6:] - fd).max(initial=0.0) <= 1e-4 * scale
    dev.close()


def test_exact_torsion_rigid_and_untorsioned_atoms():
    """n_rot = 0 has no torsion entries; atoms with torsion -1 contribute to
    no group (score_reference's k >= 0 test)."""
    dev = Device(0)
    dev.set_exact_torsion(True)
    rng = derive_rng(3, "gpu/exact/rigid")
    inst = random_instance(rng, 0, 12, 16)
    poses = np.stack([random_pose(rng, 0, 0.5) for _ in range(8)])
    base = Device(0)
    assert np.array_equal(bits(dev.score_batch(inst, poses)[1]), bits(base.score_batch(inst, poses)[1]))
    dev.close()
    base.close()


def test_exact_torsion_local_search_and_lga(instances):
    dev = Device(0)
    dev.set_exact_torsion(True)
    inst = instances["synth20"]
    rng = derive_rng(41, "gpu/exact/ls")
    starts = np.stack([random_pose(rng, inst.n_rot, 0.6) for _ in range(64)])
    e0 = dev.score_batch(inst, starts)[0].astype(np.float64)
    r1 = dev.local_search_batch(inst, starts, 200, 1e-4, BASELINE, SINGLE, 64)
    r2 = dev.local_search_batch(inst, starts, 200, 1e-4, BASELINE, SINGLE, 64)
    e1 = np.array([r.energy for r in r1])
    assert np.array_equal(e1, np.array([r.energy for r in r2]))  # deterministic
    assert np.all(e1 <= e0 + 1e-6 * np.maximum(np.abs(e0), 1.0))
    s = LgaSettings()
    seeds = np.arange(8, dtype=np.uint64) + np.uint64(4040)
    a = dev.lga_run_batch(instances["s2"], BASELINE, SINGLE, s, seeds)
    b = dev.lga_run_batch(instances["s2"], BASELINE, SINGLE, s, seeds)
    assert [r.best_energy for r in a] == [r.best_energy for r in b]
    assert all(0 < r.evaluations for r in a)
    dev.close()


def test_exact_torsion_atom_limit():
    dev = Device(0)
    dev.set_exact_torsion(True)
    rng = derive_rng(5, "gpu/exact/limit")
    inst = random_instance(rng, 2, 1025, 4)
    with pytest.raises(SizeError):
        dev.score_batch(inst, np.stack([random_pose(rng, inst.n_rot, 0.5)]))
    dev.set_exact_torsion(False)
    dev.score_batch(inst, np.stack([random_pose(rng, inst.n_rot, 0.5)]))
    dev.close()
