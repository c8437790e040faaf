"""RMSD clustering of docked poses.

CPU part: the oracle's pose -> coordinates transform is pinned to the
reference (the reference's own analytic energy, recomputed from those
coordinates, equals score_reference bit for bit up to summation order), and
its clustering to an independent Python restatement of AutoDock's rule.
GPU part (-m gpu): the device coordinates match the oracle to 1e-12 and the
cluster assignment is identical (RMSDs to 1e-9)."""
import numpy as np
import pytest

from paper_2410_10447_b200._abi import derive_rng, random_instance, random_pose


def _energy_from_coords(inst, xyz):
    """The reference's site well (docking.cpp:109-123) at given coordinates."""
    e = 0.0
    for (x, y, z, w), p in zip(inst.atoms, xyz):
        for sx, sy, sz, depth, d0 in inst.sites:
            dx, dy, dz = p[0] - sx, p[1] - sy, p[2] - sz
            c2 = 0.5625 * d0 * d0
            u = dx * dx + dy * dy + dz * dz + c2
            rho2 = (d0 * d0 + c2) / u
            rho6 = rho2 ** 3
            e += w * depth * (rho6 * rho6 - 2 * rho6)
    return e


def test_pose_coords_reproduce_reference_energy(port, ref):
    inst = random_instance(derive_rng(3, "cl/inst"), 4, 15, 6)
    rng = derive_rng(3, "cl/pose")
    for _ in range(5):
        g = random_pose(rng, inst.n_rot, 2.0)
        xyz = port.pose_coords(inst, g)
        e_ref, _, _ = ref.score_reference(inst, g)
        assert _energy_from_coords(inst, xyz) == pytest.approx(e_ref, rel=1e-12, abs=1e-12)


def _cluster_py(xyz, energy, tol):
    order = sorted(range(len(energy)), key=lambda i: (energy[i], i))
    seeds, cl, rm = [], [0] * len(energy), [0.0] * len(energy)
    for p in order:
        for k, s in enumerate(seeds):
            r = float(np.sqrt(((xyz[p] - xyz[s]) ** 2).sum() / xyz.shape[1]))
            if r < tol:
                cl[p], rm[p] = k, r
                break
        else:
            cl[p] = len(seeds)
            seeds.append(p)
    return np.array(cl), np.array(rm), len(seeds)


def _pose_family(inst, n, seed):
    """Poses around a few centres so that clusters of several members form."""
    rng = derive_rng(seed, "cl/family")
    centres = [random_pose(rng, inst.n_rot, 3.0) for _ in range(4)]
    poses, energies = [], []
    for k in range(n):
        c = centres[rng.next_index(4)]
        poses.append(c + np.array([rng.uniform(-0.6, 0.6) for _ in range(inst.dim)]))
        energies.append(rng.uniform(-10.0, 0.0))
    return np.array(poses), np.array(energies)


@pytest.mark.parametrize("tol", [0.5, 1.0, 2.0])
def test_oracle_clustering_matches_python_restatement(port, tol):
    inst = random_instance(derive_rng(4, "cl/inst"), 5, 20, 8)
    poses, energies = _pose_family(inst, 60, 4)
    c, r, nc = port.cluster_poses(inst, poses, energies, tol)
    xyz = np.stack([port.pose_coords(inst, g) for g in poses])
    wc, wr, wnc = _cluster_py(xyz, energies, tol)
    assert nc == wnc and np.array_equal(c, wc)
    assert np.allclose(r, wr, rtol=0, atol=1e-12)
    assert c[np.argmin(energies)] == 0 and 1 < nc < len(poses)


def test_clustering_edge_cases(port):
    inst = random_instance(derive_rng(5, "cl/inst"), 2, 6, 4)
    g = random_pose(derive_rng(5, "cl/p"), inst.n_rot, 1.0)
    # identical poses: one cluster, rmsd 0; equal energies keep index order
    c, r, nc = port.cluster_poses(inst, np.stack([g, g, g]), np.array([1.0, 1.0, 0.5]), 2.0)
    assert nc == 1 and list(c) == [0, 0, 0] and np.all(r == 0)
    # a rigid translation by d gives rmsd exactly d: split at tol == d (strict <)
    h = g.copy()
    h[0] += 1.5
    c, r, nc = port.cluster_poses(inst, np.stack([g, h]), np.array([0.0, 1.0]), 1.5)
    assert nc == 2
    c, r, nc = port.cluster_poses(inst, np.stack([g, h]), np.array([0.0, 1.0]), 1.5 + 1e-9)
    assert nc == 1 and r[1] == pytest.approx(1.5, rel=1e-12)


@pytest.mark.gpu
def test_device_coords_and_clustering_match_oracle(port, dev):
    inst = random_instance(derive_rng(6, "cl/inst"), 8, 40, 8)
    poses, energies = _pose_family(inst, 200, 6)
    xyz = dev.pose_coords(inst, poses)
    want = np.stack([port.pose_coords(inst, g) for g in poses])
    assert np.abs(xyz - want).max() <= 1e-12
    for tol in (0.75, 2.0):
        c, r, nc = dev.cluster_poses(inst, poses, energies, tol)
        wc, wr, wnc = port.cluster_poses(inst, poses, energies, tol)
        assert nc == wnc and np.array_equal(c, wc)
        assert np.abs(r - wr).max() <= 1e-9


@pytest.mark.gpu
def test_lga_batch_clustering(port, dev, instances):
    """Best poses of 32 device LGA runs, clustered on the device, equal the
    oracle's clustering of the same poses."""
    import ctypes as C

    from paper_2410_10447_b200 import BASELINE, SINGLE
    from paper_2410_10447_b200._abi import LgaSettings

    inst = instances["s3"]
    s = LgaSettings(generations=4)
    lib = dev.lib
    di = lib.mdr_instance_upload(dev.ctx, inst.cref())
    b = lib.mdr_lga_batch_create(dev.ctx, di, BASELINE, SINGLE, C.byref(s), 32)
    import torch

    seeds = torch.arange(32, dtype=torch.int64, device="cuda") + 77
    assert lib.mdr_lga_batch_run_dev(dev.ctx, b, C.c_void_p(seeds.data_ptr())) == 0
    be, bg = np.zeros(32), np.zeros((32, inst.dim))
    assert lib.mdr_lga_batch_download(dev.ctx, b, be.ctypes.data, bg.ctypes.data, None, None, None, None,
                                      None) == 0
    c = np.zeros(32, np.int32)
    r = np.zeros(32)
    nc = np.zeros(1, np.int32)
    assert lib.mdr_lga_batch_cluster(dev.ctx, b, 1.0, c.ctypes.data, r.ctypes.data, nc.ctypes.data) == 0
    wc, wr, wnc = port.cluster_poses(inst, bg, be, 1.0)
    assert int(nc[0]) == wnc and np.array_equal(c, wc) and np.abs(r - wr).max() <= 1e-9
    lib.mdr_lga_batch_destroy(dev.ctx, b)
    lib.mdr_instance_free(dev.ctx, di)
