"""Grid-map scoring mode: pin the CPU restatement (oracle/mdr_oracle.c,
orc_grid_*) before it is used as the checker of the device kernels.

There is no reference implementation of this mode (SPEC.md:425 puts grid maps
out of scope), so it is pinned three ways:
  * against the reference itself: type-0 maps are sampled from the
    reference's analytic well, so a grid-mode score without charges or
    intramolecular terms must converge to the reference's score_reference
    (oracle/_ref) as the lattice is refined, and equal it at lattice points;
  * the exact gradient (translation, Euler axes, per-group torsion torque with
    the intramolecular forces) against central finite differences;
  * the LGA / local-search control flow is the one pinned bit-for-bit by
    tests/test_oracle.py (shared lga_core / ls_core).
"""
import numpy as np
import pytest

from paper_2410_10447_b200._abi import (
    GRID_OUTSIDE_K,
    Grid,
    Instance,
    LgaSettings,
    LigandParams,
    centered_grid,
    derive_rng,
    random_instance,
    random_ligand_params,
    random_pose,
    random_receptor_fields,
)


def _setup(n_atoms=20, n_rot=5, n_sites=16, n=41, spacing=0.375, n_types=4, seed=7):
    inst = random_instance(derive_rng(seed, "grid/inst"), n_rot, n_atoms, n_sites)
    rf = random_receptor_fields(derive_rng(seed, "grid/rec"), n_sites, n_types)
    lp = random_ligand_params(derive_rng(seed, "grid/lig"), n_atoms, n_types)
    return inst, rf, lp, centered_grid(n, spacing, n_types)


@pytest.fixture(scope="module")
def small(port):
    inst, rf, lp, G = _setup()
    G.maps = port.grid_build(inst, rf, G)
    return inst, rf, lp, G


def _fd(port, inst, G, lp, g, h=1e-6):
    fd = np.zeros(inst.dim)
    for d in range(inst.dim):
        gp, gm = g.copy(), g.copy()
        gp[d] += h
        gm[d] -= h
        fd[d] = (port.grid_score(inst, G, lp, gp)[0] - port.grid_score(inst, G, lp, gm)[0]) / (2 * h)
    return fd


@pytest.mark.parametrize("intra", [True, False])
def test_grid_gradient_matches_finite_differences(port, small, intra):
    inst, rf, lp, G = small
    lp = LigandParams(lp.atom_type, lp.charge, lp.radius, lp.epsilon, lp.elec_scale, intra)
    rng = derive_rng(11, "grid/fd")
    for k in range(12):
        g = random_pose(rng, inst.n_rot, 3.0 if k < 9 else 9.0)  # the last poses leave the lattice
        e, grad, _, ei = port.grid_score(inst, G, lp, g)
        if not intra:
            assert ei == 0.0
        fd = _fd(port, inst, G, lp, g)
        # piecewise-trilinear energy: exact away from cell faces; tolerance 1e-6 of the gradient scale
        assert np.abs(fd - grad).max() <= 1e-6 * max(1.0, np.abs(grad).max()), (k, fd, grad)


def test_grid_torsion_gradient_is_exact_per_group(port, small):
    """Each torsion entry is the torque of its own group (score_reference
    semantics, docking.cpp:244-268), not the total torque of score()."""
    inst, rf, lp, G = small
    g = random_pose(derive_rng(3, "grid/tors"), inst.n_rot, 2.0)
    _, grad, tq, _ = port.grid_score(inst, G, lp, g)
    fd = _fd(port, inst, G, lp, g)
    assert np.allclose(grad[6:], fd[6:], rtol=0, atol=1e-6 * max(1.0, np.abs(grad).max()))


def test_grid_builder_type0_is_reference_well(ref):
    """Type-0 map value at a lattice point == the reference's analytic site
    energy of a unit-weight atom there (score_reference, docking.cpp:235-270)."""
    from oracle.oracle import Oracle

    port = Oracle("port")
    inst, rf, lp, G = _setup(n=9, spacing=0.5)
    G.maps = port.grid_build(inst, rf, G)
    pts = [(0, 0, 0), (4, 4, 4), (8, 1, 3), (2, 7, 5)]
    for ix, iy, iz in pts:
        p = np.array(G.origin) + G.spacing * np.array([ix, iy, iz])
        one = Instance(np.array([[0.0, 0.0, 0.0, 1.0]]), np.array([-1]), inst.sites, 0)
        e_ref, _, _ = ref.score_reference(one, np.array([p[0], p[1], p[2], 0.0, 0.0, 0.0]))
        assert G.maps[0, iz, iy, ix] == np.float32(e_ref)


def test_grid_converges_to_reference_analytic_score(ref, port):
    """Charges off, intramolecular off, all atoms type 0: the grid energy and
    gradient converge to the reference's analytic score_reference as the
    lattice is refined: energy at second order (trilinear error O(h^2)),
    gradient at first order (the interpolant's derivative is piecewise
    linear along each axis)."""
    inst = random_instance(derive_rng(5, "grid/conv"), 3, 12, 8)
    rf = random_receptor_fields(derive_rng(5, "grid/conv/rec"), inst.n_sites, 1)
    lp = LigandParams(np.zeros(inst.n_atoms), np.zeros(inst.n_atoms), np.full(inst.n_atoms, 0.4),
                      np.full(inst.n_atoms, 0.05), intra=False)
    poses = [random_pose(derive_rng(5, "grid/conv/pose"), inst.n_rot, 2.0)]
    rng = derive_rng(6, "grid/conv/pose")
    poses += [random_pose(rng, inst.n_rot, 2.0) for _ in range(5)]
    errs = {}
    for spacing in (0.2, 0.1, 0.05):
        G = centered_grid(int(round(10.0 / spacing)) + 1, spacing, 1)
        G.maps = port.grid_build(inst, rf, G)
        e_err, g_err = [], []
        for g in poses:
            e, grad, _, _ = port.grid_score(inst, G, lp, g)
            e_ref, grad_ref, _ = ref.score_reference(inst, g)
            e_err.append(abs(e - e_ref) / max(1.0, abs(e_ref)))
            g_err.append(np.abs(grad - grad_ref).max() / max(1.0, np.abs(grad_ref).max()))
        errs[spacing] = (np.mean(e_err), np.mean(g_err))
    assert errs[0.2][0] / errs[0.05][0] > 8.0 and errs[0.2][1] / errs[0.05][1] > 2.5, errs
    assert errs[0.05][0] < 0.01 and errs[0.05][1] < 0.08, errs


def test_grid_outside_restraint(port, small):
    """An atom beyond the lattice pays k_out |p - clamp(p)|^2 and is pushed back."""
    inst, rf, lp, G = small
    one = Instance(np.array([[0.0, 0.0, 0.0, 1.0]]), np.array([-1]), inst.sites, 0)
    lp1 = LigandParams(np.array([0]), np.array([0.0]), np.array([0.4]), np.array([0.05]))
    edge = np.array(G.origin) + G.spacing * (np.array(G.shape) - 1)
    g_in = np.array([edge[0], 0.0, 0.0, 0.0, 0.0, 0.0])
    g_out = g_in + np.array([1.5, 0, 0, 0, 0, 0])
    e_in, grad_in, _, _ = port.grid_score(one, G, lp1, g_in)
    e_out, grad_out, _, _ = port.grid_score(one, G, lp1, g_out)
    assert e_out == pytest.approx(e_in + GRID_OUTSIDE_K * 1.5 ** 2, rel=1e-12, abs=1e-9)
    assert grad_out[0] == pytest.approx(2 * GRID_OUTSIDE_K * 1.5, rel=1e-12)


def test_grid_local_search_descends(port, small):
    inst, rf, lp, G = small
    rng = derive_rng(9, "grid/ls")
    for _ in range(4):
        g = random_pose(rng, inst.n_rot, 2.0)
        e0 = port.grid_score(inst, G, lp, g)[0]
        r = port.grid_local_search(inst, G, lp, g, 150, 1e-4)
        assert r["energy"] <= e0
        assert port.grid_score(inst, G, lp, r["genotype"])[0] == pytest.approx(r["energy"], rel=1e-12)


def test_grid_lga_is_deterministic_and_tracks_best(port, small):
    inst, rf, lp, G = small
    s = LgaSettings(generations=3)
    a = port.grid_lga_run(inst, G, lp, s, 20260816)
    b = port.grid_lga_run(inst, G, lp, s, 20260816)
    assert a["best_energy"] == b["best_energy"] and a["evaluations"] == b["evaluations"]
    assert np.array_equal(a["best_genotype"], b["best_genotype"])
    assert a["best_energy"] <= min(r[0] for r in a["runs"])
    assert port.grid_score(inst, G, lp, a["best_genotype"])[0] == pytest.approx(a["best_energy"], rel=1e-12)


def test_grid_oracle_correctly_rounded_math():
    """The grid-mode oracle's sin / cos / log (oracle/crmath.h, correctly
    rounded) agree with glibc except where glibc itself is not correctly
    rounded (~0.1 % of calls), and then by one ulp."""
    import math

    from oracle.oracle import cr_values

    n = 20000
    v = cr_values(0, n)
    mix = lambda z: _mix64(z)  # noqa: E731
    off = 0
    for i in range(n):
        a = -math.pi + 2.0 * math.pi * ((mix(((4 * i + 1) * 0x9E3779B97F4A7C15) & M64) >> 11) * 2.0**-53)
        u1 = ((mix(((4 * i + 2) * 0x9E3779B97F4A7C15) & M64) >> 11) + 1) * 2.0**-53
        z = 2.0 * math.pi * ((mix(((4 * i + 3) * 0x9E3779B97F4A7C15) & M64) >> 11) * 2.0**-53)
        for got, want in zip(v[i], (math.sin(a), math.cos(a), math.log(u1), math.cos(z))):
            if got != want:
                off += 1
                assert abs(got - want) <= math.ulp(want), (i, got, want)
    assert off <= 0.01 * 4 * n, off


M64 = (1 << 64) - 1


def _mix64(z):
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9 & M64
    z = (z ^ (z >> 27)) * 0x94D049BB133111EB & M64
    return z ^ (z >> 31)
