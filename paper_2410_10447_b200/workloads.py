"""Synthetic workloads of BASELINE.json's configs, shared by
bench.py, the tools and the tests.  Everything is derived from the
reference's counter RNG (derive_rng, rng.hpp:41-43) and its random_instance
recipe (tests/test_docking.cpp:39-59), so CPU and GPU see identical inputs.

  C3  small ligand: 20 atoms, 5 torsions, 64 analytic sites   ("synth/small")
  C4  large flexible ligand: 100 atoms, 30 torsions ("synth/large"), in two
      forms: analytic (the reference's scoring against its 64 sites,
      partition 128) and grid mode on 126^3 maps at 0.375 A (4 atom types +
      electrostatic + desolvation), sampled from the 64 sites by
      mdr_grid_build; intramolecular pairs on
  C5  virtual screen: ligand j has U[10,100] atoms and U[0,30] torsions
      ("synth/lig/<j>") against the C4 receptor
"""
from __future__ import annotations

from ._abi import (
    LgaSettings,
    centered_grid,
    derive_rng,
    random_instance,
    random_ligand_params,
    random_receptor_fields,
)

SEED = 12345  # cli.cpp:25 kDefaultSeed
N_TYPES = 4


def c3():
    inst = random_instance(derive_rng(SEED, "synth/small"), 5, 20, 64)
    inst.name = "synth/small"
    return inst


def c4_analytic():
    """C4 in the reference's own (analytic) scoring: the C4 ligand (100 atoms,
    30 torsions) against its 64 sites, partition 128, so the
    reference library itself can dock it (docking.cpp:392-517)."""
    inst = random_instance(derive_rng(SEED, "synth/large"), 30, 100, 64)
    inst.name = "synth/large"
    return inst, LgaSettings(partition=128)


def c4_receptor(n: int = 126, spacing: float = 0.375, n_sites: int = 64):
    """Sites (as an instance carrying no ligand atoms of interest), receptor
    chemistry and the lattice shape of the C4 / C5 receptor."""
    sites = random_instance(derive_rng(SEED, "synth/large"), 30, 100, n_sites)
    fields = random_receptor_fields(derive_rng(SEED, "synth/large/receptor"), n_sites, N_TYPES)
    return sites, fields, centered_grid(n, spacing, N_TYPES)


def c4():
    """(instance, ligand params, receptor fields, grid shape, LGA settings)."""
    inst = random_instance(derive_rng(SEED, "synth/large"), 30, 100, 64)
    inst.name = "synth/large"
    params = random_ligand_params(derive_rng(SEED, "synth/large/chem"), inst.n_atoms, N_TYPES)
    _, fields, grid = c4_receptor()
    return inst, params, fields, grid, LgaSettings(partition=64)  # 64 measured faster than 128 (profiles/r1_c4_probe.json)


def c5_ligand(j: int, receptor_sites):
    """Ligand j of the virtual screen: natoms U[10,100], nrot U[0,30], the
    receptor's sites (which define the search box, docking.cpp:362-374)."""
    rng = derive_rng(SEED, f"synth/lig/{j}")
    natoms = 10 + rng.next_index(91)
    nrot = rng.next_index(31)
    lig = random_instance(rng, nrot, natoms, 0)
    lig.sites = receptor_sites.sites.copy()
    lig.name = f"synth/lig/{j}"
    params = random_ligand_params(derive_rng(SEED, f"synth/lig/{j}/chem"), natoms, N_TYPES)
    return lig, params


def partition_for(inst) -> int:
    """Grid-mode CTA size: a multiple of 32 covering the genotype and about
    one thread per atom (64 .. 256)."""
    need = max(6 + inst.n_rot, inst.n_atoms)
    return min(256, max(64, (need + 31) // 32 * 32))
