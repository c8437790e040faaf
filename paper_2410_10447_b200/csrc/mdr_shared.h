// mdr_shared.h — plain structs shared by host (capi.cpp) and device code.
#pragma once

#include <stdint.h>

#include "mdr.h"

#include <vector_types.h>  // double4 / float4 / float2 for host and device

namespace mdr {

// Limits of the device path (documented in DESIGN.md; validated by capi.cpp
// before any launch, reported as MDR_ERR_SIZE).
constexpr int kMaxDim = 64;        // genotype dimensions: lanes d and d + 32
constexpr int kMaxRot = kMaxDim - 6;
constexpr int kMaxSites = 2048;    // per-CTA shared-memory copy
constexpr int kMaxAtoms = 4096;
constexpr int kWindow = 16;        // local_search convergence window, docking.cpp:314
constexpr int kMaxExactAtoms = 1024;
constexpr int kMaxChunkItems = 256;        // policy limit (pick_chunks / pick_search_items)
constexpr int kMaxChunkItemsForced = 512;  // with a pinned chunk length (timing / tests)
//    // atoms x site chunks staged per warp (32 B each)  // exact-torsion mode stages one float4 torque per atom per warp

// One receptor site with the two pair-loop constants precomputed on the host
// in the reference's evaluation order (docking.cpp:114-116):
//   c2 = 0.5625 * d0 * d0 ; num = d0 * d0 + c2.
struct SiteD {
  double x, y, z, depth, c2, num;
};

// Device view of an uploaded ligand / receptor pair.
struct LigandView {
  int n_atoms, n_sites, n_rot;
  int exact_torsion;  // 1: torsion gradient = exact per-group torque (mdr_ctx_set_exact_torsion)
  int n_chunks;       // FP64-fast: sites split into n_chunks ranges of chunk_len (1 = lane per atom)
  int chunk_len;
  int ls_pair;        // 1: Lamarckian searches may run on several warps (MDR_LS_PAIR=0: one warp)
  int ls_warps;       // Lamarckian search form of the LGA (mdr_ctx_set_ls_warps): 3 pool, 2 helper, 1 one warp, 0 legacy
  int ls_n_chunks;    // site chunking of that search (its own lane count), see capi.cpp pick_chunks
  int ls_chunk_len;
  int pad_;
  int ls_group;       // atoms per chunk item of that search (register blocking: 1 or 3)
  const SiteD* sites;
  const double4* atoms;  // local x, y, z, weight
  const int* tors;
  const double* taxes;      // torsion_axis(k) computed on the host (glibc)
  const float4* sites_f;    // fast-mode copy: x, y, z, depth
  const float2* sites_f2;   // fast-mode copy: c2, num
  const double* box;        // device: lo[3], hi[3] random_genotype bounds incl. margin
};

// Grid-map scoring mode (mdr.h).  Maps are FP32,
// [(n_types + 2)][nz][ny][nx] (type maps, electrostatic, desolvation).
struct GridView {
  int nx, ny, nz, n_types;
  double ox, oy, oz, h, inv_h;
  long long stride;  // nx * ny * nz
  const float* maps;
};

// Ligand chemistry of grid mode, prepared on the host (capi.cpp):
//   chem[i] = {radius_i, sqrt(epsilon_i), charge_i, elec_scale * charge_i};
//   grp_atoms: the torsioned atoms grouped by torsion (ascending k, then
//   ascending atom index), grp_off[k] .. grp_off[k + 1] delimiting group k.
struct FlexView {
  const int* type;
  const float4* chem;
  const double4* chem64;  // {radius, epsilon, charge, 0} in double (strict FP64 grid mode; single-ligand calls)
  double elec_scale;
  const int* grp_off;    // n_rot + 1
  const int* grp_atoms;  // n_tors_atoms
  int n_tors_atoms, intra;
};

// Per-run ligand tables of a grid-mode LGA batch (device arrays): one
// ligand (run_lig == nullptr) or a virtual-screen batch (run r docks ligand
// run_lig[r]).
struct GridLigands {
  const LigandView* L;
  const FlexView* F;
  const int* run_lig;
};

// All device state of a batch of LGA runs (docking.cpp:392-517).
struct LgaDev {
  int R, P, dim, off, L, gens, ls_iters, maxrec, partition, half_mode;
  long long max_evals;
  double tol, sigma;
  uint64_t label_hash;  // mix64(fnv1a64("lga")), rng.cpp:31-32
  const uint64_t* seeds;
  double* pop[2];   // [R][P][dim]
  double* pope[2];  // [R][P]
  int* cur;         // [R]
  double* lsg;      // [R][L][dim]
  double* lse;      // [R][L]
  int* lsit;        // [R][L]
  int* lscv;        // [R][L]
  int* lstarget;    // [R][L]
  double* best_e;   // [R]
  double* best_g;   // [R][dim]
  long long* evals; // [R]
  int* active;      // [R]
  int* nrec;        // [R]
  mdr_ls_record* recs;  // [R][maxrec]
  int* conv;        // [R]
  int* status;      // [R]
  int* ls_next;     // [gens + 1]: next search of generation g / next polish ([gens]) for the persistent search kernel (zeroed at init)
  int* ls_done;     // [R]: searches of the current generation finished per run (persistent search kernel; the last one finalizes)
};

}  // namespace mdr
