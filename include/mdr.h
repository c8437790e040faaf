/*
 * mdr.h — C-ABI of the B200 scoring / reduction / ADADELTA / LGA hot path.
 *
 * This is the drop-in boundary for the reference's operator API (namespace
 * `mdreduce`, /root/reference/proj/include/mdreduce/<name>.hpp).  The reference has
 * no C-ABI of its own; each entry point below names the C++ function it
 * replaces.  The C++ header `include/mdreduce_b200.hpp` re-exposes these as the
 * reference's exact C++ signatures (same structs, same exception types), so a
 * reference caller recompiles unchanged.
 *
 * Conventions
 *  - plain pointers + explicit counts, no torch / CUDA types in signatures;
 *  - every call returns an int status (MDR_OK == 0); a failing call performs
 *    no work (validation happens before any launch), mirroring the reference
 *    throwing before work (SURVEY §8b "Errors");
 *  - `*_batch` calls take HOST buffers and do H2D, kernels and D2H inside;
 *    `*_dev` calls take DEVICE pointers, enqueue on the context stream and
 *    return without synchronising (the resident-input path the bench times);
 *  - one context per device; calls on one context are serialised.
 */
#ifndef MDR_H
#define MDR_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ---- status codes (exception taxonomy of errors.hpp:10-42) ------------- */
enum {
  MDR_OK = 0,
  MDR_ERR_SIZE = 1,           /* SizeError                errors.hpp:10-13 */
  MDR_ERR_BLOCK_SIZE = 2,     /* UnsupportedBlockSizeError errors.hpp:16-20 */
  MDR_ERR_NUMERIC_DOMAIN = 3, /* NumericDomainError        errors.hpp:23-26 */
  MDR_ERR_PARSE = 4,          /* ParseError                errors.hpp:29-42 */
  MDR_ERR_CUDA = 5,           /* device / driver failure (new)           */
  MDR_ERR_INVALID = 6         /* null pointer, bad enum (new)            */
};

/* ---- enums (reduce.hpp:13, mma.hpp:13-14) ------------------------------ */
enum {
  MDR_METHOD_BASELINE = 0,  /* ReduceMethod::Baseline: fp32 shuffle trees  */
  MDR_METHOD_TCU = 1,       /* ReduceMethod::Tcu: paper's f16 MMA (compat) */
  MDR_METHOD_TCU_SPLIT = 2  /* new: tf32 hi/lo error-compensated MMA       */
};
enum { MDR_ACCUM_HALF = 0, MDR_ACCUM_SINGLE = 1 };
enum { MDR_LAYOUT_ROW = 0, MDR_LAYOUT_COL = 1 };
/* pair-term arithmetic of the scoring kernel: FP64 reproduces the
 * reference's double evaluate_atoms (docking.cpp:95-128) bit for bit;
 * FP64_FAST (FMA, one reciprocal per pair, sites split across the warps of
 * a CTA) and FP32 are the fast modes (tolerance parity). */
enum { MDR_PAIR_FP64 = 0, MDR_PAIR_FP32 = 1, MDR_PAIR_FP64_FAST = 2 };

/* ---- plain-data structs ------------------------------------------------ */
/* SyncStats reduce.hpp:33-54 (field order preserved). */
typedef struct mdr_sync_stats {
  uint64_t block_syncs;
  uint64_t warp_shuffles;
  uint64_t atomic_adds;
  uint64_t memory_fences;
  uint64_t mma_ops;
  uint64_t shared_mem_bytes;
  uint64_t precision_conversions;
} mdr_sync_stats;

/* LigandInstance instance_io.hpp:13-30, flattened (caller-owned). */
typedef struct mdr_instance {
  int32_t n_atoms;
  int32_t n_sites;
  int32_t n_rot;
  int32_t reserved;
  const double* atom_xyzw;     /* n_atoms x {x, y, z, weight}            */
  const int32_t* atom_torsion; /* n_atoms, -1 = rigid                    */
  const double* site_xyzdd;    /* n_sites x {x, y, z, depth, d0}         */
} mdr_instance;

/* LgaSettings docking.hpp:106-115 (same defaults via mdr_lga_defaults). */
typedef struct mdr_lga_settings {
  int32_t population_size;
  int32_t generations;
  int64_t max_evaluations;
  double ls_fraction;
  int32_t ls_max_iters;
  int32_t partition;
  double ls_convergence_tol;
  double mutation_sigma;
} mdr_lga_settings;

/* LsRunRecord docking.hpp:117-123. */
typedef struct mdr_ls_record {
  double best_energy;
  int32_t iterations;
  int32_t converged;
} mdr_ls_record;

typedef struct mdr_ctx mdr_ctx;

/* ---- context ------------------------------------------------------------ */
mdr_ctx* mdr_ctx_create(int device);
void mdr_ctx_destroy(mdr_ctx* ctx);
/* Use an external cudaStream_t (passed as void*); NULL restores the
 * context's own stream. */
int mdr_ctx_set_stream(mdr_ctx* ctx, void* cuda_stream);
void* mdr_ctx_stream(mdr_ctx* ctx);
int mdr_ctx_set_pair_precision(mdr_ctx* ctx, int pair_precision);
/* Warps per CTA of the warp-per-pose kernels (1..16, default 2). */
int mdr_ctx_set_warps_per_block(mdr_ctx* ctx, int warps);
/* Warps cooperating on one pose in the CTA-per-pose local-search kernels
 * used by the fast pair modes (1..16, default 4). */
int mdr_ctx_set_cta_warps(mdr_ctx* ctx, int warps);

/* Analytic (site) mode torsion gradient.  0 (default): every torsion entry is
 * the TOTAL ligand torque projected on that torsion's world axis — score()'s
 * documented approximation (reference docking.cpp:228-231, docking.hpp:42-43),
 * the quantity parity is defined on.  1: entry 6+k is the torque of torsion
 * group k alone (the atoms moved by torsion k), the exact gradient that
 * score_reference() computes in double (docking.cpp:244-268).  The per-atom
 * torques are staged in the pose's warp scratch during the evaluation, so the
 * cost is 16 B of shared memory per atom and one group sum per torsion lane;
 * ligands are limited to 1024 atoms and the LS runs warp per pose.  Applies to
 * every analytic score / local-search / LGA launch made through `ctx` (an LGA
 * batch keeps the mode it was created with).  Grid mode always uses the
 * exact per-group torque. */
int mdr_ctx_set_exact_torsion(mdr_ctx* ctx, int on);

/* Site-chunking policy of the warp-per-pose evaluation (host-only, no GPU
 * needed): for FP64-fast pair terms a small ligand's sites are split into
 * *n_chunks ranges of *chunk_len (a multiple of 8) so the n_atoms x n_chunks
 * (atom, chunk) items fill all 32 lanes of the warp-per-pose kernels (score,
 * LGA init / offspring, one-warp search, polish); *n_chunks = 1 means lane
 * per atom (always the case for the other pair modes).  DESIGN.md §3. */
int mdr_site_chunking(int pair_precision, int n_atoms, int n_sites, int* n_chunks, int* chunk_len);
/* The same policy for the LGA's Lamarckian search in form `warps` (1 = one
 * warp; 2 and 3 = the multi-warp forms of mdr_ctx_set_ls_warps, which share
 * one policy).  In the multi-warp forms an item is (chunk, group of
 * *atoms_per_item atoms): 1, or 3 when register blocking shortens nothing on
 * the critical path but cuts the shared-memory site loads. */
int mdr_search_chunking(int pair_precision, int n_atoms, int n_sites, int warps, int* n_chunks, int* chunk_len,
                        int* atoms_per_item);
/* Form of the LGA's Lamarckian search (env MDR_LS_WARPS): 3 (default) = one
 * leader warp per search plus a pool of item warps shared by the CTA's
 * searches (ls_multi.cu); 2 = a leader and a dedicated helper warp per
 * search; 1 = one warp per search; 0 = the legacy warp-pair kernel.  Every
 * choice gives bit-identical results for the same chunking.  Set before the
 * first docking of the context. */
int mdr_ctx_set_ls_warps(mdr_ctx* ctx, int warps);
/* Message of the last failing call on this context (thread-local copy). */
const char* mdr_last_error(mdr_ctx* ctx);
/* Number of kernel launches this context has enqueued so far. */
uint64_t mdr_ctx_launch_count(mdr_ctx* ctx);
int mdr_ctx_synchronize(mdr_ctx* ctx);
const char* mdr_version(void);

/* ---- L0 numeric units (half.hpp, mma.hpp) ------------------------------ */
/* f32_to_half half.cpp:8-54 / half_to_f32 half.cpp:56-74, on the device
 * (cvt.rn.f16.f32, subnormals kept). */
int mdr_f32_to_half_batch(mdr_ctx* ctx, const float* in, size_t n, uint16_t* out);
int mdr_half_to_f32_batch(mdr_ctx* ctx, const uint16_t* in, size_t n, float* out);
/* mma mma.cpp:41-64 on tensor cores: n_tiles independent 16x16x16 tiles,
 * a/b row-major binary16 (256 each), c/d row-major fp32 (256 each).
 * accum == HALF rounds d to binary16 once (Accum16 Half mode). */
int mdr_mma_batch(mdr_ctx* ctx, const uint16_t* a, const uint16_t* b,
                  const float* c, int n_tiles, int accum, float* d);

/* ---- L1 block reductions (reduce.hpp) ---------------------------------- */
/* reduce4 reduce.cpp:80-111.  n_red reductions of n float4 {x,y,z,e}.
 * method TCU: reference-compatible f16 MMA with AccumMode semantics;
 * method TCU_SPLIT: tf32 hi/lo MMA, fp32-accurate;
 * method BASELINE: simulate_block baseline (4 x baseline_block_reduce,
 *   simblock.cpp:447-462; n must be a legal block size).
 * stats = SyncStats of ONE reduction as the reference counts it. */
int mdr_reduce4_batch(mdr_ctx* ctx, const float* vecs, int n, int n_red,
                      int method, int accum, float* out, mdr_sync_stats* stats);
/* Device-pointer form of mdr_reduce4_batch (enqueue on the context's stream,
 * no copies, no sync).  TCU_SPLIT batches of n % 32 == 0 records and at
 * least 148*32 reductions run as one batched tcgen05 contraction (tf32 hi/lo,
 * 32 reductions per 128-row tile, accumulator in TMEM); smaller or ragged
 * batches run the warp-per-reduction mma.sync kernel.  Same contract. */
int mdr_reduce4_dev(mdr_ctx* ctx, const float* d_vecs, int n, int n_red,
                    int method, int accum, float* d_out);
/* baseline_block_reduce reduce.cpp:136-163, n_red blocks of `threads`. */
int mdr_block_reduce_batch(mdr_ctx* ctx, const float* values, int threads,
                           int n_red, float* out, mdr_sync_stats* stats);
/* baseline_warp_reduce reduce.cpp:113-134, n_red warps of 32 lanes. */
int mdr_warp_reduce_batch(mdr_ctx* ctx, const float* lanes, int n_red,
                          float* out, mdr_sync_stats* stats);
/* reduce7 reduce.cpp:165-209.  recs: n_red x n x {e,gx,gy,gz,tx,ty,tz}. */
int mdr_reduce7_batch(mdr_ctx* ctx, const float* recs, int n, int n_red,
                      int method, int accum, float* out, mdr_sync_stats* stats);
/* Device-pointer form of mdr_reduce7_batch; TCU_SPLIT batches route to the
 * tcgen05 contraction as in mdr_reduce4_dev (16 reductions x 8 rows per
 * tile). */
int mdr_reduce7_dev(mdr_ctx* ctx, const float* d_recs, int n, int n_red,
                    int method, int accum, float* d_out);
/* 1 when a TCU_SPLIT reduce4/reduce7 call of this shape runs on tcgen05. */
int mdr_reduce_uses_tc05(mdr_ctx* ctx, int method, int n, int n_red);
/* Route TCU_SPLIT batches to tcgen05 (default 1; env MDR_TC05=0). */
int mdr_ctx_set_tc05(mdr_ctx* ctx, int on);

/* Self test: bit mismatches of the branch-free FP64 division of the strict
 * pair loop against IEEE div.rn.f64 over n counter-generated operand pairs. */
/* Self test: bit mismatches of the branch-free FP64 square root of the LGA
 * search against IEEE sqrt.rn.f64 over n counter-generated arguments. */
int mdr_selftest_dsqrt(mdr_ctx* ctx, uint64_t seed, int64_t n, uint64_t* mismatches);
/* Self test: bit mismatches (sin and cos counted separately) of the
 * branch-free sincos of the LGA search against libdevice sincos. */
int mdr_selftest_sincos(mdr_ctx* ctx, uint64_t seed, int64_t n, uint64_t* mismatches);
int mdr_selftest_ddiv(mdr_ctx* ctx, uint64_t seed, int64_t n, uint64_t* mismatches);
/* Self test: the device's correctly rounded sin, cos (angles in [-pi, pi)),
 * log (Box-Muller u1) and cos(2 pi u2) (crmath.cuh), then CUDA libdevice's,
 * against this host's glibc over n counter-generated inputs.  mismatches[8]:
 * cr sin, cr cos, cr log, cr cos2pi, libdevice sin, cos, log, cos2pi. */
int mdr_selftest_crmath(mdr_ctx* ctx, int64_t n, uint64_t* mismatches);
/* The raw values behind mdr_selftest_crmath for inputs i0 .. i0+n-1:
 * out[8 i + 0..3] = correctly rounded sin a, cos a, log u1, cos z (the
 * grid-mode and Box-Muller math), out[8 i + 4..7] = libdevice's. */
int mdr_crmath_values(mdr_ctx* ctx, int64_t i0, int n, double* out);

/* C2 microbench (no reference counterpart; cli.cpp:195-266 is its CPU
 * analogue): kernel k in [0, mdr_reduce_bench_kernels()) reduces float4 per
 * thread over blocks of `block` threads.  chain_steps > 0: n_red/chain_steps
 * blocks each run a dependent chain of chain_steps reduce-and-broadcast
 * steps on one input set (d_in: blocks x block x 4 floats); chain_steps == 0:
 * n_red distinct input sets streamed from HBM.  d_out: one float4 per block
 * (chain) or per reduction (stream).  Device pointers, enqueue only. */
/* C2 inputs, device-generated and offset-addressable:
 * d_out[i] = (float) uniform(-1, 1) of draw i + 1 of derive_rng(seed, label)
 * (rng.hpp:41-43), the values the reference's RngStream yields on the host.
 * Enqueue only. */
int mdr_fill_uniform_dev(mdr_ctx* ctx, uint64_t seed, const char* label, int64_t n, float* d_out);
int mdr_reduce_bench_kernels(void);
const char* mdr_reduce_bench_kernel_name(int kernel);
int mdr_reduce_bench_dev(mdr_ctx* ctx, int kernel, int block, const float* d_in,
                         int n_red, int chain_steps, float* d_out);
/* Chain mode of mdr_reduce_bench_dev that also writes, per block, the SM
 * clock cycles of its whole dependent chain (d_cycles: n_red / chain_steps
 * int64): the latency metric, cycles per reduce-and-broadcast step. */
int mdr_reduce_bench_chain_cycles_dev(mdr_ctx* ctx, int kernel, int block, const float* d_in, int n_red,
                                      int chain_steps, float* d_out, int64_t* d_cycles);

/* ---- L2 scoring (docking.hpp:44-63) ------------------------------------ */
/* score docking.cpp:191-233 for n genotypes (n x dim, dim = 6 + n_rot,
 * order x,y,z,phi,theta,alpha,torsions).  gradient n x dim, torque n x 3.
 * stats = SyncStats of ONE score call. */
int mdr_score_batch(mdr_ctx* ctx, const mdr_instance* inst,
                    const double* genotypes, int n, int method, int accum,
                    int partition, float* energy, float* gradient,
                    float* torque, mdr_sync_stats* stats);
/* score_reference docking.cpp:235-270 (double sums, exact per-group torsion
 * torque). */
int mdr_score_reference_batch(mdr_ctx* ctx, const mdr_instance* inst,
                              const double* genotypes, int n, double* energy,
                              double* gradient, double* torque);

/* ---- L3 search drivers ------------------------------------------------- */
/* adadelta_step docking.cpp:281-308 for n independent states (n x dim
 * each).  Updates avg_sq_grad / avg_sq_update / genotype in place. */
int mdr_adadelta_step_batch(mdr_ctx* ctx, int dim, int n, double rho,
                            double epsilon, double* avg_sq_grad,
                            double* avg_sq_update, double* genotype,
                            const double* grad);
/* local_search docking.cpp:310-351 for n starts, one device-resident
 * ADADELTA loop per start.  stats = accumulated SyncStats per search. */
int mdr_local_search_batch(mdr_ctx* ctx, const mdr_instance* inst,
                           const double* starts, int n, int max_iters,
                           double convergence_tol, int method, int accum,
                           int partition, double* out_genotype,
                           double* out_energy, int32_t* out_iterations,
                           int32_t* out_converged, mdr_sync_stats* stats);

/* lga_run docking.cpp:392-517 for n_runs independent seeds.
 * best_genotype n_runs x dim; records n_runs x mdr_lga_max_records(s);
 * n_records[i] valid records of run i; total_stats per run. */
void mdr_lga_defaults(mdr_lga_settings* s);
int mdr_lga_max_records(const mdr_lga_settings* s);
int mdr_lga_run_batch(mdr_ctx* ctx, const mdr_instance* inst, int method,
                      int accum, const mdr_lga_settings* settings,
                      const uint64_t* seeds, int n_runs, double* best_energy,
                      double* best_genotype, int64_t* evaluations,
                      int32_t* converged, int32_t* n_records,
                      mdr_ls_record* records, mdr_sync_stats* total_stats);

/* ---- resident-input (device pointer) variants -------------------------- */
/* A device-resident ligand: uploaded once, reused by every _dev call. */
typedef struct mdr_dev_instance mdr_dev_instance;
mdr_dev_instance* mdr_instance_upload(mdr_ctx* ctx, const mdr_instance* inst);
void mdr_instance_free(mdr_ctx* ctx, mdr_dev_instance* dinst);

int mdr_score_dev(mdr_ctx* ctx, const mdr_dev_instance* dinst,
                  const double* d_genotypes, int n, int method, int accum,
                  int partition, float* d_energy, float* d_gradient,
                  float* d_torque);
int mdr_local_search_dev(mdr_ctx* ctx, const mdr_dev_instance* dinst,
                         const double* d_starts, int n, int max_iters,
                         double convergence_tol, int method, int accum,
                         int partition, double* d_out_genotype,
                         double* d_out_energy, int32_t* d_out_iterations,
                         int32_t* d_out_converged, int32_t* d_status);

/* LGA batch with all state on the device.  d_seeds: n_runs uint64 on the
 * device.  Results stay on the device in an opaque batch object; read them
 * with mdr_lga_batch_download.  The whole docking is one CUDA graph. */
typedef struct mdr_lga_batch mdr_lga_batch;
mdr_lga_batch* mdr_lga_batch_create(mdr_ctx* ctx, const mdr_dev_instance* dinst,
                                    int method, int accum,
                                    const mdr_lga_settings* settings,
                                    int n_runs);
void mdr_lga_batch_destroy(mdr_ctx* ctx, mdr_lga_batch* b);
int mdr_lga_batch_run_dev(mdr_ctx* ctx, mdr_lga_batch* b, const uint64_t* d_seeds);
int mdr_lga_batch_download(mdr_ctx* ctx, mdr_lga_batch* b, double* best_energy,
                           double* best_genotype, int64_t* evaluations,
                           int32_t* converged, int32_t* n_records,
                           mdr_ls_record* records, mdr_sync_stats* total_stats);
/* Sum of evaluations over the batch's runs, reduced on the device into a
 * single int64 at d_total (for D2H of one word per step). */
int mdr_lga_batch_total_evals_dev(mdr_ctx* ctx, mdr_lga_batch* b, int64_t* d_total);
/* Profiling replay (no graph): the same docking with CUDA events around the
 * local-search kernels.  ls_ms = summed LS-kernel time (incl. polish),
 * step_ms = whole step, ls_evals = evaluations done inside LS kernels. */
int mdr_lga_batch_profile_dev(mdr_ctx* ctx, mdr_lga_batch* b, const uint64_t* d_seeds,
                              float* ls_ms, float* step_ms, int64_t* ls_evals);

/* ---- grid-map scoring mode (north_star subsystem 1) -------
 * The reference scores a pose against analytic receptor "sites"
 * (evaluate_atoms docking.cpp:95-128) and puts AutoDock's grid maps out of
 * scope.  This mode is the AutoDock-GPU form of the same
 * operator: per-atom trilinear interpolation of precomputed receptor maps,
 * intramolecular pair terms between atoms of different rigid groups, and the
 * exact per-torsion gradient (torque of the moving group about its axis).
 * Genotype, torsion model (one group per atom, rotate_axis docking.cpp:57-60),
 * ADADELTA and LGA are the reference's.  Formulas: DESIGN.md §11; CPU
 * restatement: oracle/mdr_oracle.c (orc_grid_*).  Parity: tolerance (FP32
 * maps and interpolation), stated in tests/test_gpu_grid.py.
 *
 * Energy of a pose (world atom p_i = t + R * rotate_axis(local_i)):
 *   E = sum_i [ w_i V_type(i)(p_i) + q_i V_elec(p_i) + |q_i| V_desolv(p_i)
 *               + k_out |p_i - clamp(p_i)|^2 ]
 *     + sum_{i<j, group_i != group_j} [ eps_ij (rho^12 - 2 rho^6) + k_e q_i q_j / u ]
 * with V(p) the trilinear interpolation at p clamped into the lattice,
 * u = r_ij^2 + c2, c2 = 0.5625 d0^2, rho^2 = (d0^2 + c2) / u,
 * d0 = radius_i + radius_j, eps_ij = sqrt(epsilon_i epsilon_j). */
/* Outside-lattice restraint k_out (kcal/mol/A^2): an atom beyond the lattice
 * samples the maps at the clamped point and pays k_out |p - clamp(p)|^2. */
#define MDR_GRID_OUTSIDE_K 10.0

typedef struct mdr_grid {
  int32_t nx, ny, nz; /* lattice points per axis (>= 2 each)                */
  int32_t n_types;    /* atom-type maps; `maps` holds n_types + 2 maps      */
  double origin[3];   /* world position of lattice point (0, 0, 0)          */
  double spacing;     /* lattice spacing (Angstrom, > 0)                    */
  const float* maps;  /* (n_types + 2) x nz x ny x nx, x fastest: the type
                         maps, then electrostatic, then desolvation          */
} mdr_grid;

/* Per-atom chemistry of a ligand in grid mode (caller-owned, n_atoms each). */
typedef struct mdr_ligand_params {
  const int32_t* atom_type;   /* map index in [0, n_types)                  */
  const double* atom_charge;  /* q_i                                        */
  const double* atom_radius;  /* intramolecular d0_ij = radius_i + radius_j */
  const double* atom_epsilon; /* eps_ij = sqrt(epsilon_i * epsilon_j)       */
  double elec_scale;          /* k_e (83.0 = 332 / 4, distance-dependent
                                 dielectric 4r, soft-cored)                 */
  int32_t intra;              /* 0: no intramolecular term                  */
  int32_t reserved;
} mdr_ligand_params;

/* Synthetic receptor maps from the instance's sites (an AutoGrid analogue
 * for the reference's site model).  At lattice point P, per site j:
 *   type t : depth_j * depth_scale[t] * (rho^12 - 2 rho^6) with
 *            d = d0_j * dist_scale[t] (type 0 with scales 1 == the
 *            reference's analytic well, docking.cpp:113-122)
 *   elec   : elec_scale * charge_j / (|P - s_j|^2 + 0.5625 d0_j^2)
 *   desolv : volume_j * exp(-|P - s_j|^2 / (2 sigma^2)). */
typedef struct mdr_receptor_fields {
  const double* site_charge;      /* n_sites                                */
  const double* site_volume;      /* n_sites                                */
  const double* type_depth_scale; /* n_types                                */
  const double* type_dist_scale;  /* n_types                                */
  double elec_scale;
  double desolv_sigma;
} mdr_receptor_fields;

typedef struct mdr_dev_grid mdr_dev_grid;
/* Upload host maps (one device copy, shared by every ligand docked
 * against this receptor). */
mdr_dev_grid* mdr_grid_upload(mdr_ctx* ctx, const mdr_grid* grid);
/* Build the maps on the device from `sites` (uses n_sites / site_xyzdd only);
 * `shape` gives nx, ny, nz, n_types, origin, spacing (its maps is ignored). */
mdr_dev_grid* mdr_grid_build(mdr_ctx* ctx, const mdr_instance* sites, const mdr_receptor_fields* fields,
                             const mdr_grid* shape);
/* Copy the device maps to host (size (n_types + 2) * nx * ny * nz floats). */
int mdr_grid_download(mdr_ctx* ctx, const mdr_dev_grid* grid, float* maps);
void mdr_grid_free(mdr_ctx* ctx, mdr_dev_grid* grid);

/* Switch a device ligand to grid scoring against `grid` (NULL: back to the
 * analytic site model).  Every _dev call and mdr_lga_batch_create on this
 * instance then uses the grid kernels (CTA per pose, `partition` threads).
 * The instance's sites still define the random_genotype box
 * (docking.cpp:362-374). */
int mdr_instance_set_grid(mdr_ctx* ctx, mdr_dev_instance* dinst, const mdr_dev_grid* grid,
                          const mdr_ligand_params* params);

/* Host-buffer grid-mode calls (ligand uploaded per call, receptor resident).
 * energy n; gradient n x dim (exact torsion gradient); torque n x 3. */
int mdr_grid_score_batch(mdr_ctx* ctx, const mdr_dev_grid* grid, const mdr_instance* inst,
                         const mdr_ligand_params* params, const double* genotypes, int n, int method,
                         int partition, float* energy, float* gradient, float* torque);
int mdr_grid_local_search_batch(mdr_ctx* ctx, const mdr_dev_grid* grid, const mdr_instance* inst,
                                const mdr_ligand_params* params, const double* starts, int n, int max_iters,
                                double convergence_tol, int method, int partition, double* out_genotype,
                                double* out_energy, int32_t* out_iterations, int32_t* out_converged);
int mdr_grid_lga_run_batch(mdr_ctx* ctx, const mdr_dev_grid* grid, const mdr_instance* inst,
                           const mdr_ligand_params* params, int method, const mdr_lga_settings* settings,
                           const uint64_t* seeds, int n_runs, double* best_energy, double* best_genotype,
                           int64_t* evaluations, int32_t* converged, int32_t* n_records,
                           mdr_ls_record* records);

/* ---- virtual screen (BASELINE config C5) -------------------
 * Dock n_ligands ligands against one device receptor in ONE launch sequence:
 * runs_per_ligand LGA runs each (run r = j * runs_per_ligand + k docks
 * ligand j with seeds[r]), grid-mode scoring, then the RMSD clustering of
 * each ligand's best poses.  Every run is exactly the run a single-ligand
 * mdr_grid_lga_run_batch would make (same kernels, same draws).  All ligands
 * share settings->partition threads per pose (>= 6 + n_rot of each).
 * Outputs per run: best_energy, evaluations, converged, cluster_of,
 * rmsd_to_seed (each n_ligands * runs_per_ligand); best_genotype packed per
 * ligand (ligand j's runs * (6 + n_rot_j) doubles follow ligand j-1's);
 * n_clusters per ligand.  Null output pointers are skipped. */
int mdr_grid_screen_batch(mdr_ctx* ctx, const mdr_dev_grid* grid, const mdr_instance* ligands,
                          const mdr_ligand_params* params, int n_ligands, int runs_per_ligand, int method,
                          const mdr_lga_settings* settings, const uint64_t* seeds, double rmsd_tol,
                          double* best_energy, double* best_genotype, int64_t* evaluations, int32_t* converged,
                          int32_t* cluster_of, double* rmsd_to_seed, int32_t* n_clusters);

/* ---- native multi-GPU host driver (north_star subsystem 4, SURVEY §8 e) --
 * One host thread + one context per listed device (a device may be listed
 * more than once).  No collective: every thread writes its results at the
 * run / ligand's own offsets of the caller's arrays (the final gather).
 * Results equal a single-device call with the same seeds. */
/* LGA runs sharded statically (run i -> devices[i % n_devices]); outputs as
 * mdr_lga_run_batch (best_genotype n_runs x dim). */
int mdr_multi_lga_run_batch(const int* devices, int n_devices, const mdr_instance* inst, int method, int accum,
                            int pair_precision, const mdr_lga_settings* settings, const uint64_t* seeds, int n_runs,
                            double* best_energy, double* best_genotype, int64_t* evaluations, int32_t* converged);
/* Virtual screen over the node: every device builds the receptor maps once,
 * then pulls batches of batch_ligands ligands from a shared atomic queue
 * (dynamic balancing of unequal ligand costs) and docks each batch with
 * mdr_grid_screen_batch.  A device that fails (device error) retires and
 * its batch goes back to the queue for the others; the call fails only if
 * no device is left or a batch is invalid.  Outputs as mdr_grid_screen_batch over all ligands;
 * device_of_ligand[j] = index into `devices` of the device that docked j. */
int mdr_multi_screen(const int* devices, int n_devices, const mdr_instance* receptor_sites,
                     const mdr_receptor_fields* fields, const mdr_grid* shape, const mdr_instance* ligands,
                     const mdr_ligand_params* params, int n_ligands, int runs_per_ligand, int method,
                     const mdr_lga_settings* settings, const uint64_t* seeds, double rmsd_tol, int batch_ligands,
                     double* best_energy, double* best_genotype, int64_t* evaluations, int32_t* cluster_of,
                     int32_t* n_clusters, int32_t* device_of_ligand);
/* Message of the last failing multi-device call on this thread. */
const char* mdr_multi_last_error(void);
/* Test hook (SURVEY §5 fault injection): make device index `device_index`
 * of the next mdr_multi_screen calls fail on its `batch`-th batch (-1: off).
 * A failed device retires and its batch is re-queued to the others. */
void mdr_multi_set_fault_injection(int device_index, int batch);

/* ---- RMSD clustering of docked poses ----------------------
 * Not in the reference.  Poses become world coordinates through
 * evaluate_atoms' transform (docking.cpp:101-106, FP64); clustering is
 * AutoDock's: poses in ascending (energy, index) order, each joins the first
 * cluster whose seed (lowest-energy member) is within RMSD < rmsd_tol, else
 * seeds a new cluster.  cluster_of[i] = cluster index in creation order
 * (0 = the cluster of the best pose); rmsd_to_seed[i] = RMSD to that seed.
 * CPU restatement: orc_cluster_poses (oracle/mdr_oracle.c). */
/* genotypes n x dim -> xyz n x n_atoms x 3 (world coordinates). */
int mdr_pose_coords_batch(mdr_ctx* ctx, const mdr_instance* inst, const double* genotypes, int n, double* xyz);
int mdr_cluster_poses(mdr_ctx* ctx, const mdr_instance* inst, const double* genotypes, const double* energies,
                      int n, double rmsd_tol, int32_t* cluster_of, double* rmsd_to_seed, int32_t* n_clusters);
/* Device variant over segments (one independent clustering per segment,
 * e.g. per ligand of a screen): poses d_seg_off[s] .. d_seg_off[s+1]. */
int mdr_cluster_segments_dev(mdr_ctx* ctx, const mdr_dev_instance* dinst, const double* d_genotypes,
                             const double* d_energies, const int32_t* d_seg_off, int n_seg, int n_total,
                             double rmsd_tol, int32_t* d_cluster_of, double* d_rmsd_to_seed,
                             int32_t* d_n_clusters);
/* Cluster the best poses of an LGA batch's runs (on the device; results to
 * host buffers of n_runs entries). */
int mdr_lga_batch_cluster(mdr_ctx* ctx, mdr_lga_batch* b, double rmsd_tol, int32_t* cluster_of,
                          double* rmsd_to_seed, int32_t* n_clusters);

/* Diagnostics: clock64 phase counters of the warp-pair Lamarckian search,
 * summed over all searches since the last reset (16 x uint64: leader phases
 * 0 ADADELTA, 1 trig+frame+positions, 2 barrier B1, 3 chunk items, 4 barrier
 * B2, 5 chunk combine + reduction, 6 projection + best/history; [7]
 * evaluations; helper 8 wait B1, 9 items, 10 wait B2; [11] searches).  Only
 * an experiment build with -DMDR_PHASE_PROF=1 records them; the product
 * build returns MDR_ERR_INVALID. */
int mdr_phase_prof(uint64_t* out16, int reset);
/* LGA searches started per SM (index = %smid) since the last reset: the
 * multi-warp analytic search plus the grid-mode search; phase-profiling
 * builds only. */
int mdr_phase_prof_sm(uint32_t* out256, int reset);

#ifdef __cplusplus
}
#endif
#endif /* MDR_H */
