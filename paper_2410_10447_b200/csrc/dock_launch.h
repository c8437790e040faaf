// dock_launch.h — host-callable launchers of the CUDA kernels (no CUDA types
// leak past capi.cpp; the public boundary is include/mdr.h).
#pragma once

#include <cuda_runtime.h>

#include "mdr_shared.h"

namespace mdr {

// dock.cu
cudaError_t launch_score(const LigandView& L, const double* genos, int n, int method, int pair, int partition,
                         int half_mode, float* energy, float* grad, float* torque, cudaStream_t s, int wpb);
cudaError_t launch_score_reference(const LigandView& L, const double* genos, int n, double* energy, double* grad,
                                   double* torque, cudaStream_t s, int wpb);
cudaError_t launch_adadelta(int dim, int n, double rho, double eps, double* sq_g, double* sq_u, double* geno,
                            const double* grad, int* status, cudaStream_t s);
cudaError_t launch_local_search(const LigandView& L, const double* starts, int n, int max_iters, double tol,
                                int method, int pair, int partition, int half_mode, double* out_g, double* out_e,
                                int* out_it, int* out_cv, int* status, cudaStream_t s, int wpb, int cta_warps);
cudaError_t prepare_lga(const LigandView& L, int method, int pair, int wpb, int cta_warps);
cudaError_t launch_lga(const LigandView& L, const LgaDev& D, int method, int pair, cudaStream_t s, int wpb,
                       int cta_warps, int* n_launches, cudaEvent_t* ls_events = nullptr);
cudaError_t launch_lga_total(const LgaDev& D, long long* out, cudaStream_t s);
cudaError_t launch_lga_init_finalize(const LgaDev& D, cudaStream_t s);
cudaError_t launch_lga_gen_finalize(const LgaDev& D, int gen, cudaStream_t s);

// grid.cu (grid-map scoring mode, CTA of `threads` per pose)
size_t grid_smem_for(const LigandView& L, const FlexView& F, int threads, int method);
// grid kernels' method code of the strict FP64 path (grid.cu kGridStrict)
constexpr int kGridStrictMethod = 3;
cudaError_t launch_grid_score(const LigandView& L, const GridView& G, const FlexView& F, const double* genos, int n,
                              int method, int threads, float* energy, float* grad, float* torque, cudaStream_t s);
cudaError_t launch_grid_local_search(const LigandView& L, const GridView& G, const FlexView& F, const double* starts,
                                     int n, int max_iters, double tol, int method, int threads, double* out_g,
                                     double* out_e, int* out_it, int* out_cv, int* status, cudaStream_t s);
size_t grid_smem_for(int n_atoms, int n_rot, int n_tors_atoms, int threads);
cudaError_t prepare_grid_lga(size_t smem, int method);
cudaError_t launch_grid_lga(const GridLigands& GL, size_t smem, const GridView& G, const LgaDev& D, int method,
                            int threads, cudaStream_t s, int* n_launches, cudaEvent_t* ls_events = nullptr);
cudaError_t launch_grid_build(const GridView& G, const double* sites, int n_sites, const double* charge,
                              const double* volume, const double* depth_scale, const double* dist_scale,
                              double elec_scale, double sigma, float* maps, cudaStream_t s);

// cluster.cu (RMSD clustering)
cudaError_t launch_pose_coords(const LigandView* Ls, const int* pose_lig, const double* genos, int gstride, int n,
                               long long xstride, double* xyz, cudaStream_t s);
cudaError_t launch_cluster(const double* xyz, long long xstride, const double* energy, const int* seg_off,
                           const int* seg_na, int n_seg, int na, double tol, int* cluster_of, double* rmsd,
                           int* n_clusters, int* order, int* seeds, cudaStream_t s);

// reduce.cu
cudaError_t launch_f32_to_half(const float* in, size_t n, uint16_t* out, cudaStream_t s);
cudaError_t launch_half_to_f32(const uint16_t* in, size_t n, float* out, cudaStream_t s);
cudaError_t launch_mma16(const uint16_t* a, const uint16_t* b, const float* c, int n_tiles, int half_mode, float* d,
                         cudaStream_t s);
cudaError_t launch_warp_reduce(const float* lanes, int n_red, float* out, cudaStream_t s);
cudaError_t launch_block_reduce(const float* values, int threads, int n_red, float* out, cudaStream_t s);
cudaError_t launch_reduce4(const float* vecs, int n, int n_red, int method, int half_mode, float* out,
                           cudaStream_t s);
cudaError_t launch_reduce7(const float* recs, int n, int n_red, int method, int half_mode, float* out,
                           cudaStream_t s);

cudaError_t launch_crmath_probe(long long i0, int n, double* out, cudaStream_t s);
bool phase_prof_read(unsigned long long* out16, bool reset);
bool phase_prof_read_multi(unsigned long long* out16, bool reset);  // adds ls_multi.cu's counters
bool sm_searches_read(unsigned* out256, bool reset);  // searches per SM (phase-profiling builds)
bool sm_grid_read(unsigned* out256, bool reset);      // grid-mode LGA searches per SM (phase-profiling builds)
cudaError_t launch_fill_uniform(uint64_t key, long long n, float* out, cudaStream_t s);
cudaError_t launch_ddiv_selftest(uint64_t seed, long long n, unsigned long long* mismatches, cudaStream_t s);
cudaError_t launch_sincos_selftest(uint64_t seed, long long n, unsigned long long* mismatches, cudaStream_t s);
cudaError_t launch_dsqrt_selftest(uint64_t seed, long long n, unsigned long long* mismatches, cudaStream_t s);

// ls_multi.cu: the LGA's Lamarckian search on L.ls_warps warps per search
#ifndef MDR_LS_FUSE_FINALIZE
#define MDR_LS_FUSE_FINALIZE 1  // the persistent search's last search of a run does the run's generation bookkeeping
#endif
bool ls_multi_supported(const LigandView& L, int pair, int wpb, int cta_warps);
cudaError_t prep_ls_multi(const LigandView& L, int method);
void launch_ls_multi(const LigandView& L, const LgaDev& D, int method, int gen, cudaStream_t s);

// bench_reduce.cu (C2 microbench)
cudaError_t launch_reduce_bench(int kernel, int block, const float* in, int n_red, int chain_steps, float* out,
                                int blocks_per_sm, cudaStream_t s, long long* cycles = nullptr);
const char* reduce_bench_name(int k);
constexpr int kReduceBenchKernels = 9;  // ids 7, 8 = tcgen05 batched (stream mode only; 8 = TMA-fed)

// tc05_reduce.cu: batched float4 reductions, 32 per tcgen05 contraction
cudaError_t launch_reduce4_tc05(const float* in, int B, int n_red, float* out, int ctas_per_sm, cudaStream_t s);
// the same contraction over Partial7 records (16 reductions x 8 rows per tile)
cudaError_t launch_reduce7_tc05(const float* in, int B, int n_red, float* out, int ctas_per_sm, cudaStream_t s);
// K2t2: the same contraction fed by TMA bulk copies into a 6-deep ring
cudaError_t launch_reduce4_tc05_tma(const float* in, int B, int n_red, float* out, cudaStream_t s);

}  // namespace mdr
