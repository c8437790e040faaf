// dock.cu — scoring, ADADELTA local search and LGA kernels (warp per pose).
//
// K3 score_kernel        : score() docking.cpp:191-233, one warp per genotype
// K3r scoreref_kernel    : score_reference() docking.cpp:235-270
// K4 ls_kernel           : local_search() docking.cpp:310-351, the whole
//                          <= max_iters+1 evaluation chain stays on the device
// K5 lga_* kernels       : lga_run() docking.cpp:392-517 split into per-phase
//                          kernels over all runs (init, offspring, LS,
//                          finalize, polish), captured once into a CUDA graph.
// Compiled with --fmad=false (see mdr_device.cuh).
#include <cuda_runtime.h>

#include "crmath.cuh"
#include "dock_launch.h"
#include "mdr_device.cuh"
#include "lga_device.cuh"
#include "warp_region.cuh"

namespace mdr {

#if MDR_PHASE_PROF
__device__ unsigned long long g_phase[16];
#endif

// --------------------------------------------------------------- K3 score
template <int METHOD, int PAIR, bool EXACT, bool CHUNK>
__global__ void MDR_LS_BOUNDS score_kernel(LigandView L, const double* __restrict__ genos, int n, int partition, int half_mode,
                             float* __restrict__ energy, float* __restrict__ grad, float* __restrict__ torque) {
  extern __shared__ __align__(16) unsigned char smem[];
  const SmemLigand S = load_ligand(L, smem);
  __syncthreads();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int item = blockIdx.x * (blockDim.x >> 5) + warp;
  if (item >= n) return;
  WarpCtx w = warp_region(smem + ligand_smem_bytes(L), warp, L);
  const int dim = 6 + L.n_rot;
  const double* g = genos + (size_t)item * dim;
  Frame f;
  const ScoreOut o = score_sums<METHOD, PAIR, EXACT, CHUNK>(S, g, partition, half_mode != 0, w.ws, f);
  for (int d = lane; d < dim; d += 32) grad[(size_t)item * dim + d] = project_dim<EXACT>(S, f, o, d, w.ws);
  if (lane == 0) {
    energy[item] = o.sums[0];
    torque[3 * (size_t)item] = o.sums[4];
    torque[3 * (size_t)item + 1] = o.sums[5];
    torque[3 * (size_t)item + 2] = o.sums[6];
  }
}

// ------------------------------------------------- K3r score_reference
__device__ __forceinline__ double warp_sum_d(double v) {
#pragma unroll
  for (int off = 16; off >= 1; off >>= 1) v += __shfl_xor_sync(kFull, v, off);
  return v;
}

__global__ void scoreref_kernel(LigandView L, const double* __restrict__ genos, int n, double* __restrict__ energy,
                                double* __restrict__ grad, double* __restrict__ torque) {
  extern __shared__ __align__(16) unsigned char smem[];
  const SmemLigand S = load_ligand(L, smem);
  __syncthreads();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int item = blockIdx.x * (blockDim.x >> 5) + warp;
  if (item >= n) return;
  const int dim = 6 + L.n_rot;
  const double* g = genos + (size_t)item * dim;
  const Frame f = build_frame(g[3], g[4], g[5]);
  const d3 tr = {g[0], g[1], g[2]};
  double e = 0.0;
  d3 gs = {0, 0, 0}, ts = {0, 0, 0};
  for (int i = lane; i < S.n_atoms; i += 32) {
    const Partial p = atom_partial<MDR_PAIR_FP64>(S, g, f.R, tr, i);
    e += p.e;
    gs = gs + p.g;
    ts = ts + p.t;
  }
  e = warp_sum_d(e);
  gs = {warp_sum_d(gs.x), warp_sum_d(gs.y), warp_sum_d(gs.z)};
  ts = {warp_sum_d(ts.x), warp_sum_d(ts.y), warp_sum_d(ts.z)};
  // exact per-group torsion torque (docking.cpp:244-268): reduce group k
  for (int k = 0; k < S.n_rot; ++k) {
    d3 tk = {0, 0, 0};
    for (int i = lane; i < S.n_atoms; i += 32)
      if (S.tors[i] == k) tk = tk + atom_partial<MDR_PAIR_FP64>(S, g, f.R, tr, i).t;
    tk = {warp_sum_d(tk.x), warp_sum_d(tk.y), warp_sum_d(tk.z)};
    if (lane == 0) {
      const d3 ax = mv(f.R, d3{S.taxes[3 * k], S.taxes[3 * k + 1], S.taxes[3 * k + 2]});
      grad[(size_t)item * dim + 6 + k] = dot(ax, tk);
    }
  }
  if (lane == 0) {
    energy[item] = e;
    double* go = grad + (size_t)item * dim;
    go[0] = gs.x;
    go[1] = gs.y;
    go[2] = gs.z;
    go[3] = dot(d3{0.0, 0.0, 1.0}, ts);
    go[4] = dot(f.ax_theta, ts);
    go[5] = dot(f.ax_alpha, ts);
    torque[3 * (size_t)item] = ts.x;
    torque[3 * (size_t)item + 1] = ts.y;
    torque[3 * (size_t)item + 2] = ts.z;
  }
}

// ---------------------------------------------------------- ADADELTA
__global__ void adadelta_kernel(int dim, int n, double rho, double eps, double* sq_g, double* sq_u, double* geno,
                                const double* grad, int* status) {
  const int item = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (item >= n) return;
  const size_t o = (size_t)item * dim;
  bool bad = false;
  for (int d = lane; d < dim; d += 32) bad |= !isfinite(grad[o + d]);
  if (__any_sync(kFull, bad)) {
    if (lane == 0) status[item] = MDR_ERR_NUMERIC_DOMAIN;
    return;
  }
  for (int d = lane; d < dim; d += 32) {
    double a = sq_g[o + d], b = sq_u[o + d], x = geno[o + d];
    adadelta_dim(a, b, x, grad[o + d], d, rho, eps);
    sq_g[o + d] = a;
    sq_u[o + d] = b;
    geno[o + d] = x;
  }
}

// ------------------------------------------------------- K4 local search
struct LsResult {
  double energy;
  int iterations, converged, status;
};

// local_search docking.cpp:310-351 run by the calling warp.  start: global
// or shared genotype.  On return w.best holds the best genotype.
template <int METHOD, int PAIR, bool EXACT, int CHUNK>
__device__ LsResult local_search_warp(const SmemLigand& S, const double* start, int max_iters, double tol,
                                      int partition, bool half_mode, const WarpCtx& w) {
  const int lane = threadIdx.x & 31;
  const int dim = 6 + S.n_rot;
  const double rho = 0.95, eps = 1e-6;  // AdadeltaState::fresh docking.hpp:67-74
  for (int d = lane; d < dim; d += 32) {
    const double x = d >= 3 ? wrap_angle(start[d]) : start[d];
    w.g[d] = x;
    w.best[d] = x;
  }
  __syncwarp();
  double sg0 = 0.0, su0 = 0.0, sg1 = 0.0, su1 = 0.0;
  Frame f;
  ScoreOut o = score_sums<METHOD, PAIR, EXACT, CHUNK>(S, w.g, partition, half_mode, w.ws, f);
  float gr0 = lane < dim ? project_dim<EXACT>(S, f, o, lane, w.ws) : 0.f;
  float gr1 = lane + 32 < dim ? project_dim<EXACT>(S, f, o, lane + 32, w.ws) : 0.f;
  LsResult r;
  r.energy = (double)o.sums[0];
  r.iterations = 0;
  r.converged = 0;
  r.status = MDR_OK;
  double hist = r.energy;  // ring slot `lane` holds best_history[iter] for iter % 16 == lane
  for (int iter = 1; iter <= max_iters; ++iter) {
    const bool bad = (lane < dim && !isfinite(gr0)) || (lane + 32 < dim && !isfinite(gr1));
    if (__any_sync(kFull, bad)) {
      r.status = MDR_ERR_NUMERIC_DOMAIN;
      break;
    }
    __syncwarp();
    if (lane < dim) {
      double x = w.g[lane];
      adadelta_dim(sg0, su0, x, (double)gr0, lane, rho, eps);
      w.g[lane] = x;
    }
    if (lane + 32 < dim) {
      double x = w.g[lane + 32];
      adadelta_dim(sg1, su1, x, (double)gr1, lane + 32, rho, eps);
      w.g[lane + 32] = x;
    }
    __syncwarp();
    if (CHUNK == 2) prof_mark(w.ws, 0);
    o = score_sums<METHOD, PAIR, EXACT, CHUNK>(S, w.g, partition, half_mode, w.ws, f);
    gr0 = lane < dim ? project_dim<EXACT>(S, f, o, lane, w.ws) : 0.f;
    gr1 = lane + 32 < dim ? project_dim<EXACT>(S, f, o, lane + 32, w.ws) : 0.f;
    if ((double)o.sums[0] < r.energy) {
      r.energy = (double)o.sums[0];
      for (int d = lane; d < dim; d += 32) w.best[d] = w.g[d];
    }
    const int slot = iter & (kWindow - 1);
    const double old = __shfl_sync(kFull, hist, slot);  // best_history[iter - 16]
    if (lane == slot) hist = r.energy;
    r.iterations = iter;
    if (CHUNK == 2) prof_mark(w.ws, 6);
    if (iter >= kWindow && old - r.energy < tol) {
      r.converged = 1;
      break;
    }
  }
  __syncwarp();
  return r;
}

template <int METHOD, int PAIR, bool EXACT, bool CHUNK>
__global__ void MDR_LS_BOUNDS ls_kernel(LigandView L, const double* __restrict__ starts, int n, int max_iters, double tol,
                          int partition, int half_mode, double* __restrict__ out_g, double* __restrict__ out_e,
                          int* __restrict__ out_it, int* __restrict__ out_cv, int* __restrict__ status) {
  extern __shared__ __align__(16) unsigned char smem[];
  const SmemLigand S = load_ligand(L, smem);
  __syncthreads();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int item = blockIdx.x * (blockDim.x >> 5) + warp;
  if (item >= n) return;
  WarpCtx w = warp_region(smem + ligand_smem_bytes(L), warp, L);
  const int dim = 6 + L.n_rot;
  const LsResult r = local_search_warp<METHOD, PAIR, EXACT, CHUNK>(S, starts + (size_t)item * dim, max_iters, tol, partition,
                                                     half_mode != 0, w);
  for (int d = lane; d < dim; d += 32) out_g[(size_t)item * dim + d] = w.best[d];
  if (lane == 0) {
    out_e[item] = r.energy;
    out_it[item] = r.iterations;
    out_cv[item] = r.converged;
    if (r.status != MDR_OK) status[item] = r.status;
  }
}

// ------------------------------------------ K4c local search, CTA per pose
// Fast pair modes only: the W warps of a CTA split the receptor sites of
// every evaluation (warp w sums sites [w*S/W, (w+1)*S/W) for all atoms, one
// atom per lane), warp 0 merges the per-warp partials, runs the slot
// reduction and the ADADELTA step; two CTA barriers per evaluation.
struct CtaCtx {
  WarpScratch ws;  // warp 0's reduction scratch
  double* g;       // [kMaxDim] current genotype
  double* best;    // [kMaxDim] best genotype
  double* part;    // [W][n_atoms][4] per-warp partial (e, gx, gy, gz)
  double* world;   // [n_atoms][4] placed atoms of the current pose (x, y, z, w)
  int* ctl;        // [0]: stop flag
};

__host__ __device__ inline size_t cta_region_bytes(int n_atoms, int warps) {
  return (size_t)kWarpScratchBytes + 2 * kMaxDim * 8 + (size_t)(warps + 1) * n_atoms * 32 + 16;
}

__device__ __forceinline__ CtaCtx cta_region(unsigned char* base, int n_atoms, int warps) {
  CtaCtx c;
  c.ws.tile = reinterpret_cast<__half*>(base);
  c.ws.rec = reinterpret_cast<float*>(base + 2 * 256 * 2);
  c.ws.tq = nullptr;  // exact-torsion mode runs warp per pose only
  c.ws.wpos = c.ws.part = nullptr;
  c.ws.trig = nullptr;
  c.ws.ctl = nullptr;
  c.ws.bar = 0;
  c.g = reinterpret_cast<double*>(base + kWarpScratchBytes);
  c.best = c.g + kMaxDim;
  c.part = c.best + kMaxDim;
  c.world = c.part + (size_t)warps * n_atoms * 4;
  c.ctl = reinterpret_cast<int*>(c.world + (size_t)n_atoms * 4);
  return c;
}

// Warp 0: frame of the current genotype and every atom's world position.
__device__ __forceinline__ Frame cta_place(const SmemLigand& S, const CtaCtx& c) {
  const int lane = threadIdx.x & 31;
  const Frame f = build_frame<false>(c.g[3], c.g[4], c.g[5]);
  const d3 tr = {c.g[0], c.g[1], c.g[2]};
  for (int i = lane; i < S.n_atoms; i += 32) {
    const d3 w = atom_world<false>(S, c.g, f.R, tr, i);
    double* q = c.world + (size_t)i * 4;
    q[0] = w.x;
    q[1] = w.y;
    q[2] = w.z;
    q[3] = S.atoms[i].w;
  }
  return f;
}

// local_search docking.cpp:310-351 by the whole CTA; the result is valid in
// warp 0, the best genotype in c.best.  Per evaluation: every warp sums its
// slice of the sites for all placed atoms (parallel part), then warp 0
// merges the slices, reduces, projects the gradient, takes the ADADELTA step
// and places the atoms of the next pose (serial part); two CTA barriers.
template <int METHOD, int PAIR>
__device__ LsResult local_search_cta(const SmemLigand& S, const double* start, int max_iters, double tol,
                                     int partition, bool half_mode, const CtaCtx& c) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, W = blockDim.x >> 5;
  const int dim = 6 + S.n_rot;
  const double rho = 0.95, eps = 1e-6;
  for (int d = threadIdx.x; d < dim; d += blockDim.x) {
    const double x = d >= 3 ? wrap_angle(start[d]) : start[d];
    c.g[d] = x;
    c.best[d] = x;
  }
  __syncthreads();
  Frame f;
  if (warp == 0) f = cta_place(S, c);
  __syncthreads();
  const int j0 = warp * S.n_sites / W, j1 = (warp + 1) * S.n_sites / W;
  double sg0 = 0.0, su0 = 0.0, sg1 = 0.0, su1 = 0.0, hist = 0.0;
  LsResult r;
  r.energy = 0.0;
  r.iterations = 0;
  r.converged = 0;
  r.status = MDR_OK;
  for (int iter = 0;; ++iter) {
    for (int i = lane; i < S.n_atoms; i += 32) {
      const double* q = c.world + (size_t)i * 4;
      double e = 0.0;
      d3 gg = {0.0, 0.0, 0.0};
      pair_range<PAIR>(S, d3{q[0], q[1], q[2]}, q[3], j0, j1, e, gg);
      double* o = c.part + ((size_t)warp * S.n_atoms + i) * 4;
      o[0] = e;
      o[1] = gg.x;
      o[2] = gg.y;
      o[3] = gg.z;
    }
    __syncthreads();
    if (warp == 0) {
      const d3 tr = {c.g[0], c.g[1], c.g[2]};
      const ScoreOut o = reduce_atoms<METHOD>(S.n_atoms, partition, half_mode, c.ws, [&](int i) {
        Partial p;
        p.e = 0.0;
        p.g = {0.0, 0.0, 0.0};
        for (int w = 0; w < W; ++w) {
          const double* q = c.part + ((size_t)w * S.n_atoms + i) * 4;
          p.e += q[0];
          p.g = p.g + d3{q[1], q[2], q[3]};
        }
        const double* q = c.world + (size_t)i * 4;
        p.t = cross(d3{q[0], q[1], q[2]} - tr, p.g);
        return p;
      });
      const float gr0 = lane < dim ? project_dim(S, f, o, lane, c.ws) : 0.f;
      const float gr1 = lane + 32 < dim ? project_dim(S, f, o, lane + 32, c.ws) : 0.f;
      const double e = (double)o.sums[0];
      bool done = false;
      if (iter == 0) {
        r.energy = e;
        hist = e;
      } else {
        if (e < r.energy) {
          r.energy = e;
          for (int d = lane; d < dim; d += 32) c.best[d] = c.g[d];
        }
        const int slot = iter & (kWindow - 1);
        const double old = __shfl_sync(kFull, hist, slot);
        if (lane == slot) hist = r.energy;
        r.iterations = iter;
        if (iter >= kWindow && old - r.energy < tol) {
          r.converged = 1;
          done = true;
        }
      }
      if (!done && iter >= max_iters) done = true;
      if (!done) {
        const bool bad = (lane < dim && !isfinite(gr0)) || (lane + 32 < dim && !isfinite(gr1));
        if (__any_sync(kFull, bad)) {
          r.status = MDR_ERR_NUMERIC_DOMAIN;
          done = true;
        } else {
          if (lane < dim) {
            double x = c.g[lane];
            adadelta_dim(sg0, su0, x, (double)gr0, lane, rho, eps);
            c.g[lane] = x;
          }
          if (lane + 32 < dim) {
            double x = c.g[lane + 32];
            adadelta_dim(sg1, su1, x, (double)gr1, lane + 32, rho, eps);
            c.g[lane + 32] = x;
          }
          __syncwarp();
          f = cta_place(S, c);  // next pose
        }
      }
      if (lane == 0) c.ctl[0] = done;
    }
    __syncthreads();
    if (c.ctl[0]) break;
  }
  return r;
}

template <int METHOD, int PAIR>
__global__ void ls_cta_kernel(LigandView L, const double* __restrict__ starts, int n, int max_iters, double tol,
                              int partition, int half_mode, double* __restrict__ out_g, double* __restrict__ out_e,
                              int* __restrict__ out_it, int* __restrict__ out_cv, int* __restrict__ status) {
  extern __shared__ __align__(16) unsigned char smem[];
  const SmemLigand S = load_ligand(L, smem);
  __syncthreads();
  const int item = blockIdx.x;
  if (item >= n) return;
  const CtaCtx c = cta_region(smem + ligand_smem_bytes(L), L.n_atoms, blockDim.x >> 5);
  const int dim = 6 + L.n_rot;
  const LsResult r = local_search_cta<METHOD, PAIR>(S, starts + (size_t)item * dim, max_iters, tol, partition,
                                                    half_mode != 0, c);
  if (threadIdx.x < 32) {
    for (int d = threadIdx.x; d < dim; d += 32) out_g[(size_t)item * dim + d] = c.best[d];
    if (threadIdx.x == 0) {
      out_e[item] = r.energy;
      out_it[item] = r.iterations;
      out_cv[item] = r.converged;
      if (r.status != MDR_OK) status[item] = r.status;
    }
  }
}

// ------------------------------------------------------------- K5 LGA
// lga init: random_genotype docking.cpp:360-388 + score, warp per individual.
template <int METHOD, int PAIR, bool EXACT, bool CHUNK>
__global__ void lga_init_kernel(LigandView L, LgaDev D) {
  extern __shared__ __align__(16) unsigned char smem[];
  const SmemLigand S = load_ligand(L, smem);
  __syncthreads();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int item = blockIdx.x * (blockDim.x >> 5) + warp;
  if (item >= D.R * D.P) return;
  const int run = item / D.P, p = item % D.P;
  WarpCtx w = warp_region(smem + ligand_smem_bytes(L), warp, L);
  const uint64_t key = run_key(D, run);
  for (int d = lane; d < D.dim; d += 32) {
    const uint64_t n = (uint64_t)p * D.dim + d + 1;
    double x;
    if (d < 3)
      x = L.box[d] + (L.box[3 + d] - L.box[d]) * draw_unit(key, n);
    else
      x = -kPi + (kPi - -kPi) * draw_unit(key, n);
    w.g[d] = x;
    D.pop[0][((size_t)run * D.P + p) * D.dim + d] = x;
  }
  __syncwarp();
  Frame f;
  const ScoreOut o = score_sums<METHOD, PAIR, false, CHUNK>(S, w.g, D.partition, D.half_mode != 0, w.ws, f);
  if (lane == 0) D.pope[0][(size_t)run * D.P + p] = (double)o.sums[0];
}


// One offspring per warp: elitism, two binary tournaments, per-dimension
// arithmetic crossover, Gaussian mutation, angle normalisation, score
// (docking.cpp:437-472).  Draw offsets: every generation consumes
// off * (4 + 3*dim) draws after the P*dim initial ones.
template <int METHOD, int PAIR, bool EXACT, bool CHUNK>
__global__ void lga_offspring_kernel(LigandView L, LgaDev D, int gen) {
  extern __shared__ __align__(16) unsigned char smem[];
  const SmemLigand S = load_ligand(L, smem);
  __syncthreads();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int item = blockIdx.x * (blockDim.x >> 5) + warp;
  if (item >= D.R * D.off) return;
  const int run = item / D.off, i = item % D.off;
  if (!D.active[run]) return;
  WarpCtx w = warp_region(smem + ligand_smem_bytes(L), warp, L);
  const int c = D.cur[run];
  const double* pop = D.pop[c] + (size_t)run * D.P * D.dim;
  const double* pe = D.pope[c] + (size_t)run * D.P;
  double* nxt = D.pop[c ^ 1] + (size_t)run * D.P * D.dim;
  double* ne = D.pope[c ^ 1] + (size_t)run * D.P;
  if (i == 0) {  // elitism of one: first index of the strict minimum
    double be = pe[0];
    int bi = 0;
    for (int p = 1; p < D.P; ++p)
      if (pe[p] < be) {
        be = pe[p];
        bi = p;
      }
    for (int d = lane; d < D.dim; d += 32) nxt[d] = pop[(size_t)bi * D.dim + d];
    if (lane == 0) ne[0] = be;
  }
  const uint64_t key = run_key(D, run);
  const uint64_t base = (uint64_t)D.P * D.dim + ((uint64_t)gen * D.off + i) * (uint64_t)(4 + 3 * D.dim);
  const int ia = (int)(draw_u64(key, base + 1) % (uint64_t)D.P);
  const int ja = (int)(draw_u64(key, base + 2) % (uint64_t)D.P);
  const int a = pe[ia] <= pe[ja] ? ia : ja;
  const int ib = (int)(draw_u64(key, base + 3) % (uint64_t)D.P);
  const int jb = (int)(draw_u64(key, base + 4) % (uint64_t)D.P);
  const int b = pe[ib] <= pe[jb] ? ib : jb;
  for (int d = lane; d < D.dim; d += 32) {
    const double lam = draw_unit(key, base + 5 + d);
    double x = lam * pop[(size_t)a * D.dim + d] + (1.0 - lam) * pop[(size_t)b * D.dim + d];
    x = x + D.sigma * draw_normal(key, base + 5 + D.dim + 2 * (uint64_t)d);
    if (d >= 3) x = wrap_angle(x);
    w.g[d] = x;
    nxt[(size_t)(1 + i) * D.dim + d] = x;
  }
  __syncwarp();
  Frame f;
  const ScoreOut o = score_sums<METHOD, PAIR, false, CHUNK>(S, w.g, D.partition, D.half_mode != 0, w.ws, f);
  if (lane == 0) ne[1 + i] = (double)o.sums[0];
}

// Fast pair modes: one CTA per local search (CTA-per-pose kernel K4c).
template <int METHOD, int PAIR>
__global__ void lga_ls_cta_kernel(LigandView L, LgaDev D) {
  extern __shared__ __align__(16) unsigned char smem[];
  const SmemLigand S = load_ligand(L, smem);
  __syncthreads();
  const int item = blockIdx.x;
  if (item >= D.R * D.L) return;
  const int run = item / D.L, r = item % D.L;
  if (!D.active[run]) return;
  const CtaCtx cc = cta_region(smem + ligand_smem_bytes(L), L.n_atoms, blockDim.x >> 5);
  const int c = D.cur[run];
  const int target = ls_target(D, run, r);
  const double* start = D.pop[c ^ 1] + ((size_t)run * D.P + target) * D.dim;
  const LsResult res = local_search_cta<METHOD, PAIR>(S, start, D.ls_iters, D.tol, D.partition, D.half_mode != 0,
                                                      cc);
  if (threadIdx.x < 32) {
    const size_t o = (size_t)run * D.L + r;
    for (int d = threadIdx.x; d < D.dim; d += 32) D.lsg[o * D.dim + d] = cc.best[d];
    if (threadIdx.x == 0) {
      D.lse[o] = res.energy;
      D.lsit[o] = res.iterations;
      D.lscv[o] = res.converged;
      D.lstarget[o] = target;
      if (res.status != MDR_OK) D.status[run] = res.status;
    }
  }
}

// Lamarckian step: the r-th best offspring (stable by index) refined by a
// device-resident local search (docking.cpp:476-489).
template <int METHOD, int PAIR, bool EXACT, bool CHUNK>
__device__ __forceinline__ void lga_ls_body(const LigandView& L, const LgaDev& D) {
  extern __shared__ __align__(16) unsigned char smem[];
  const SmemLigand S = load_ligand(L, smem);
  __syncthreads();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int item = blockIdx.x * (blockDim.x >> 5) + warp;
  if (item >= D.R * D.L) return;
  const int run = item / D.L, r = item % D.L;
  if (!D.active[run]) return;
  WarpCtx w = warp_region(smem + ligand_smem_bytes(L), warp, L);
  const int c = D.cur[run];
  const int target = ls_target(D, run, r);
  const double* start = D.pop[c ^ 1] + ((size_t)run * D.P + target) * D.dim;
  const LsResult res = local_search_warp<METHOD, PAIR, EXACT, CHUNK>(S, start, D.ls_iters, D.tol, D.partition,
                                                       D.half_mode != 0, w);
  const size_t o = (size_t)run * D.L + r;
  for (int d = lane; d < D.dim; d += 32) D.lsg[o * D.dim + d] = w.best[d];
  if (lane == 0) {
    D.lse[o] = res.energy;
    D.lsit[o] = res.iterations;
    D.lscv[o] = res.converged;
    D.lstarget[o] = target;
    if (res.status != MDR_OK) D.status[run] = res.status;
  }
}

// The dominant kernel.  FP32 pair terms run without the register hint (the
// hint costs that mode 218.7 -> 205.4 M evals/s; the FP64 modes and the
// tensor-core reductions gain from it, TcuSplit 113 -> 150 M).
template <int METHOD, int PAIR, bool EXACT, bool CHUNK>
__global__ void MDR_LS_BOUNDS lga_ls_kernel(LigandView L, LgaDev D) {
  lga_ls_body<METHOD, PAIR, EXACT, CHUNK>(L, D);
}
template <int METHOD, int PAIR, bool EXACT, bool CHUNK>
__global__ void lga_ls_kernel_nb(LigandView L, LgaDev D) {
  lga_ls_body<METHOD, PAIR, EXACT, CHUNK>(L, D);
}

// Warp-pair search (FP64-fast, chunked sites): two warps per Lamarckian
// search; the leader runs local_search_warp<..., CHUNK = 2> and the helper
// takes half of each evaluation's chunk items (pair_helper).  Same items,
// same per-item arithmetic, same combine order as the one-warp kernel, so
// the results are bit-identical; per evaluation two named barriers.
template <int METHOD>
__global__ void MDR_LS_BOUNDS lga_ls_pair_kernel(LigandView L, LgaDev D) {
  extern __shared__ __align__(16) unsigned char smem[];
  SmemLigand S = load_ligand(L, smem);
  S.nch = L.ls_n_chunks;  // the search's own chunking (64 lanes)
  S.clen = L.ls_chunk_len;
  __syncthreads();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, pose = warp >> 1;
  const int item = blockIdx.x * (blockDim.x >> 6) + pose;
  if (item >= D.R * D.L) return;
  const int run = item / D.L, r = item % D.L;
  if (!D.active[run]) return;
  WarpCtx w = warp_region(smem + ligand_smem_bytes(L), pose, L);
  w.ws.bar = 1 + 2 * pose;  // B1; B2 = bar + 1
#if MDR_PHASE_PROF
  // leader: phases 0-6 (+ [7] evaluations); helper: 8-10 (own slots)
  if (lane == 0) {
    if (!(warp & 1))
      for (int k = 0; k < 16; ++k) w.ws.prof[k] = 0;
  }
  pair_bar(w.ws.bar);
  if (lane == 0) w.ws.prof[(warp & 1) ? 14 : 15] = clock64();
  pair_bar(w.ws.bar);
  if (warp & 1) {
    // the helper keeps its own last stamp in slot 14
    long long* pf = w.ws.prof;
    for (;;) {
      nbar_sync(w.ws.bar, 64);
      if (lane == 0) { const long long t = clock64(); pf[8] += t - pf[14]; pf[14] = t; }
      if (*w.ws.ctl == 0) break;
      fast_sums_items(S, w.ws, 32 + lane, 64);
      if (lane == 0) { const long long t = clock64(); pf[9] += t - pf[14]; pf[14] = t; }
      __syncwarp();
      nbar_arrive(w.ws.bar + 1, 64);
      if (lane == 0) { const long long t = clock64(); pf[10] += t - pf[14]; pf[14] = t; }
    }
    if (lane == 0)
      for (int k = 8; k <= 10; ++k) atomicAdd(&g_phase[k], (unsigned long long)pf[k]);
    return;
  }
#else
  if (warp & 1) {
    pair_helper(S, w.ws);
    return;
  }
#endif
  const int c = D.cur[run];
  const int target = ls_target(D, run, r);
  const double* start = D.pop[c ^ 1] + ((size_t)run * D.P + target) * D.dim;
  const LsResult res = local_search_warp<METHOD, MDR_PAIR_FP64_FAST, false, 2>(S, start, D.ls_iters, D.tol,
                                                                              D.partition, D.half_mode != 0, w);
  if (lane == 0) *w.ws.ctl = 0;
  __syncwarp();
  nbar_arrive(w.ws.bar, 64);  // release the helper
#if MDR_PHASE_PROF
  if (lane == 0) {
    for (int k = 0; k <= 6; ++k) atomicAdd(&g_phase[k], (unsigned long long)w.ws.prof[k]);
    atomicAdd(&g_phase[7], (unsigned long long)(res.iterations + 1));
    atomicAdd(&g_phase[11], 1ull);
  }
#endif
  const size_t o = (size_t)run * D.L + r;
  for (int d = lane; d < D.dim; d += 32) D.lsg[o * D.dim + d] = w.best[d];
  if (lane == 0) {
    D.lse[o] = res.energy;
    D.lsit[o] = res.iterations;
    D.lscv[o] = res.converged;
    D.lstarget[o] = target;
    if (res.status != MDR_OK) D.status[run] = res.status;
  }
}


// Initial population bookkeeping (docking.cpp:405-422), warp per run:
// track_best over the P scored individuals in index order.
__global__ void lga_init_finalize(LgaDev D) {
  const int lane = threadIdx.x & 31;
  const int run = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (run >= D.R) return;
  const double* pe = D.pope[0] + (size_t)run * D.P;
  const int w = warp_first_min(D.P, 1.7976931348623157e308, [&](int p) { return pe[p]; });
  const double* g = D.pop[0] + ((size_t)run * D.P + (w < 0 ? 0 : w)) * D.dim;
  for (int d = lane; d < D.dim; d += 32) D.best_g[(size_t)run * D.dim + d] = w < 0 ? 0.0 : g[d];
  if (lane == 0) {
    D.best_e[run] = w < 0 ? 1.7976931348623157e308 : pe[w];  // numeric_limits<double>::max()
    D.evals[run] = D.P;
    D.cur[run] = 0;
    D.nrec[run] = 0;
    D.conv[run] = 0;
    D.status[run] = MDR_OK;
    D.active[run] = D.gens > 0 && budget_ok(D, D.P);
    D.ls_done[run] = 0;
  }
  if (run == 0)  // work counters of the persistent search kernel: one per generation, one for the polish
    for (int g = lane; g <= D.gens; g += 32) D.ls_next[g] = 0;
}

// Bookkeeping of one generation, warp per run, with the reference's
// sequential semantics (docking.cpp:472-496): track_best over offspring
// 1..off, then for each LS rank r: write back, track_best, record.  The
// sequential best tracking is the first occurrence of the minimum over that
// candidate order; write-backs go to distinct offspring and run in parallel.
__global__ void lga_gen_finalize(LgaDev D, int gen) {
  const int run = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (run >= D.R || !D.active[run]) return;
  gen_finalize_run(D, gen, run);
}

// Final polish from the incumbent best (docking.cpp:501-515), warp per run.
template <int METHOD, int PAIR, bool EXACT, bool CHUNK>
__global__ void MDR_LS_BOUNDS lga_polish_kernel(LigandView L, LgaDev D) {
  extern __shared__ __align__(16) unsigned char smem[];
  const SmemLigand S = load_ligand(L, smem);
  __syncthreads();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int run = blockIdx.x * (blockDim.x >> 5) + warp;
  if (run >= D.R || D.status[run] != MDR_OK) return;
  const long long remaining = D.max_evals - D.evals[run];
  if (remaining <= 1) {
    if (lane == 0) D.conv[run] = 0;
    return;
  }
  const int iters = (int)((long long)D.ls_iters < remaining - 1 ? (long long)D.ls_iters : remaining - 1);
  WarpCtx w = warp_region(smem + ligand_smem_bytes(L), warp, L);
  const LsResult res = local_search_warp<METHOD, PAIR, EXACT, CHUNK>(S, D.best_g + (size_t)run * D.dim, iters, D.tol,
                                                       D.partition, D.half_mode != 0, w);
  if (lane == 0) {
    if (res.status != MDR_OK) {
      D.status[run] = res.status;
      return;
    }
    D.evals[run] += res.iterations + 1;
    track_best(D, run, w.best, res.energy);
    push_record(D, run, res.energy, res.iterations, res.converged);
    D.conv[run] = res.converged;
  }
}

template <int METHOD, int PAIR>
__global__ void lga_polish_cta_kernel(LigandView L, LgaDev D) {
  extern __shared__ __align__(16) unsigned char smem[];
  const SmemLigand S = load_ligand(L, smem);
  __syncthreads();
  const int run = blockIdx.x;
  if (run >= D.R || D.status[run] != MDR_OK) return;
  const long long remaining = D.max_evals - D.evals[run];
  if (remaining <= 1) {
    if (threadIdx.x == 0) D.conv[run] = 0;
    return;
  }
  const int iters = (int)((long long)D.ls_iters < remaining - 1 ? (long long)D.ls_iters : remaining - 1);
  const CtaCtx cc = cta_region(smem + ligand_smem_bytes(L), L.n_atoms, blockDim.x >> 5);
  const LsResult res = local_search_cta<METHOD, PAIR>(S, D.best_g + (size_t)run * D.dim, iters, D.tol, D.partition,
                                                      D.half_mode != 0, cc);
  __syncthreads();  // every warp has finished reading best_g before it is updated
  if (threadIdx.x == 0) {
    if (res.status != MDR_OK) {
      D.status[run] = res.status;
      return;
    }
    D.evals[run] += res.iterations + 1;
    track_best(D, run, cc.best, res.energy);
    push_record(D, run, res.energy, res.iterations, res.converged);
    D.conv[run] = res.converged;
  }
}

__global__ void lga_total_evals(LgaDev D, long long* out) {
  long long s = 0;
  for (int r = threadIdx.x; r < D.R; r += blockDim.x) s += D.evals[r];
#pragma unroll
  for (int off = 16; off >= 1; off >>= 1) s += __shfl_xor_sync(kFull, s, off);
  __shared__ long long part[32];
  if ((threadIdx.x & 31) == 0) part[threadIdx.x >> 5] = s;
  __syncthreads();
  if (threadIdx.x == 0) {
    long long t = 0;
    for (int i = 0; i < (int)(blockDim.x >> 5); ++i) t += part[i];
    *out = t;
  }
}

// ------------------------------------------------------------ host side
static size_t warp_smem(const LigandView& L, int wpb) { return ligand_smem_bytes(L) + (size_t)wpb * warp_region_bytes(L); }

template <class K>
static cudaError_t prep(K kernel, size_t smem) {
  if (smem > 48 * 1024) return cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  return cudaSuccess;
}

#define MDR_GEN_DISPATCH(KERNEL)                                                                     \
  template <class... A>                                                                              \
  static void dispatch_##KERNEL(int method, int pair, dim3 g, dim3 b, size_t smem, cudaStream_t s,   \
                                A... args) {                                                         \
    switch (method * 3 + pair) {                                                                     \
      case 0: KERNEL<MDR_METHOD_BASELINE, MDR_PAIR_FP64><<<g, b, smem, s>>>(args...); break;         \
      case 1: KERNEL<MDR_METHOD_BASELINE, MDR_PAIR_FP32><<<g, b, smem, s>>>(args...); break;         \
      case 2: KERNEL<MDR_METHOD_BASELINE, MDR_PAIR_FP64_FAST><<<g, b, smem, s>>>(args...); break;    \
      case 3: KERNEL<MDR_METHOD_TCU, MDR_PAIR_FP64><<<g, b, smem, s>>>(args...); break;              \
      case 4: KERNEL<MDR_METHOD_TCU, MDR_PAIR_FP32><<<g, b, smem, s>>>(args...); break;              \
      case 5: KERNEL<MDR_METHOD_TCU, MDR_PAIR_FP64_FAST><<<g, b, smem, s>>>(args...); break;         \
      case 6: KERNEL<MDR_METHOD_TCU_SPLIT, MDR_PAIR_FP64><<<g, b, smem, s>>>(args...); break;        \
      case 7: KERNEL<MDR_METHOD_TCU_SPLIT, MDR_PAIR_FP32><<<g, b, smem, s>>>(args...); break;        \
      default: KERNEL<MDR_METHOD_TCU_SPLIT, MDR_PAIR_FP64_FAST><<<g, b, smem, s>>>(args...); break;  \
    }                                                                                                \
  }                                                                                                  \
  static cudaError_t prep_##KERNEL(int method, int pair, size_t smem) {                              \
    switch (method * 3 + pair) {                                                                     \
      case 0: return prep(KERNEL<MDR_METHOD_BASELINE, MDR_PAIR_FP64>, smem);                         \
      case 1: return prep(KERNEL<MDR_METHOD_BASELINE, MDR_PAIR_FP32>, smem);                         \
      case 2: return prep(KERNEL<MDR_METHOD_BASELINE, MDR_PAIR_FP64_FAST>, smem);                    \
      case 3: return prep(KERNEL<MDR_METHOD_TCU, MDR_PAIR_FP64>, smem);                              \
      case 4: return prep(KERNEL<MDR_METHOD_TCU, MDR_PAIR_FP32>, smem);                              \
      case 5: return prep(KERNEL<MDR_METHOD_TCU, MDR_PAIR_FP64_FAST>, smem);                         \
      case 6: return prep(KERNEL<MDR_METHOD_TCU_SPLIT, MDR_PAIR_FP64>, smem);                        \
      case 7: return prep(KERNEL<MDR_METHOD_TCU_SPLIT, MDR_PAIR_FP32>, smem);                        \
      default: return prep(KERNEL<MDR_METHOD_TCU_SPLIT, MDR_PAIR_FP64_FAST>, smem);                  \
    }                                                                                                \
  }

// Kernels with an exact-torsion variant: the flag (LigandView::exact_torsion)
// selects a separate instantiation, so the default kernels carry no trace of it.
#define MDR_GEN_DISPATCH_EXACT(KERNEL)                                                                   \
  template <bool X, bool CH>                                                                             \
  struct KERNEL##_x {                                                                                    \
    template <int M, int P>                                                                              \
    static constexpr auto k = KERNEL##_sel<M, P, X, CH && P == MDR_PAIR_FP64_FAST>::k();                 \
  };                                                                                                     \
  template <class... A>                                                                                  \
  static void dispatch_##KERNEL(int method, int pair, const LigandView& L, dim3 g, dim3 b, size_t smem,  \
                                cudaStream_t s, A... args) {                                             \
    const bool x = L.exact_torsion != 0, ch = L.n_chunks > 1;                           \
    if (x && ch)                                                                                         \
      dispatch_mp<KERNEL##_x<true, true>>(method, pair, g, b, smem, s, args...);                         \
    else if (x)                                                                                          \
      dispatch_mp<KERNEL##_x<true, false>>(method, pair, g, b, smem, s, args...);                        \
    else if (ch)                                                                                         \
      dispatch_mp<KERNEL##_x<false, true>>(method, pair, g, b, smem, s, args...);                        \
    else                                                                                                 \
      dispatch_mp<KERNEL##_x<false, false>>(method, pair, g, b, smem, s, args...);                       \
  }                                                                                                      \
  static cudaError_t prep_##KERNEL(int method, int pair, const LigandView& L, size_t smem) {             \
    const bool x = L.exact_torsion != 0, ch = L.n_chunks > 1;                           \
    if (x && ch) return prep_mp<KERNEL##_x<true, true>>(method, pair, smem);                             \
    if (x) return prep_mp<KERNEL##_x<true, false>>(method, pair, smem);                                  \
    if (ch) return prep_mp<KERNEL##_x<false, true>>(method, pair, smem);                                 \
    return prep_mp<KERNEL##_x<false, false>>(method, pair, smem);                                        \
  }

// Kernels that only score (no gradient projection): chunking variant only.
#define MDR_GEN_DISPATCH_CHUNK(KERNEL)                                                                   \
  template <bool CH>                                                                                     \
  struct KERNEL##_x {                                                                                    \
    template <int M, int P>                                                                              \
    static constexpr auto k = KERNEL<M, P, false, CH && P == MDR_PAIR_FP64_FAST>;                        \
  };                                                                                                     \
  template <class... A>                                                                                  \
  static void dispatch_##KERNEL(int method, int pair, const LigandView& L, dim3 g, dim3 b, size_t smem,  \
                                cudaStream_t s, A... args) {                                             \
    if (L.n_chunks > 1)                                                                 \
      dispatch_mp<KERNEL##_x<true>>(method, pair, g, b, smem, s, args...);                               \
    else                                                                                                 \
      dispatch_mp<KERNEL##_x<false>>(method, pair, g, b, smem, s, args...);                              \
  }                                                                                                      \
  static cudaError_t prep_##KERNEL(int method, int pair, const LigandView& L, size_t smem) {             \
    return L.n_chunks > 1 ? prep_mp<KERNEL##_x<true>>(method, pair, smem)                                \
                          : prep_mp<KERNEL##_x<false>>(method, pair, smem);                              \
  }

template <class T, class... A>
static void dispatch_mp(int method, int pair, dim3 g, dim3 b, size_t smem, cudaStream_t s, A... args) {
  switch (method * 3 + pair) {
    case 0: T::template k<MDR_METHOD_BASELINE, MDR_PAIR_FP64><<<g, b, smem, s>>>(args...); break;
    case 1: T::template k<MDR_METHOD_BASELINE, MDR_PAIR_FP32><<<g, b, smem, s>>>(args...); break;
    case 2: T::template k<MDR_METHOD_BASELINE, MDR_PAIR_FP64_FAST><<<g, b, smem, s>>>(args...); break;
    case 3: T::template k<MDR_METHOD_TCU, MDR_PAIR_FP64><<<g, b, smem, s>>>(args...); break;
    case 4: T::template k<MDR_METHOD_TCU, MDR_PAIR_FP32><<<g, b, smem, s>>>(args...); break;
    case 5: T::template k<MDR_METHOD_TCU, MDR_PAIR_FP64_FAST><<<g, b, smem, s>>>(args...); break;
    case 6: T::template k<MDR_METHOD_TCU_SPLIT, MDR_PAIR_FP64><<<g, b, smem, s>>>(args...); break;
    case 7: T::template k<MDR_METHOD_TCU_SPLIT, MDR_PAIR_FP32><<<g, b, smem, s>>>(args...); break;
    default: T::template k<MDR_METHOD_TCU_SPLIT, MDR_PAIR_FP64_FAST><<<g, b, smem, s>>>(args...); break;
  }
}

template <class T>
static cudaError_t prep_mp(int method, int pair, size_t smem) {
  switch (method * 3 + pair) {
    case 0: return prep(T::template k<MDR_METHOD_BASELINE, MDR_PAIR_FP64>, smem);
    case 1: return prep(T::template k<MDR_METHOD_BASELINE, MDR_PAIR_FP32>, smem);
    case 2: return prep(T::template k<MDR_METHOD_BASELINE, MDR_PAIR_FP64_FAST>, smem);
    case 3: return prep(T::template k<MDR_METHOD_TCU, MDR_PAIR_FP64>, smem);
    case 4: return prep(T::template k<MDR_METHOD_TCU, MDR_PAIR_FP32>, smem);
    case 5: return prep(T::template k<MDR_METHOD_TCU, MDR_PAIR_FP64_FAST>, smem);
    case 6: return prep(T::template k<MDR_METHOD_TCU_SPLIT, MDR_PAIR_FP64>, smem);
    case 7: return prep(T::template k<MDR_METHOD_TCU_SPLIT, MDR_PAIR_FP32>, smem);
    default: return prep(T::template k<MDR_METHOD_TCU_SPLIT, MDR_PAIR_FP64_FAST>, smem);
  }
}

// Kernel instantiation a dispatch uses: the kernel itself, except the
// FP32-pair LGA search (lga_ls_kernel_nb, no register hint).
#define MDR_SEL_DEFAULT(KERNEL)                              \
  template <int M, int P, bool X, bool C>                    \
  struct KERNEL##_sel {                                      \
    static constexpr auto k() { return &KERNEL<M, P, X, C>; } \
  };
MDR_SEL_DEFAULT(score_kernel)
MDR_SEL_DEFAULT(ls_kernel)
MDR_SEL_DEFAULT(lga_polish_kernel)
template <int M, int P, bool X, bool C>
struct lga_ls_kernel_sel {
  static constexpr auto k() {
    if constexpr (P == MDR_PAIR_FP32)
      return &lga_ls_kernel_nb<M, P, X, C>;
    else
      return &lga_ls_kernel<M, P, X, C>;
  }
};

MDR_GEN_DISPATCH_EXACT(score_kernel)
MDR_GEN_DISPATCH_EXACT(ls_kernel)
MDR_GEN_DISPATCH(ls_cta_kernel)
MDR_GEN_DISPATCH_CHUNK(lga_init_kernel)
MDR_GEN_DISPATCH_CHUNK(lga_offspring_kernel)
MDR_GEN_DISPATCH_EXACT(lga_ls_kernel)
MDR_GEN_DISPATCH(lga_ls_cta_kernel)
MDR_GEN_DISPATCH_EXACT(lga_polish_kernel)
MDR_GEN_DISPATCH(lga_polish_cta_kernel)

static inline int blocks_for(long long items, int wpb) { return (int)((items + wpb - 1) / wpb); }
static size_t cta_smem(const LigandView& L, int cw) { return ligand_smem_bytes(L) + cta_region_bytes(L.n_atoms, cw); }

cudaError_t launch_score(const LigandView& L, const double* genos, int n, int method, int pair, int partition,
                         int half_mode, float* energy, float* grad, float* torque, cudaStream_t s, int wpb) {
  if (n <= 0) return cudaSuccess;
  const size_t smem = warp_smem(L, wpb);
  cudaError_t e = prep_score_kernel(method, pair, L, smem);
  if (e != cudaSuccess) return e;
  dispatch_score_kernel(method, pair, L, blocks_for(n, wpb), 32 * wpb, smem, s, L, genos, n, partition, half_mode,
                        energy, grad, torque);
  return cudaGetLastError();
}

cudaError_t launch_score_reference(const LigandView& L, const double* genos, int n, double* energy, double* grad,
                                   double* torque, cudaStream_t s, int wpb) {
  if (n <= 0) return cudaSuccess;
  const size_t smem = warp_smem(L, wpb);
  cudaError_t e = prep(scoreref_kernel, smem);
  if (e != cudaSuccess) return e;
  scoreref_kernel<<<blocks_for(n, wpb), 32 * wpb, smem, s>>>(L, genos, n, energy, grad, torque);
  return cudaGetLastError();
}

cudaError_t launch_adadelta(int dim, int n, double rho, double eps, double* sq_g, double* sq_u, double* geno,
                            const double* grad, int* status, cudaStream_t s) {
  if (n <= 0) return cudaSuccess;
  adadelta_kernel<<<blocks_for(n, 4), 128, 0, s>>>(dim, n, rho, eps, sq_g, sq_u, geno, grad, status);
  return cudaGetLastError();
}

cudaError_t launch_local_search(const LigandView& L, const double* starts, int n, int max_iters, double tol,
                                int method, int pair, int partition, int half_mode, double* out_g, double* out_e,
                                int* out_it, int* out_cv, int* status, cudaStream_t s, int wpb, int cta_warps) {
  if (n <= 0) return cudaSuccess;
  cudaError_t e;
  if (cta_warps > 0) {
    const size_t smem = cta_smem(L, cta_warps);
    e = prep_ls_cta_kernel(method, pair, smem);
    if (e != cudaSuccess) return e;
    dispatch_ls_cta_kernel(method, pair, n, 32 * cta_warps, smem, s, L, starts, n, max_iters, tol, partition,
                           half_mode, out_g, out_e, out_it, out_cv, status);
  } else {
    const size_t smem = warp_smem(L, wpb);
    e = prep_ls_kernel(method, pair, L, smem);
    if (e != cudaSuccess) return e;
    dispatch_ls_kernel(method, pair, L, blocks_for(n, wpb), 32 * wpb, smem, s, L, starts, n, max_iters, tol, partition,
                       half_mode, out_g, out_e, out_it, out_cv, status);
  }
  return cudaGetLastError();
}

// Legacy warp-pair Lamarckian search (lga_ls_pair_kernel): FP64-fast chunked
// ligands the two-warp kernel does not take (n_atoms or dim > 32), at most 7
// searches per CTA (two named barriers each, ids 1..14).
#ifndef MDR_LS_PAIR
#define MDR_LS_PAIR 1
#endif
static bool use_ls_pair(const LigandView& L, int pair, int wpb, int cta_warps) {
  return MDR_LS_PAIR && L.ls_pair && L.ls_warps != 1 && cta_warps == 0 && pair == MDR_PAIR_FP64_FAST &&
         L.ls_n_chunks > 1 && !L.exact_torsion && L.n_atoms * L.ls_n_chunks > 32 && wpb <= 7;  // 2 barriers per search
}
static cudaError_t prep_ls_pair(int method, size_t smem) {
  switch (method) {
    case MDR_METHOD_BASELINE: return prep(lga_ls_pair_kernel<MDR_METHOD_BASELINE>, smem);
    case MDR_METHOD_TCU: return prep(lga_ls_pair_kernel<MDR_METHOD_TCU>, smem);
    default: return prep(lga_ls_pair_kernel<MDR_METHOD_TCU_SPLIT>, smem);
  }
}
static void launch_ls_pair(int method, int blocks, int threads, size_t smem, cudaStream_t s, const LigandView& L,
                           const LgaDev& D) {
  switch (method) {
    case MDR_METHOD_BASELINE: lga_ls_pair_kernel<MDR_METHOD_BASELINE><<<blocks, threads, smem, s>>>(L, D); break;
    case MDR_METHOD_TCU: lga_ls_pair_kernel<MDR_METHOD_TCU><<<blocks, threads, smem, s>>>(L, D); break;
    default: lga_ls_pair_kernel<MDR_METHOD_TCU_SPLIT><<<blocks, threads, smem, s>>>(L, D); break;
  }
}

// Warps of the CTA-per-pose final polish in the fast pair modes (the polish
// runs one search per LGA run, so its latency, not throughput, counts).
#ifndef MDR_POLISH_CTA
#define MDR_POLISH_CTA 4  // measured: 0 / 2 / 4 / 8 -> 139.3 / 139.4 / 141.3 / 141.3 M evals/s on C3
#endif
// The final polish: on the two-warp persistent search when the searches run
// there; otherwise, for ligands that would qualify for it (A/B contexts:
// MDR_LS_WARPS 0 or 1), on the one-warp search kernel, so every search
// configuration gives bit-identical dockings; else the CTA-per-pose polish.
static bool polish_multi(const LigandView& L, int pair, int wpb, int cta_warps) {
  return ls_multi_supported(L, pair, wpb, cta_warps);
}
static bool polish_one_warp(const LigandView& L, int pair, int wpb, int cta_warps) {
  LigandView M = L;
  M.ls_pair = 1;
  M.ls_warps = 2;
  return !polish_multi(L, pair, wpb, cta_warps) && ls_multi_supported(M, pair, wpb, cta_warps);
}
static int polish_warps(const LigandView& L, int pair, int cta_warps) {
  if (L.exact_torsion) return 0;  // exact-torsion staging lives in the warp-per-pose region
  return cta_warps > 0 ? cta_warps : (pair != MDR_PAIR_FP64 ? MDR_POLISH_CTA : 0);
}

cudaError_t prepare_lga(const LigandView& L, int method, int pair, int wpb, int cta_warps) {
  const size_t smem = warp_smem(L, wpb);
  const int pw = polish_multi(L, pair, wpb, cta_warps) || polish_one_warp(L, pair, wpb, cta_warps)
                     ? 0
                     : polish_warps(L, pair, cta_warps);
  cudaError_t e = prep_lga_init_kernel(method, pair, L, smem);
  if (e == cudaSuccess) e = prep_lga_offspring_kernel(method, pair, L, smem);
  if (cta_warps > 0) {
    if (e == cudaSuccess) e = prep_lga_ls_cta_kernel(method, pair, cta_smem(L, cta_warps));
  } else if (ls_multi_supported(L, pair, wpb, cta_warps)) {
    if (e == cudaSuccess) e = prep_ls_multi(L, method);
  } else if (use_ls_pair(L, pair, wpb, cta_warps)) {
    if (e == cudaSuccess) e = prep_ls_pair(method, smem);
  } else {
    if (e == cudaSuccess) e = prep_lga_ls_kernel(method, pair, L, smem);
  }
  if (pw > 0) {
    if (e == cudaSuccess) e = prep_lga_polish_cta_kernel(method, pair, cta_smem(L, pw));
  } else {
    if (e == cudaSuccess) e = prep_lga_polish_kernel(method, pair, L, smem);
  }
  return e;
}

// Enqueue a whole docking batch; prepare_lga() must have run (it is not
// capture-safe, launch_lga is).  cta_warps > 0 selects the CTA-per-pose
// local-search kernels.
cudaError_t launch_lga(const LigandView& L, const LgaDev& D, int method, int pair, cudaStream_t s, int wpb,
                       int cta_warps, int* n_launches, cudaEvent_t* ls_events) {
  // ls_events (optional, profiling replay only): 2 per generation bracketing
  // the LS kernel, then 2 bracketing the polish, then 2 bracketing the step.
  const size_t smem = warp_smem(L, wpb);
  const size_t cs = cta_smem(L, cta_warps > 0 ? cta_warps : 1);
  int launches = 0;
  if (ls_events) cudaEventRecord(ls_events[2 * D.gens + 2], s);
  dispatch_lga_init_kernel(method, pair, L, blocks_for((long long)D.R * D.P, wpb), 32 * wpb, smem, s, L, D);
  lga_init_finalize<<<(D.R + 3) / 4, 128, 0, s>>>(D);
  launches += 2;
  for (int gen = 0; gen < D.gens; ++gen) {
    dispatch_lga_offspring_kernel(method, pair, L, blocks_for((long long)D.R * D.off, wpb), 32 * wpb, smem, s, L, D,
                                  gen);
    if (ls_events) cudaEventRecord(ls_events[2 * gen], s);
    if (D.L > 0) {
      if (cta_warps > 0)
        dispatch_lga_ls_cta_kernel(method, pair, D.R * D.L, 32 * cta_warps, cs, s, L, D);
      else if (ls_multi_supported(L, pair, wpb, cta_warps))
        launch_ls_multi(L, D, method, gen, s);  // finalizes each run inside (MDR_LS_FUSE_FINALIZE)
      else if (use_ls_pair(L, pair, wpb, cta_warps))
        launch_ls_pair(method, blocks_for((long long)D.R * D.L, wpb), 64 * wpb, smem, s, L, D);
      else
        dispatch_lga_ls_kernel(method, pair, L, blocks_for((long long)D.R * D.L, wpb), 32 * wpb, smem, s, L, D);
    }
    if (ls_events) cudaEventRecord(ls_events[2 * gen + 1], s);
    const bool fused = MDR_LS_FUSE_FINALIZE && D.L > 0 && cta_warps == 0 && ls_multi_supported(L, pair, wpb, cta_warps);
    if (!fused) lga_gen_finalize<<<(D.R + 3) / 4, 128, 0, s>>>(D, gen);
    launches += (D.L > 0 ? 2 : 1) + (fused ? 0 : 1);
  }
  if (ls_events) cudaEventRecord(ls_events[2 * D.gens], s);
  if (polish_multi(L, pair, wpb, cta_warps)) {
    launch_ls_multi(L, D, method, D.gens, s);
  } else if (polish_one_warp(L, pair, wpb, cta_warps)) {
    LigandView P = L;  // the search's own chunking, as the two-warp polish would use
    P.n_chunks = L.ls_n_chunks;
    P.chunk_len = L.ls_chunk_len;
    dispatch_lga_polish_kernel(method, pair, P, blocks_for(D.R, wpb), 32 * wpb, smem, s, P, D);
  } else {
    const int pw = polish_warps(L, pair, cta_warps);
    if (pw > 0)
      dispatch_lga_polish_cta_kernel(method, pair, D.R, 32 * pw, cta_smem(L, pw), s, L, D);
    else
      dispatch_lga_polish_kernel(method, pair, L, blocks_for(D.R, wpb), 32 * wpb, smem, s, L, D);
  }
  if (ls_events) cudaEventRecord(ls_events[2 * D.gens + 1], s);
  if (ls_events) cudaEventRecord(ls_events[2 * D.gens + 3], s);
  launches += 1;
  if (n_launches) *n_launches = launches;
  return cudaGetLastError();
}

// ---- self test of the correctly rounded math (crmath.cuh) against glibc:
// for input i (counter-generated like RngStream), 8 results: cr sin, cos of
// a = -pi + 2 pi u, cr log(u1), cr cos(2 pi u2), then the same with libdevice.
__global__ void crmath_probe_kernel(long long i0, int n, double* __restrict__ out) {
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= n) return;
  const uint64_t i = (uint64_t)(i0 + t);
  const double a = -kPi + 2.0 * kPi * draw_unit(0, 4 * i + 1);
  const double u1 = (double)((draw_u64(0, 4 * i + 2) >> 11) + 1) * 0x1p-53;
  const double z = 2.0 * kPi * draw_unit(0, 4 * i + 3);
  double* o = out + 8 * (size_t)t;
  cr::sincos(a, &o[0], &o[1]);
  o[2] = cr::log(u1);
  o[3] = cr::cos(z);
  ::sincos(a, &o[4], &o[5]);
  o[6] = ::log(u1);
  o[7] = ::cos(z);
}

cudaError_t launch_crmath_probe(long long i0, int n, double* out, cudaStream_t s) {
  crmath_probe_kernel<<<(n + 255) / 256, 256, 0, s>>>(i0, n, out);
  return cudaGetLastError();
}

cudaError_t launch_lga_init_finalize(const LgaDev& D, cudaStream_t s) {
  lga_init_finalize<<<(D.R + 3) / 4, 128, 0, s>>>(D);
  return cudaGetLastError();
}

cudaError_t launch_lga_gen_finalize(const LgaDev& D, int gen, cudaStream_t s) {
  lga_gen_finalize<<<(D.R + 3) / 4, 128, 0, s>>>(D, gen);
  return cudaGetLastError();
}

cudaError_t launch_lga_total(const LgaDev& D, long long* out, cudaStream_t s) {
  lga_total_evals<<<1, 256, 0, s>>>(D, out);
  return cudaGetLastError();
}

// Phase-profile counters of an MDR_PHASE_PROF build (false otherwise).
bool phase_prof_read(unsigned long long* out16, bool reset) {
#if MDR_PHASE_PROF
  if (cudaMemcpyFromSymbol(out16, g_phase, sizeof(unsigned long long) * 16) != cudaSuccess) return false;
  if (reset) {
    unsigned long long z[16] = {};
    if (cudaMemcpyToSymbol(g_phase, z, sizeof(z)) != cudaSuccess) return false;
  }
  return phase_prof_read_multi(out16, reset);  // ls_multi.cu's counters (one search kernel runs at a time)
#else
  (void)out16;
  (void)reset;
  return false;
#endif
}

}  // namespace mdr
