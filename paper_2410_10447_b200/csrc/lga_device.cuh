// lga_device.cuh — device helpers of the LGA driver shared by the analytic
// (dock.cu) and grid-map (grid.cu) kernels: lga_run docking.cpp:392-517.
#pragma once

#include "mdr_device.cuh"

namespace mdr {

__device__ __forceinline__ uint64_t run_key(const LgaDev& D, int run) {
  return mix64(D.seeds[run] ^ D.label_hash);  // RngStream ctor rng.cpp:31-32
}

__device__ __forceinline__ void track_best(const LgaDev& D, int run, const double* g, double e) {
  if (e < D.best_e[run]) {  // strict: first occurrence wins (docking.cpp:408-413)
    D.best_e[run] = e;
    for (int d = 0; d < D.dim; ++d) D.best_g[(size_t)run * D.dim + d] = g[d];
  }
}

__device__ __forceinline__ bool budget_ok(const LgaDev& D, long long evals) {
  // docking.cpp:430-435
  return evals + D.off + (long long)D.L * (D.ls_iters + 1) <= D.max_evals;
}

// Index (1..off) of the offspring of rank r in the stable (energy, index)
// order of docking.cpp:476-483; every lane of the calling warp gets it.
__device__ __forceinline__ int ls_target(const LgaDev& D, int run, int r) {
  const int lane = threadIdx.x & 31;
  const double* ne = D.pope[D.cur[run] ^ 1] + (size_t)run * D.P;
  int target = -1;
  for (int j = 1 + lane; j <= D.off; j += 32) {
    const double ej = ne[j];
    int rank = 0;
    for (int k = 1; k <= D.off; ++k) {
      const double ek = ne[k];
      rank += (ek < ej) || (ek == ej && k < j);
    }
    if (rank == r) target = j;
  }
#pragma unroll
  for (int off = 16; off >= 1; off >>= 1) target = max(target, __shfl_xor_sync(kFull, target, off));
  return target;
}

__device__ __forceinline__ void push_record(const LgaDev& D, int run, double e, int it, int cv) {
  const int k = D.nrec[run];
  if (k < D.maxrec) {
    mdr_ls_record rec;
    rec.best_energy = e;
    rec.iterations = it;
    rec.converged = cv;
    D.recs[(size_t)run * D.maxrec + k] = rec;
  }
  D.nrec[run] = k + 1;
}

// First occurrence of the strict minimum of candidate energies e(0..n-1)
// (NaN never wins), by the calling warp: the result of applying
// track_best (docking.cpp:408-413) to the candidates in order, starting from
// `cur`.  Returns -1 when no candidate is below `cur`.
template <class E>
__device__ __forceinline__ int warp_first_min(int n, double cur, E&& energy) {
  const int lane = threadIdx.x & 31;
  double m = cur;
  int idx = -1;
  for (int k = lane; k < n; k += 32) {
    const double e = energy(k);
    if (e < m) {  // per lane, k ascending: first occurrence kept
      m = e;
      idx = k;
    }
  }
#pragma unroll
  for (int off = 16; off >= 1; off >>= 1) {
    const double om = __shfl_xor_sync(kFull, m, off);
    const int oi = __shfl_xor_sync(kFull, idx, off);
    if (oi >= 0 && (idx < 0 || om < m || (om == m && oi < idx))) {
      m = om;
      idx = oi;
    }
  }
  return idx;
}

// Bookkeeping of generation `gen` for one active run by the calling warp
// (lga_gen_finalize, or the persistent search's last search of the run).
// The searches' outputs are read through L2 (ld.cg): inside the persistent
// search kernel they were written by other SMs during the same launch.
__device__ __forceinline__ void gen_finalize_run(const LgaDev& D, int gen, int run) {
  const int lane = threadIdx.x & 31;
  const int c = D.cur[run];
  double* nxt = D.pop[c ^ 1] + (size_t)run * D.P * D.dim;
  double* ne = D.pope[c ^ 1] + (size_t)run * D.P;
  const size_t o0 = (size_t)run * D.L;
  const int n = D.off + D.L;
  const int w =
      warp_first_min(n, D.best_e[run], [&](int k) { return k < D.off ? ne[1 + k] : __ldcg(&D.lse[o0 + k - D.off]); });
  if (w >= 0) {  // copy the winner before any write-back overwrites it
    if (w < D.off) {
      const double* g = nxt + (size_t)(1 + w) * D.dim;
      for (int d = lane; d < D.dim; d += 32) D.best_g[(size_t)run * D.dim + d] = g[d];
    } else {
      const double* g = D.lsg + (o0 + w - D.off) * D.dim;
      for (int d = lane; d < D.dim; d += 32) D.best_g[(size_t)run * D.dim + d] = __ldcg(&g[d]);
    }
    if (lane == 0) D.best_e[run] = w < D.off ? ne[1 + w] : __ldcg(&D.lse[o0 + w - D.off]);
  }
  __syncwarp();
  long long it = 0;
  for (int r = lane; r < D.L; r += 32) it += __ldcg(&D.lsit[o0 + r]) + 1;
  for (int q = lane; q < D.L * D.dim; q += 32) {
    const int r = q / D.dim, d = q % D.dim;
    nxt[(size_t)__ldcg(&D.lstarget[o0 + r]) * D.dim + d] = __ldcg(&D.lsg[(o0 + r) * D.dim + d]);
  }
  const int k0 = D.nrec[run];
  for (int r = lane; r < D.L; r += 32) {
    const double e = __ldcg(&D.lse[o0 + r]);
    ne[__ldcg(&D.lstarget[o0 + r])] = e;
    if (k0 + r < D.maxrec) {
      mdr_ls_record rec;
      rec.best_energy = e;
      rec.iterations = __ldcg(&D.lsit[o0 + r]);
      rec.converged = __ldcg(&D.lscv[o0 + r]);
      D.recs[(size_t)run * D.maxrec + k0 + r] = rec;
    }
  }
#pragma unroll
  for (int off = 16; off >= 1; off >>= 1) it += __shfl_xor_sync(kFull, it, off);
  if (lane == 0) {
    const long long evals = D.evals[run] + D.off + it;
    D.nrec[run] = k0 + D.L;
    D.evals[run] = evals;
    D.cur[run] = c ^ 1;
    D.active[run] = (gen + 1 < D.gens) && __ldcg(&D.status[run]) == MDR_OK && budget_ok(D, evals);
  }
}

}  // namespace mdr
