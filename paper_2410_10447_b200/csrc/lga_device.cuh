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

}  // namespace mdr
