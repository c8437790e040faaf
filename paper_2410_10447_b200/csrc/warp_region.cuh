// warp_region.cuh — per-search shared-memory layout of the warp-per-pose
// kernels (dock.cu) and the multi-warp Lamarckian search (ls_multi.cu).
#pragma once

#include "mdr_device.cuh"

namespace mdr {

// Register-allocation hint for the warp-per-pose search kernels (at most 16
// warps per CTA).  Without it ptxas gives the chunked-site variant 100
// registers and a 2-site-deep schedule (117 M evals/s on C3); with it, 128
// registers and the latency hidden (150 M).  The lane-per-atom variant is
// unaffected (126 -> 128 registers, same speed).
#ifndef MDR_LS_LB
#define MDR_LS_LB 1
#endif
#ifndef MDR_LS_MAXT
#define MDR_LS_MAXT 512  // threads per CTA the register allocation is sized for
#endif
#if MDR_LS_LB > 0
#define MDR_LS_BOUNDS __launch_bounds__(MDR_LS_MAXT, MDR_LS_LB)
#else
#define MDR_LS_BOUNDS
#endif

// Per-warp shared-memory region: scratch | genotype | best genotype | angle
// trig table | [exact-torsion torques] | [chunked: positions, chunk sums].
constexpr int kWarpRegion = kWarpScratchBytes + 2 * kMaxDim * 8 + kMaxDim * 16 + 16 + (MDR_PHASE_PROF ? 128 : 0);

struct WarpCtx {
  WarpScratch ws;
  double* g;
  double* best;
};

__host__ __device__ inline size_t warp_region_bytes(const LigandView& L) {
  const int nch = L.n_chunks > L.ls_n_chunks ? L.n_chunks : L.ls_n_chunks;
  return (size_t)kWarpRegion + (L.exact_torsion ? (size_t)16 * L.n_atoms : 0) +
         (nch > 1 ? (size_t)32 * L.n_atoms * (1 + nch) : 0);
}

__device__ __forceinline__ WarpCtx warp_region(unsigned char* base, int warp, const LigandView& L) {
  unsigned char* p = base + (size_t)warp * warp_region_bytes(L);
  WarpCtx w;
  w.ws.tile = reinterpret_cast<__half*>(p);
  w.ws.rec = reinterpret_cast<float*>(p + 2 * 256 * 2);
  w.g = reinterpret_cast<double*>(p + kWarpScratchBytes);
  w.best = w.g + kMaxDim;
  w.ws.trig = reinterpret_cast<double2*>(w.best + kMaxDim);
  w.ws.ctl = reinterpret_cast<int*>(w.ws.trig + kMaxDim);
  w.ws.bar = 0;
  w.ws.prof = MDR_PHASE_PROF ? reinterpret_cast<long long*>(w.ws.ctl + 4) : nullptr;
  unsigned char* q = p + kWarpRegion;
  w.ws.tq = L.exact_torsion ? reinterpret_cast<float4*>(q) : nullptr;
  if (L.exact_torsion) q += (size_t)16 * L.n_atoms;
  const bool ch = L.n_chunks > 1 || L.ls_n_chunks > 1;
  w.ws.wpos = ch ? reinterpret_cast<double4*>(q) : nullptr;
  w.ws.part = ch ? reinterpret_cast<double4*>(q) + L.n_atoms : nullptr;
  return w;
}


}  // namespace mdr
