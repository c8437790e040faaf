// cluster.cu — RMSD clustering of docked poses.
//
// K6a pose_coords_kernel : genotype -> world atom coordinates, warp per pose,
//                          FP64 in the reference's operation order
//                          (evaluate_atoms' transform, docking.cpp:101-106)
// K6b cluster_kernel     : AutoDock's greedy clustering, one CTA per segment
//                          (a docking's runs): poses ranked by (energy,
//                          index); in that order each pose joins the first
//                          cluster whose seed is within rmsd < tol, else it
//                          seeds a new one.  The RMSDs of one pose against
//                          all current seeds are computed in parallel (thread
//                          per seed, atoms summed in index order, as the
//                          oracle does), the first hit is a block min-reduce.
#include <cuda_runtime.h>

#include "dock_launch.h"
#include "mdr_device.cuh"

namespace mdr {

// Warp per pose; pose i docks ligand pose_lig[i] (nullptr: ligand 0) with
// genotype stride gstride; coordinates at xyz + i * xstride.
__global__ void pose_coords_kernel(const LigandView* __restrict__ Ls, const int* __restrict__ pose_lig,
                                   const double* __restrict__ genos, int gstride, int n, long long xstride,
                                   double* __restrict__ xyz) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int item = blockIdx.x * (blockDim.x >> 5) + warp;
  if (item >= n) return;
  const LigandView L = Ls[pose_lig ? pose_lig[item] : 0];
  SmemLigand S;  // read the ligand in place (global, L1-cached)
  S.sites = L.sites;
  S.atoms = L.atoms;
  S.tors = L.tors;
  S.taxes = L.taxes;
  S.sites_f = L.sites_f;
  S.sites_f2 = L.sites_f2;
  S.n_atoms = L.n_atoms;
  S.n_sites = L.n_sites;
  S.n_rot = L.n_rot;
  const double* g = genos + (size_t)item * gstride;
  const Frame f = build_frame(g[3], g[4], g[5]);
  const d3 tr = {g[0], g[1], g[2]};
  double* out = xyz + (size_t)item * xstride;
  for (int i = lane; i < L.n_atoms; i += 32) {
    const d3 w = atom_world(S, g, f.R, tr, i);
    out[3 * i] = w.x;
    out[3 * i + 1] = w.y;
    out[3 * i + 2] = w.z;
  }
}

__device__ __forceinline__ double rmsd_xyz(const double* a, const double* b, int na) {
  double s = 0.0;
  for (int i = 0; i < 3 * na; ++i) {
    const double d = a[i] - b[i];
    s += d * d;
  }
  return sqrt(s / na);
}

// seg_off[s] .. seg_off[s + 1]: the poses of segment s (cluster ids are
// per segment), each of seg_na[s] atoms (nullptr: na) at xyz + pose *
// xstride.  order / seeds: scratch of one int per pose.
__global__ void cluster_kernel(const double* __restrict__ xyz, long long xstride, const double* __restrict__ energy,
                               const int* __restrict__ seg_off, const int* __restrict__ seg_na, int na_all,
                               double tol, int* __restrict__ cluster_of, double* __restrict__ rmsd,
                               int* __restrict__ n_clusters, int* __restrict__ order, int* __restrict__ seeds) {
  const int seg = blockIdx.x;
  const int lo = seg_off[seg], n = seg_off[seg + 1] - lo;
  const int na = seg_na ? seg_na[seg] : na_all;
  int* ord = order + lo;
  int* sd = seeds + lo;
  // rank of each pose in the stable (energy, index) order
  for (int p = threadIdx.x; p < n; p += blockDim.x) {
    const double e = energy[lo + p];
    int r = 0;
    for (int q = 0; q < n; ++q) {
      const double eq = energy[lo + q];
      r += (eq < e) || (eq == e && q < p);
    }
    ord[r] = p;
  }
  __shared__ int s_hit, s_nc;
  if (threadIdx.x == 0) s_nc = 0;
  __syncthreads();
  for (int q = 0; q < n; ++q) {
    const int p = ord[q];
    const double* xp = xyz + (size_t)(lo + p) * xstride;
    if (threadIdx.x == 0) s_hit = 0x7fffffff;
    __syncthreads();
    const int nc = s_nc;
    for (int k = threadIdx.x; k < nc; k += blockDim.x) {
      const double d = rmsd_xyz(xp, xyz + (size_t)(lo + sd[k]) * xstride, na);
      if (d < tol) atomicMin(&s_hit, k);
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      int c = s_hit;
      double r = 0.0;
      if (c == 0x7fffffff) {
        c = nc;
        sd[nc] = p;
        s_nc = nc + 1;
      } else {
        r = rmsd_xyz(xp, xyz + (size_t)(lo + sd[c]) * xstride, na);
      }
      cluster_of[lo + p] = c;
      rmsd[lo + p] = r;
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) n_clusters[seg] = s_nc;
}

cudaError_t launch_pose_coords(const LigandView* Ls, const int* pose_lig, const double* genos, int gstride, int n,
                               long long xstride, double* xyz, cudaStream_t s) {
  if (n <= 0) return cudaSuccess;
  pose_coords_kernel<<<(n + 3) / 4, 128, 0, s>>>(Ls, pose_lig, genos, gstride, n, xstride, xyz);
  return cudaGetLastError();
}

cudaError_t launch_cluster(const double* xyz, long long xstride, const double* energy, const int* seg_off,
                           const int* seg_na, int n_seg, int na, double tol, int* cluster_of, double* rmsd,
                           int* n_clusters, int* order, int* seeds, cudaStream_t s) {
  if (n_seg <= 0) return cudaSuccess;
  cluster_kernel<<<n_seg, 128, 0, s>>>(xyz, xstride, energy, seg_off, seg_na, na, tol, cluster_of, rmsd, n_clusters,
                                       order, seeds);
  return cudaGetLastError();
}

}  // namespace mdr
