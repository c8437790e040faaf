// grid.cu — grid-map scoring mode (north_star subsystem 1):
// one CTA of `partition` threads evaluates one pose, AutoDock-GPU style.
//
// Per evaluation (three CTA barriers):
//   A  threads 3..dim-1 take sincos of their own genotype angle (FP32,
//      widened) into a double-buffered table                      -> S1
//   B  thread per atom: rotate_axis (docking.cpp:57-60), R*local + t
//      (build_frame docking.cpp:78-91, FP64), trilinear interpolation of the
//      atom's combined map w*type + q*elec + |q|*desolv (FP32, L1/L2-resident
//      maps), force and torque partials                         -> S2
//   C  intramolecular pairs (torsioned atom x partner chunk, FP32, partners
//      broadcast from shared memory) + the block reduction of the seven
//      partial sums {E, F, tau} (the paper's operation: shuffle trees, or the
//      ones-matrix MMA in f16 / tf32 hi-lo), one record per warp -> S3
//   D  every thread sums the warp records in warp order (energy); thread d
//      forms gradient component d: translation, Euler axis . tau, or the
//      exact torque of torsion group d-6 about its axis (score_reference
//      docking.cpp:244-268 semantics, plus the intramolecular forces); the
//      same thread then takes the ADADELTA step of dimension d, so no
//      barrier separates the gradient from the update.
// The local search, the LGA phases and the polish reuse the analytic
// driver's bookkeeping kernels (lga_device.cuh, dock.cu).
#include <cuda_runtime.h>

#ifndef MDR_GRID_NO_GATHER
#define MDR_GRID_NO_GATHER 0
#endif

#include "dock_launch.h"
#include "lga_device.cuh"
#include "mdr_device.cuh"
#include "crmath.cuh"

// Phase A trig in FP32: C4 43.7 -> 55.3 M evals/s (the other threads wait
// at S1 for it), device-vs-oracle error 1.0e-6 -> 1.4e-6 (energy), 1.6e-6 ->
// 1.1e-6 (gradient) (profiles/r1_grid_probe.json; tolerances 1e-5 / 2e-5).
#ifndef MDR_GRID_F32_TRIG
#define MDR_GRID_F32_TRIG 1
#endif
#ifndef MDR_GRID_UNROLL
#define MDR_GRID_UNROLL 4  // partners in flight per thread in phase C
#endif

namespace mdr {

// ------------------------------------------------------------ smem layout
__host__ __device__ inline size_t al16_(size_t b) { return (b + 15) & ~size_t(15); }

// Method code of the strict FP64 grid path (the context's pair precision
// MDR_PAIR_FP64): the oracle's double arithmetic in the oracle's order,
// correctly rounded trig (csrc/crmath.cuh, oracle/crmath.h).
constexpr int kGridStrict = 3;

struct GridSmem {
  double4* atoms;   // na: local x, y, z, weight
  int* tors;        // na
  int* type;        // na
  float4* chem;     // na: 1.25 radius, sqrt eps, q, energy share (1 rigid, 1/2 torsioned)
  float* keq;       // na: k_e q (the unit side of the Coulomb term)
  double* taxes;    // 3 * nr
  int* grp_off;     // nr + 1
  int* grp_atoms;   // nta
  double2* trig[2]; // (3 + nr) x (sin, cos), double buffered
  float4* pos;      // na: R * local (lever arm), FP32; w = torsion group (int bits)
  float4* force;    // na: grid force
  float4* fintra;   // nta * C: intramolecular force partials
  float* wpart;     // W x 8
  double* g;        // dim
  double* best;     // dim
  unsigned char* scratch;  // W x kWarpScratchBytes (MMA staging)
  int na, nr, nta, C, W;
  // strict FP64 mode (METHOD == kGridStrict) only:
  double4* xr;          // na: lever arm r_i = R local_i (x, y, z)
  double4* xf;          // na: grid force F_i (x, y, z) and energy term (w)
  double4* xfi;         // na: intramolecular force Fi_i
  double* xep;          // na (na - 1) / 2: pair energies, row i holds pairs (i, j > i)
  double* xtot;         // 8: energy, sum F (3), sum r x F (3)
  const double4* chem64;  // na: radius, epsilon, charge (double, as the oracle)
  double elec_scale;
};

// Strict FP64 grid mode: the extra shared memory (after the MMA scratch).
__host__ __device__ inline size_t grid_strict_bytes(int na) {
  return al16_(sizeof(double4) * (size_t)na) * 3 + al16_(sizeof(double) * ((size_t)na * (na - 1) / 2 + 1)) +
         al16_(sizeof(double) * 8);
}

__host__ __device__ inline size_t al16(size_t b) { return (b + 15) & ~size_t(15); }

__host__ __device__ inline int grid_chunks(int nta, int T) {
  // partner chunks per torsioned atom: spread the pair loop over the CTA
  if (nta <= 0) return 1;
  const int c = T / nta;
  return c < 1 ? 1 : (c > 32 ? 32 : c);
}

__host__ __device__ inline size_t grid_smem_bytes(int na, int nr, int nta, int T) {
  const int W = T / 32, C = grid_chunks(nta, T), dim = 6 + nr;
  size_t b = 0;
  b += al16(sizeof(double4) * na);
  b += al16(sizeof(int) * na) * 2;
  b += al16(sizeof(float4) * na);
  b += al16(sizeof(float) * na);
  b += al16(sizeof(double) * 3 * (nr > 0 ? nr : 1));
  b += al16(sizeof(int) * (nr + 1));
  b += al16(sizeof(int) * (nta > 0 ? nta : 1));
  b += al16(sizeof(double2) * (3 + nr)) * 2;
  b += al16(sizeof(float4) * na) * 2;
  b += al16(sizeof(float4) * (size_t)(nta > 0 ? nta : 1) * C);
  b += al16(sizeof(float) * 8 * W);
  b += al16(sizeof(double) * dim) * 2;
  b += (size_t)kWarpScratchBytes * W;
  return b;
}

__device__ GridSmem grid_load(const LigandView& L, const FlexView& F, unsigned char* base, bool strict = false) {
  GridSmem S;
  S.na = L.n_atoms;
  S.nr = L.n_rot;
  S.nta = F.n_tors_atoms;
  S.W = blockDim.x >> 5;
  S.C = grid_chunks(S.nta, blockDim.x);
  const int na = S.na, nr = S.nr, nta = S.nta, dim = 6 + nr;
  unsigned char* p = base;
  auto take = [&](size_t bytes) {
    unsigned char* r = p;
    p += al16(bytes);
    return r;
  };
  S.atoms = reinterpret_cast<double4*>(take(sizeof(double4) * na));
  S.tors = reinterpret_cast<int*>(take(sizeof(int) * na));
  S.type = reinterpret_cast<int*>(take(sizeof(int) * na));
  S.chem = reinterpret_cast<float4*>(take(sizeof(float4) * na));
  S.keq = reinterpret_cast<float*>(take(sizeof(float) * na));
  S.taxes = reinterpret_cast<double*>(take(sizeof(double) * 3 * (nr > 0 ? nr : 1)));
  S.grp_off = reinterpret_cast<int*>(take(sizeof(int) * (nr + 1)));
  S.grp_atoms = reinterpret_cast<int*>(take(sizeof(int) * (nta > 0 ? nta : 1)));
  S.trig[0] = reinterpret_cast<double2*>(take(sizeof(double2) * (3 + nr)));
  S.trig[1] = reinterpret_cast<double2*>(take(sizeof(double2) * (3 + nr)));
  S.pos = reinterpret_cast<float4*>(take(sizeof(float4) * na));
  S.force = reinterpret_cast<float4*>(take(sizeof(float4) * na));
  S.fintra = reinterpret_cast<float4*>(take(sizeof(float4) * (size_t)(nta > 0 ? nta : 1) * S.C));
  S.wpart = reinterpret_cast<float*>(take(sizeof(float) * 8 * S.W));
  S.g = reinterpret_cast<double*>(take(sizeof(double) * dim));
  S.best = reinterpret_cast<double*>(take(sizeof(double) * dim));
  S.scratch = p;
  S.xr = S.xf = S.xfi = nullptr;
  S.xep = S.xtot = nullptr;
  S.chem64 = F.chem64;
  S.elec_scale = F.elec_scale;
  if (strict) {
    p += (size_t)kWarpScratchBytes * S.W;
    S.xr = reinterpret_cast<double4*>(take(sizeof(double4) * na));
    S.xf = reinterpret_cast<double4*>(take(sizeof(double4) * na));
    S.xfi = reinterpret_cast<double4*>(take(sizeof(double4) * na));
    S.xep = reinterpret_cast<double*>(take(sizeof(double) * ((size_t)na * (na - 1) / 2 + 1)));
    S.xtot = reinterpret_cast<double*>(take(sizeof(double) * 8));
  }
  for (int i = threadIdx.x; i < na; i += blockDim.x) {
    S.atoms[i] = L.atoms[i];
    S.tors[i] = L.tors[i];
    S.type[i] = F.type[i];
    // phase C's per-partner constants: radius pre-scaled by 1.25 (so
    // d0'^2 = 1.5625 d0^2), the pair-energy share of this partner in w
    const float4 ch = F.chem[i];
    S.chem[i] = make_float4(1.25f * ch.x, ch.y, ch.z, L.tors[i] < 0 ? 1.0f : 0.5f);
    S.keq[i] = ch.w;
  }
  for (int i = threadIdx.x; i < 3 * nr; i += blockDim.x) S.taxes[i] = L.taxes[i];
  for (int i = threadIdx.x; i <= nr; i += blockDim.x) S.grp_off[i] = F.grp_off[i];
  for (int i = threadIdx.x; i < nta; i += blockDim.x) S.grp_atoms[i] = F.grp_atoms[i];
  return S;
}

// ------------------------------------------------------- interpolation
// Energy and force of one atom at world point p (mdr.h grid formulas): the
// combined map c = w*type + q*elec + |q|*desolv is interpolated once.
__device__ __forceinline__ float grid_atom(const GridView& G, int type, float w, float q, double px, double py,
                                           double pz, float3& F) {
  const double gc[3] = {(px - G.ox) * G.inv_h, (py - G.oy) * G.inv_h, (pz - G.oz) * G.inv_h};
  const int n[3] = {G.nx, G.ny, G.nz};
  int i0[3];
  float f[3], off[3];
  bool in[3];
#pragma unroll
  for (int a = 0; a < 3; ++a) {
    const double hi = (double)(n[a] - 1);
    const double c = fmin(fmax(gc[a], 0.0), hi);
    int i = (int)floor(c);
    i = i > n[a] - 2 ? n[a] - 2 : i;
    i0[a] = i;
    f[a] = (float)(c - (double)i);
    in[a] = gc[a] >= 0.0 && gc[a] <= hi;
    off[a] = (float)(G.h * (gc[a] - c));
  }
  const long long nx = G.nx, nxy = (long long)G.nx * G.ny;
  const long long o = (long long)i0[2] * nxy + (long long)i0[1] * nx + i0[0];
  const float* mt = G.maps + (long long)type * G.stride + o;
  const float* me = G.maps + (long long)G.n_types * G.stride + o;
  const float* md = me + G.stride;
  const float aq = fabsf(q);
  const long long co[8] = {0, 1, nx, nx + 1, nxy, nxy + 1, nxy + nx, nxy + nx + 1};
  float c[8];
#if MDR_GRID_NO_GATHER
  // timing probe only (wrong results): the map values replaced by a function
  // of the corner offset, to bound what any map layout / staging could gain
#pragma unroll
  for (int k = 0; k < 8; ++k) c[k] = fmaf(w, (float)(o & 7) * 0.01f, q * 0.001f * (float)k + aq * 0.0001f);
  (void)mt;
  (void)me;
  (void)md;
  (void)co;
#else
#pragma unroll
  for (int k = 0; k < 8; ++k)
    c[k] = fmaf(w, __ldg(mt + co[k]), fmaf(q, __ldg(me + co[k]), aq * __ldg(md + co[k])));
#endif
  // x pass (k = dz*4 + dy*2 + dx), y pass, z pass
  float gx[4], vx[4];
#pragma unroll
  for (int r = 0; r < 4; ++r) {
    gx[r] = c[2 * r + 1] - c[2 * r];
    vx[r] = fmaf(f[0], gx[r], c[2 * r]);
  }
  float vy[2], gyy[2], gxy[2];
#pragma unroll
  for (int z = 0; z < 2; ++z) {
    gyy[z] = vx[2 * z + 1] - vx[2 * z];
    vy[z] = fmaf(f[1], gyy[z], vx[2 * z]);
    gxy[z] = fmaf(f[1], gx[2 * z + 1] - gx[2 * z], gx[2 * z]);
  }
  const float v = fmaf(f[2], vy[1] - vy[0], vy[0]);
  const float dfx = fmaf(f[2], gxy[1] - gxy[0], gxy[0]);
  const float dfy = fmaf(f[2], gyy[1] - gyy[0], gyy[0]);
  const float dfz = vy[1] - vy[0];
  const float ih = (float)G.inv_h, k2 = (float)(2.0 * MDR_GRID_OUTSIDE_K);
  F.x = fmaf(k2, off[0], in[0] ? dfx * ih : 0.f);
  F.y = fmaf(k2, off[1], in[1] ? dfy * ih : 0.f);
  F.z = fmaf(k2, off[2], in[2] ? dfz * ih : 0.f);
  const float pen = fmaf(off[0], off[0], fmaf(off[1], off[1], off[2] * off[2]));
  return fmaf((float)MDR_GRID_OUTSIDE_K, pen, v);
}

__device__ __forceinline__ float3 cross3f(float3 a, float3 b) {
  return make_float3(a.y * b.z - a.z * b.y, a.z * b.x - a.x * b.z, a.x * b.y - a.y * b.x);
}

// ------------------------------------------------- warp-level 7-reduction
// rec = {E, Fx, Fy, Fz, tx, ty, tz}; returns the warp totals, valid in lane
// c for component c (lanes >= 7 undefined).
template <int METHOD>
__device__ __forceinline__ float warp_reduce7(const float (&rec)[7], unsigned char* scratch, int lane) {
  if (METHOD == MDR_METHOD_BASELINE) {
    float mine = 0.f;
#pragma unroll
    for (int c = 0; c < 7; ++c) {
      const float s = warp_tree(rec[c]);
      if (lane == c) mine = s;
    }
    return mine;
  } else if (METHOD == MDR_METHOD_TCU) {
    // the paper's f16 ones-matrix contraction (Single accumulation): the
    // warp's 32 records are one 64-vector chunk with the upper half zero
    __half* tile = reinterpret_cast<__half*>(scratch);
    float vg[4] = {0.f, 0.f, 0.f, 0.f}, vt[4] = {0.f, 0.f, 0.f, 0.f};
    const float4 z = make_float4(0.f, 0.f, 0.f, 0.f);
    tcu_tile(vg, make_float4(rec[1], rec[2], rec[3], rec[0]), z, tile, false, lane);
    tcu_tile(vt, make_float4(rec[4], rec[5], rec[6], 0.f), z, tile + 256, false, lane);
    const float wg = tcu_q_step(vg, false, lane);  // W_c in lane 4c: gx, gy, gz, E
    const float wt = tcu_q_step(vt, false, lane);  // tx, ty, tz, 0
    const int src_g = lane == 0 ? 12 : 4 * (lane - 1);
    const float a = __shfl_sync(kFull, wg, lane < 4 ? src_g : 0);
    const float b = __shfl_sync(kFull, wt, lane >= 4 && lane < 7 ? 4 * (lane - 4) : 0);
    return lane < 4 ? a : b;
  } else {  // TcuSplit: tf32 hi/lo against ones, fp32 accumulation
    float acc[4] = {0.f, 0.f, 0.f, 0.f};
    split_group(acc, rec, reinterpret_cast<float*>(scratch + 2 * 256 * 2), lane);
    const float tot = acc[0] + acc[2];  // component lane >> 2, in lanes 4c
    return __shfl_sync(kFull, tot, lane < 7 ? 4 * lane : 0);
  }
}

// ---------------------------------------------------------- evaluation
struct GridEval {
  float e;   // total energy (all threads)
  float gd;  // gradient component threadIdx.x (threads < dim)
};
struct GridEvalD {  // the strict FP64 path's (double energy and gradient, as the oracle)
  double e;
  double gd;
};
template <int METHOD>
struct GridEvalT {
  using type = GridEval;
};
template <>
struct GridEvalT<kGridStrict> {
  using type = GridEvalD;
};

// Trilinear sample of the combined map in double, operation for operation
// the oracle's grid_sample (oracle/mdr_oracle.c): IEEE divisions by the
// spacing, no contraction (the library is built with --fmad=false).
__device__ __forceinline__ double grid_sample_f64(const GridView& G, int type, double w, double q, const double p[3],
                                                  double dvdp[3], double off[3]) {
  const int n[3] = {G.nx, G.ny, G.nz};
  const double org[3] = {G.ox, G.oy, G.oz};
  int i0[3];
  double f[3];
  bool inside[3];
#pragma unroll
  for (int a = 0; a < 3; ++a) {
    const double gc = (p[a] - org[a]) / G.h;
    double gcc = gc < 0.0 ? 0.0 : gc;
    gcc = gcc > (double)(n[a] - 1) ? (double)(n[a] - 1) : gcc;
    int i = (int)floor(gcc);
    if (i > n[a] - 2) i = n[a] - 2;
    i0[a] = i;
    f[a] = gcc - i;
    inside[a] = gc >= 0.0 && gc <= (double)(n[a] - 1);
    off[a] = G.h * (gc - gcc);
  }
  const size_t stride = (size_t)G.stride;
  const float* mt = G.maps + (size_t)type * stride;
  const float* me = G.maps + (size_t)G.n_types * stride;
  const float* md = me + stride;
  const double aq = fabs(q);
  double c[2][2][2];
#pragma unroll
  for (int dz = 0; dz < 2; ++dz)
#pragma unroll
    for (int dy = 0; dy < 2; ++dy)
#pragma unroll
      for (int dx = 0; dx < 2; ++dx) {
        const size_t o = ((size_t)(i0[2] + dz) * G.ny + (i0[1] + dy)) * G.nx + (i0[0] + dx);
        c[dz][dy][dx] = w * (double)__ldg(mt + o) + q * (double)__ldg(me + o) + aq * (double)__ldg(md + o);
      }
  double vx[2][2], gx[2][2];
#pragma unroll
  for (int dz = 0; dz < 2; ++dz)
#pragma unroll
    for (int dy = 0; dy < 2; ++dy) {
      gx[dz][dy] = c[dz][dy][1] - c[dz][dy][0];
      vx[dz][dy] = c[dz][dy][0] + f[0] * gx[dz][dy];
    }
  double vy[2], gxy[2], gyy[2];
#pragma unroll
  for (int dz = 0; dz < 2; ++dz) {
    gyy[dz] = vx[dz][1] - vx[dz][0];
    vy[dz] = vx[dz][0] + f[1] * gyy[dz];
    gxy[dz] = gx[dz][0] + f[1] * (gx[dz][1] - gx[dz][0]);
  }
  const double v = vy[0] + f[2] * (vy[1] - vy[0]);
  const double dfx = gxy[0] + f[2] * (gxy[1] - gxy[0]);
  const double dfy = gyy[0] + f[2] * (gyy[1] - gyy[0]);
  const double dfz = vy[1] - vy[0];
  dvdp[0] = inside[0] ? dfx / G.h : 0.0;
  dvdp[1] = inside[1] ? dfy / G.h : 0.0;
  dvdp[2] = inside[2] ? dfz / G.h : 0.0;
  return v;
}

// One pair term (i < j, different torsion groups) of the oracle's
// orc_grid_score: sc and the energy term, in its operation order.
__device__ __forceinline__ void strict_pair(const GridSmem& S, int i, int j, double& sc, double& e, d3& d) {
  const double4 ri = S.xr[i], rj = S.xr[j];
  d = {ri.x - rj.x, ri.y - rj.y, ri.z - rj.z};
  const double4 ci = S.chem64[i], cj = S.chem64[j];
  const double d0 = ci.x + cj.x;
  const double c2 = 0.5625 * d0 * d0;
  const double u = dot(d, d) + c2;
  const double rho2 = (d0 * d0 + c2) / u;
  const double rho6 = rho2 * rho2 * rho2;
  const double rho12 = rho6 * rho6;
  const double eps = sqrt(ci.y * cj.y);
  const double qq = S.elec_scale * ci.z * cj.z;
  e = eps * (rho12 - 2.0 * rho6) + qq / u;
  sc = -12.0 * eps * (rho12 - rho6) / u - 2.0 * qq / (u * u);
}

// orc_grid_score (oracle/mdr_oracle.c) on the device, bit for bit: double
// arithmetic in the oracle's order, correctly rounded trig, the oracle's
// sequential sums (over atoms, over pairs in (i, j) order) run by single
// threads.  A parity mode: per-run comparisons of grid dockings against the
// oracle, at a fraction of the FP32 path's speed.
__device__ __noinline__ GridEvalD grid_eval_strict(const GridSmem& S, const GridView& G, int buf, bool intra,
                                                  bool bad_in, bool& bad_out) {
  const int tid = threadIdx.x, T = blockDim.x;
  const int na = S.na, nr = S.nr, dim = 6 + nr;
  double2* trig = S.trig[buf];
  if (tid >= 3 && tid < dim) {
    double s, c;
    cr::sincos(S.g[tid], &s, &c);
    trig[tid - 3] = make_double2(s, c);
  }
  bad_out = __syncthreads_or(bad_in) != 0;
  GridEvalD out;
  out.e = 0.0;
  out.gd = 0.0;
  if (bad_out) return out;
  const double2 t1 = trig[0], t2 = trig[1], t3 = trig[2];
  const Frame fr = frame_from_trig(t1.x, t1.y, t2.x, t2.y, t3.x, t3.y);
  const d3 t = {S.g[0], S.g[1], S.g[2]};
  for (int i = tid; i < na; i += T) {
    const double4 at = S.atoms[i];
    d3 local = {at.x, at.y, at.z};
    const int k = S.tors[i];
    if (k >= 0) {  // rotate_axis docking.cpp:57-60 (oracle: add3(add3(c v, s a x v), ((1 - c) a.v) a))
      const d3 ax = {S.taxes[3 * k], S.taxes[3 * k + 1], S.taxes[3 * k + 2]};
      const double2 sc = trig[3 + k];
      local = (sc.y * local + sc.x * cross(ax, local)) + ((1.0 - sc.y) * dot(ax, local)) * ax;
    }
    const d3 r = mv(fr.R, local);
    const d3 wp = t + r;
    const double p[3] = {wp.x, wp.y, wp.z};
    double dv[3], off[3];
    double e = grid_sample_f64(G, S.type[i], at.w, S.chem64[i].z, p, dv, off);
    double F[3];
#pragma unroll
    for (int a = 0; a < 3; ++a) {
      e += MDR_GRID_OUTSIDE_K * off[a] * off[a];
      F[a] = dv[a] + 2.0 * MDR_GRID_OUTSIDE_K * off[a];
    }
    S.xr[i] = make_double4(r.x, r.y, r.z, 0.0);
    S.xf[i] = make_double4(F[0], F[1], F[2], e);
  }
  __syncthreads();
  if (intra) {
    // atom a's intramolecular force in the oracle's update order: the pairs
    // (i, a), i < a (subtracted), then (a, j), j > a (added); pair energies
    // of row a stored for the sequential sum
    for (int a = tid; a < na; a += T) {
      d3 fi = {0.0, 0.0, 0.0};
      const int ga = S.tors[a];
      for (int i = 0; i < a; ++i) {
        if (S.tors[i] == ga) continue;
        double sc, e;
        d3 d;
        strict_pair(S, i, a, sc, e, d);
        fi = fi - sc * d;
      }
      double* row = S.xep + (size_t)a * (2 * na - a - 1) / 2;
      for (int j = a + 1; j < na; ++j) {
        if (S.tors[j] == ga) continue;
        double sc, e;
        d3 d;
        strict_pair(S, a, j, sc, e, d);
        fi = fi + sc * d;
        row[j - a - 1] = e;
      }
      S.xfi[a] = make_double4(fi.x, fi.y, fi.z, 0.0);
    }
  } else {
    for (int a = tid; a < na; a += T) S.xfi[a] = make_double4(0.0, 0.0, 0.0, 0.0);
  }
  __syncthreads();
  // the oracle's sequential sums: grid terms over atoms (thread 0), pair
  // energies over (i, j) (thread 32, a second warp)
  if (tid == 0) {
    double e_inter = 0.0;
    d3 gs = {0.0, 0.0, 0.0}, ts = {0.0, 0.0, 0.0};
    for (int i = 0; i < na; ++i) {
      const double4 f4 = S.xf[i], r4 = S.xr[i];
      const d3 F = {f4.x, f4.y, f4.z};
      e_inter += f4.w;
      gs = gs + F;
      ts = ts + cross(d3{r4.x, r4.y, r4.z}, F);
    }
    S.xtot[0] = e_inter;
    S.xtot[1] = gs.x;
    S.xtot[2] = gs.y;
    S.xtot[3] = gs.z;
    S.xtot[4] = ts.x;
    S.xtot[5] = ts.y;
    S.xtot[6] = ts.z;
  }
  if (tid == (T > 32 ? 32 : 0)) {
    double e_intra = 0.0;
    if (intra)
      for (int i = 0; i < na; ++i) {
        const double* row = S.xep + (size_t)i * (2 * na - i - 1) / 2;
        const int gi = S.tors[i];
        for (int j = i + 1; j < na; ++j)
          if (S.tors[j] != gi) e_intra += row[j - i - 1];
      }
    S.xtot[7] = e_intra;
  }
  __syncthreads();
  out.e = S.xtot[0] + S.xtot[7];
  if (tid < dim) {
    const d3 ts = {S.xtot[4], S.xtot[5], S.xtot[6]};
    if (tid < 3) {
      out.gd = S.xtot[1 + tid];
    } else if (tid == 3) {
      out.gd = dot(d3{0.0, 0.0, 1.0}, ts);
    } else if (tid == 4) {
      out.gd = dot(fr.ax_theta, ts);
    } else if (tid == 5) {
      out.gd = dot(fr.ax_alpha, ts);
    } else {
      const int k = tid - 6;
      d3 tk = {0.0, 0.0, 0.0};
      for (int i = 0; i < na; ++i)
        if (S.tors[i] == k) {
          const double4 f4 = S.xf[i], q4 = S.xfi[i], r4 = S.xr[i];
          tk = tk + cross(d3{r4.x, r4.y, r4.z}, d3{f4.x, f4.y, f4.z} + d3{q4.x, q4.y, q4.z});
        }
      const d3 tw = mv(fr.R, d3{S.taxes[3 * k], S.taxes[3 * k + 1], S.taxes[3 * k + 2]});
      out.gd = dot(tw, tk);
    }
  }
  return out;
}

template <int METHOD>
__device__ __forceinline__ GridEval grid_eval_fp32(const GridSmem& S, const GridView& G, int buf, bool intra, bool bad_in, bool& bad_out) {
  const int tid = threadIdx.x, T = blockDim.x, lane = tid & 31, warp = tid >> 5;
  const int nr = S.nr, dim = 6 + nr;
  // A: angles owned by threads 3..dim-1
  double2* trig = S.trig[buf];
  if (tid >= 3 && tid < dim) {
#if MDR_GRID_F32_TRIG
    float s, c;  // FP32 trig (grid mode is tolerance parity; shortens the barrier wait)
    sincosf((float)S.g[tid], &s, &c);
    trig[tid - 3] = make_double2((double)s, (double)c);
#else
    double s, c;
    sincos(S.g[tid], &s, &c);
    trig[tid - 3] = make_double2(s, c);
#endif
  }
  bad_out = __syncthreads_or(bad_in) != 0;  // S1
  GridEval out;
  out.e = 0.f;
  out.gd = 0.f;
  if (bad_out) return out;
  // B: frame (reference product order Rz(phi) Ry(theta) Rz(alpha)), atoms
  const double2 t1 = trig[0], t2 = trig[1], t3 = trig[2];
  const m3 rz1 = {{t1.y, -t1.x, 0.0, t1.x, t1.y, 0.0, 0.0, 0.0, 1.0}};
  const m3 ry2 = {{t2.y, 0.0, t2.x, 0.0, 1.0, 0.0, -t2.x, 0.0, t2.y}};
  const m3 rz3 = {{t3.y, -t3.x, 0.0, t3.x, t3.y, 0.0, 0.0, 0.0, 1.0}};
  const m3 ab = mm(rz1, ry2);
  const m3 R = mm(ab, rz3);
  const double tx = S.g[0], ty = S.g[1], tz = S.g[2];
  float rec[7] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
  for (int i = tid; i < S.na; i += T) {
    const double4 at = S.atoms[i];
    d3 local = {at.x, at.y, at.z};
    const int k = S.tors[i];
    if (k >= 0) {  // rotate_axis docking.cpp:57-60
      const d3 ax = {S.taxes[3 * k], S.taxes[3 * k + 1], S.taxes[3 * k + 2]};
      const double2 sc = trig[3 + k];
      local = (sc.y * local + sc.x * cross(ax, local)) + ((1.0 - sc.y) * dot(ax, local)) * ax;
    }
    const d3 r = mv(R, local);
    const float4 ch = S.chem[i];
    float3 F;
    const float e = grid_atom(G, S.type[i], (float)at.w, ch.z, tx + r.x, ty + r.y, tz + r.z, F);
    const float3 rf = make_float3((float)r.x, (float)r.y, (float)r.z);
    S.pos[i] = make_float4(rf.x, rf.y, rf.z, __int_as_float(k));
    S.force[i] = make_float4(F.x, F.y, F.z, 0.f);
    const float3 tq = cross3f(rf, F);
    rec[0] += e;
    rec[1] += F.x;
    rec[2] += F.y;
    rec[3] += F.z;
    rec[4] += tq.x;
    rec[5] += tq.y;
    rec[6] += tq.z;
  }
  __syncthreads();  // S2
  // C: intramolecular pairs, unit u = (torsioned atom a = grp_atoms[u / C],
  // partner chunk u % C); the pair energy is shared by both ends when both
  // atoms are torsioned (each end visits it), whole when the partner is rigid.
  if (intra) {
    // partners in flight per thread (C4, unroll 2 / 4 / 6 / 8: Baseline
    // 46.4 / 59.8 / 59.1 / 59.1 M evals/s, TcuSplit 54.4 / 54.9 / 54.8 /
    // 55.0, Tcu 43.1 / 45.5 / 45.0 / 45.5)
    constexpr int kUnroll = MDR_GRID_UNROLL;
    const int C = S.C, U = S.nta * C;
    for (int u = tid; u < U; u += T) {
      const int a = S.grp_atoms[u / C];
      const int ga = S.tors[a];
      const float4 pa = S.pos[a], ca = S.chem[a];
      const float ea12 = -12.0f * ca.y, qa = S.keq[a];
      float fx = 0.f, fy = 0.f, fz = 0.f, ee = 0.f;
      // branch-free: a same-group partner (incl. j == a) contributes with
      // weight 0 instead of a divergent `continue`; its u is offset by 1 so
      // the masked terms stay finite even for zero radii
#pragma unroll kUnroll
      for (int j = u % C; j < S.na; j += C) {
        const float4 pj = S.pos[j], cj = S.chem[j];
        const int gj = __float_as_int(pj.w);
        const float dx = pa.x - pj.x, dy = pa.y - pj.y, dz = pa.z - pj.z;
        const float d0 = ca.x + cj.x;  // 1.25 (r_a + r_j)
        const float d02 = d0 * d0;      // 1.5625 (r_a + r_j)^2
        const bool same = gj == ga;
        const float u2 = fmaf(dx, dx, fmaf(dy, dy, fmaf(dz, dz, fmaf(0.36f, d02, same ? 1.0f : 0.0f))));
        float iu;
        asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(iu) : "f"(u2));
        const float rho2 = d02 * iu;
        const float rho6 = rho2 * rho2 * rho2;
        const float rho12 = rho6 * rho6;
        const float eps = ca.y * cj.y;
        const float qi = qa * cj.z * iu;
        const float e = fmaf(eps, fmaf(-2.0f, rho6, rho12), qi);
        const float s = fmaf(ea12 * cj.y, rho12 - rho6, -2.0f * qi) * (same ? 0.0f : iu);
        ee = fmaf(same ? 0.0f : cj.w, e, ee);
        fx = fmaf(s, dx, fx);
        fy = fmaf(s, dy, fy);
        fz = fmaf(s, dz, fz);
      }
      S.fintra[u] = make_float4(fx, fy, fz, 0.f);
      rec[0] += ee;
    }
  }
  {
    const float w = warp_reduce7<METHOD>(rec, S.scratch + (size_t)warp * kWarpScratchBytes, lane);
    if (lane < 7) S.wpart[warp * 8 + lane] = w;
  }
  __syncthreads();  // S3
  // D: totals in warp order (each thread reads only the components it
  // needs: the energy, plus force / torque for gradient entries 0..5)
  auto total = [&](int c) {
    float s = 0.f;
    for (int w = 0; w < S.W; ++w) s += S.wpart[w * 8 + c];
    return s;
  };
  out.e = total(0);
  if (tid < dim) {
    if (tid < 3) {
      out.gd = total(1 + tid);
    } else if (tid < 6) {
      const float sums[7] = {0.f, 0.f, 0.f, 0.f, total(4), total(5), total(6)};
      d3 ax;
      if (tid == 3)
        ax = {0.0, 0.0, 1.0};
      else if (tid == 4)
        ax = mv(rz1, d3{0.0, 1.0, 0.0});
      else
        ax = mv(ab, d3{0.0, 0.0, 1.0});
      out.gd = (float)ax.x * sums[4] + (float)ax.y * sums[5] + (float)ax.z * sums[6];
    } else {
      const int k = tid - 6, C = S.C;
      float3 tk = make_float3(0.f, 0.f, 0.f);
      for (int p = S.grp_off[k]; p < S.grp_off[k + 1]; ++p) {
        const int m = S.grp_atoms[p];
        const float4 f4 = S.force[m];
        float3 F = make_float3(f4.x, f4.y, f4.z);
        if (intra)
          for (int c = 0; c < C; ++c) {
            const float4 fi = S.fintra[p * C + c];
            F.x += fi.x;
            F.y += fi.y;
            F.z += fi.z;
          }
        const float4 r4 = S.pos[m];
        const float3 t = cross3f(make_float3(r4.x, r4.y, r4.z), F);
        tk.x += t.x;
        tk.y += t.y;
        tk.z += t.z;
      }
      const d3 ax = mv(R, d3{S.taxes[3 * k], S.taxes[3 * k + 1], S.taxes[3 * k + 2]});
      out.gd = (float)ax.x * tk.x + (float)ax.y * tk.y + (float)ax.z * tk.z;
    }
  }
  return out;
}

template <int METHOD>
__device__ __forceinline__ typename GridEvalT<METHOD>::type grid_eval(const GridSmem& S, const GridView& G, int buf,
                                                                        bool intra, bool bad_in, bool& bad_out) {
  if constexpr (METHOD == kGridStrict) {
    return grid_eval_strict(S, G, buf, intra, bad_in, bad_out);
  } else {
    return grid_eval_fp32<METHOD>(S, G, buf, intra, bad_in, bad_out);
  }
}

// ------------------------------------------------------- local search
struct GridLs {
  double energy;
  int iterations, converged, status;
};

// local_search docking.cpp:310-351 by the whole CTA over grid evaluations.
// Thread d owns genotype dimension d (ADADELTA state in registers); the
// 16-deep best history is a per-warp register ring (slot = iter mod 16).
// On return S.best holds the best genotype (after a barrier).
template <int METHOD>
__device__ __forceinline__ GridLs grid_local_search(const GridSmem& S, const GridView& G, bool intra, const double* start,
                                    int max_iters, double tol) {
  const int tid = threadIdx.x, lane = tid & 31;
  const int dim = 6 + S.nr;
  const double rho = 0.95, eps = 1e-6;  // AdadeltaState::fresh docking.hpp:67-74
  double sg = 0.0, su = 0.0;
  if (tid < dim) {
    const double x = tid >= 3 ? wrap_angle(start[tid]) : start[tid];
    S.g[tid] = x;
    S.best[tid] = x;
  }
  bool bad = false;
  auto ev = grid_eval<METHOD>(S, G, 0, intra, false, bad);
  GridLs r;
  r.energy = (double)ev.e;
  r.iterations = 0;
  r.converged = 0;
  r.status = MDR_OK;
  double hist = r.energy;
  for (int iter = 1; iter <= max_iters; ++iter) {
    const bool mine_bad = tid < dim && !isfinite(ev.gd);
    if (tid < dim) {
      double x = S.g[tid];
      adadelta_dim(sg, su, x, (double)ev.gd, tid, rho, eps);
      S.g[tid] = x;
    }
    ev = grid_eval<METHOD>(S, G, iter & 1, intra, mine_bad, bad);
    if (bad) {  // NumericDomainError (docking.cpp:289-293): raised before the step
      r.status = MDR_ERR_NUMERIC_DOMAIN;
      break;
    }
    if ((double)ev.e < r.energy) {
      r.energy = (double)ev.e;
      if (tid < dim) S.best[tid] = S.g[tid];
    }
    const int slot = iter & (kWindow - 1);
    const double old = __shfl_sync(kFull, hist, slot);
    if (lane == slot) hist = r.energy;
    r.iterations = iter;
    if (iter >= kWindow && old - r.energy < tol) {
      r.converged = 1;
      break;
    }
  }
  __syncthreads();
  return r;
}

// --------------------------------------------------------------- kernels
template <int METHOD>
__global__ void grid_score_kernel(LigandView L, GridView G, FlexView F, const double* __restrict__ genos, int n,
                                  float* __restrict__ energy, float* __restrict__ grad, float* __restrict__ torque) {
  extern __shared__ __align__(16) unsigned char smem[];
  const GridSmem S = grid_load(L, F, smem, METHOD == kGridStrict);
  const int item = blockIdx.x;
  const int dim = 6 + L.n_rot;
  if (threadIdx.x < dim) S.g[threadIdx.x] = genos[(size_t)item * dim + threadIdx.x];
  __syncthreads();
  bool bad;
  const auto ev = grid_eval<METHOD>(S, G, 0, F.intra != 0, false, bad);
  if (threadIdx.x < dim) grad[(size_t)item * dim + threadIdx.x] = (float)ev.gd;
  if (threadIdx.x == 0) {
    energy[item] = (float)ev.e;
    float t[3] = {0.f, 0.f, 0.f};
    if constexpr (METHOD == kGridStrict) {
      for (int c = 0; c < 3; ++c) t[c] = (float)S.xtot[4 + c];
    } else {
      for (int w = 0; w < S.W; ++w)
        for (int c = 0; c < 3; ++c) t[c] += S.wpart[w * 8 + 4 + c];
    }
    torque[3 * (size_t)item] = t[0];
    torque[3 * (size_t)item + 1] = t[1];
    torque[3 * (size_t)item + 2] = t[2];
  }
}

template <int METHOD>
__global__ void grid_ls_kernel(LigandView L, GridView G, FlexView F, const double* __restrict__ starts, int n,
                               int max_iters, double tol, double* __restrict__ out_g, double* __restrict__ out_e,
                               int* __restrict__ out_it, int* __restrict__ out_cv, int* __restrict__ status) {
  extern __shared__ __align__(16) unsigned char smem[];
  const GridSmem S = grid_load(L, F, smem, METHOD == kGridStrict);
  __syncthreads();
  const int item = blockIdx.x;
  const int dim = 6 + L.n_rot;
  const GridLs r = grid_local_search<METHOD>(S, G, F.intra != 0, starts + (size_t)item * dim, max_iters, tol);
  if (threadIdx.x < dim) out_g[(size_t)item * dim + threadIdx.x] = S.best[threadIdx.x];
  if (threadIdx.x == 0) {
    out_e[item] = r.energy;
    out_it[item] = r.iterations;
    out_cv[item] = r.converged;
    if (r.status != MDR_OK) status[item] = r.status;
  }
}

// ------------------------------------------------------------- LGA phases
// All phases take a GridLigands table: a batch docks one ligand (n = 1) or
// a virtual-screen batch of many (run r docks ligand run_lig[r]).  D.dim is
// the genotype stride (the batch's largest dimension); each run uses its
// own ligand's dimension, and its RNG draw offsets (docking.cpp:437-465)
// follow that dimension exactly as a single-ligand lga_run would.
__device__ __forceinline__ int run_ligand(const GridLigands& GL, int run) { return GL.run_lig ? GL.run_lig[run] : 0; }

// random_genotype docking.cpp:360-388 + score, CTA per individual.
template <int METHOD>
__global__ void grid_lga_init_kernel(GridLigands GL, GridView G, LgaDev D) {
  extern __shared__ __align__(16) unsigned char smem[];
  const int item = blockIdx.x;
  const int run = item / D.P, p = item % D.P;
  const int lig = run_ligand(GL, run);
  const LigandView L = GL.L[lig];
  const FlexView F = GL.F[lig];
  const GridSmem S = grid_load(L, F, smem, METHOD == kGridStrict);
  const int dim = 6 + L.n_rot;
  const int d = threadIdx.x;
  if (d < dim) {
    const uint64_t key = run_key(D, run);
    const uint64_t n = (uint64_t)p * dim + d + 1;
    const double x = d < 3 ? L.box[d] + (L.box[3 + d] - L.box[d]) * draw_unit(key, n)
                           : -kPi + (kPi - -kPi) * draw_unit(key, n);
    S.g[d] = x;
    D.pop[0][((size_t)run * D.P + p) * D.dim + d] = x;
  }
  __syncthreads();
  bool bad;
  const auto ev = grid_eval<METHOD>(S, G, 0, F.intra != 0, false, bad);
  if (threadIdx.x == 0) D.pope[0][(size_t)run * D.P + p] = (double)ev.e;
}

// Offspring (docking.cpp:437-472), CTA per child; thread d forms dimension d.
template <int METHOD>
__global__ void grid_lga_offspring_kernel(GridLigands GL, GridView G, LgaDev D, int gen) {
  extern __shared__ __align__(16) unsigned char smem[];
  const int item = blockIdx.x;
  const int run = item / D.off, i = item % D.off;
  if (!D.active[run]) return;  // uniform over the CTA
  const int lig = run_ligand(GL, run);
  const LigandView L = GL.L[lig];
  const FlexView F = GL.F[lig];
  const GridSmem S = grid_load(L, F, smem, METHOD == kGridStrict);
  const int dim = 6 + L.n_rot;
  const int c = D.cur[run];
  const double* pop = D.pop[c] + (size_t)run * D.P * D.dim;
  const double* pe = D.pope[c] + (size_t)run * D.P;
  double* nxt = D.pop[c ^ 1] + (size_t)run * D.P * D.dim;
  double* ne = D.pope[c ^ 1] + (size_t)run * D.P;
  if (i == 0 && threadIdx.x < 32) {  // elitism of one: first index of the strict minimum
    double be = pe[0];
    int bi = 0;
    for (int p = 1; p < D.P; ++p)
      if (pe[p] < be) {
        be = pe[p];
        bi = p;
      }
    for (int d = threadIdx.x; d < dim; d += 32) nxt[d] = pop[(size_t)bi * D.dim + d];
    if (threadIdx.x == 0) ne[0] = be;
  }
  const uint64_t key = run_key(D, run);
  const uint64_t base = (uint64_t)D.P * dim + ((uint64_t)gen * D.off + i) * (uint64_t)(4 + 3 * dim);
  const int d = threadIdx.x;
  if (d < dim) {
    const int ia = (int)(draw_u64(key, base + 1) % (uint64_t)D.P);
    const int ja = (int)(draw_u64(key, base + 2) % (uint64_t)D.P);
    const int a = pe[ia] <= pe[ja] ? ia : ja;
    const int ib = (int)(draw_u64(key, base + 3) % (uint64_t)D.P);
    const int jb = (int)(draw_u64(key, base + 4) % (uint64_t)D.P);
    const int b = pe[ib] <= pe[jb] ? ib : jb;
    const double lam = draw_unit(key, base + 5 + d);
    double x = lam * pop[(size_t)a * D.dim + d] + (1.0 - lam) * pop[(size_t)b * D.dim + d];
    x = x + D.sigma * draw_normal(key, base + 5 + dim + 2 * (uint64_t)d);
    if (d >= 3) x = wrap_angle(x);
    S.g[d] = x;
    nxt[(size_t)(1 + i) * D.dim + d] = x;
  }
  __syncthreads();
  bool bad;
  const auto ev = grid_eval<METHOD>(S, G, 0, F.intra != 0, false, bad);
  if (threadIdx.x == 0) ne[1 + i] = (double)ev.e;
}

#if MDR_PHASE_PROF
__device__ unsigned int g_sm_grid[256];  // grid LGA searches started per SM (phase-profiling builds)
#endif

template <int METHOD>
__global__ void grid_lga_ls_kernel(GridLigands GL, GridView G, LgaDev D) {
  extern __shared__ __align__(16) unsigned char smem[];
  __shared__ int s_target;
  const int item = blockIdx.x;
#if MDR_PHASE_PROF
  if (threadIdx.x == 0) {
    unsigned sm;
    asm volatile("mov.u32 %0, %%smid;" : "=r"(sm));
    atomicAdd(&g_sm_grid[sm & 255], 1u);
  }
#endif
  const int run = item / D.L, r = item % D.L;
  if (!D.active[run]) return;
  const int lig = run_ligand(GL, run);
  const LigandView L = GL.L[lig];
  const FlexView F = GL.F[lig];
  const GridSmem S = grid_load(L, F, smem, METHOD == kGridStrict);
  const int dim = 6 + L.n_rot;
  if (threadIdx.x < 32) {
    const int t = ls_target(D, run, r);
    if (threadIdx.x == 0) s_target = t;
  }
  __syncthreads();
  const int target = s_target;
  const int c = D.cur[run];
  const double* start = D.pop[c ^ 1] + ((size_t)run * D.P + target) * D.dim;
  const GridLs res = grid_local_search<METHOD>(S, G, F.intra != 0, start, D.ls_iters, D.tol);
  const size_t o = (size_t)run * D.L + r;
  if (threadIdx.x < dim) D.lsg[o * D.dim + threadIdx.x] = S.best[threadIdx.x];
  if (threadIdx.x == 0) {
    D.lse[o] = res.energy;
    D.lsit[o] = res.iterations;
    D.lscv[o] = res.converged;
    D.lstarget[o] = target;
    if (res.status != MDR_OK) D.status[run] = res.status;
  }
}

// Final polish from the incumbent best (docking.cpp:501-515), CTA per run.
template <int METHOD>
__global__ void grid_lga_polish_kernel(GridLigands GL, GridView G, LgaDev D) {
  extern __shared__ __align__(16) unsigned char smem[];
  const int run = blockIdx.x;
  const int lig = run_ligand(GL, run);
  const LigandView L = GL.L[lig];
  const FlexView F = GL.F[lig];
  const GridSmem S = grid_load(L, F, smem, METHOD == kGridStrict);
  __syncthreads();
  if (D.status[run] != MDR_OK) return;
  const long long remaining = D.max_evals - D.evals[run];
  if (remaining <= 1) {
    if (threadIdx.x == 0) D.conv[run] = 0;
    return;
  }
  const int iters = (int)((long long)D.ls_iters < remaining - 1 ? (long long)D.ls_iters : remaining - 1);
  const GridLs res = grid_local_search<METHOD>(S, G, F.intra != 0, D.best_g + (size_t)run * D.dim, iters, D.tol);
  if (threadIdx.x == 0) {
    if (res.status != MDR_OK) {
      D.status[run] = res.status;
      return;
    }
    D.evals[run] += res.iterations + 1;
    track_best(D, run, S.best, res.energy);
    push_record(D, run, res.energy, res.iterations, res.converged);
    D.conv[run] = res.converged;
  }
}

// -------------------------------------------------------- map builder
// mdr_grid_build: thread per lattice point, FP64 in the oracle's order.
__global__ void grid_build_kernel(GridView G, const double* __restrict__ sites, int n_sites,
                                  const double* __restrict__ charge, const double* __restrict__ volume,
                                  const double* __restrict__ depth_scale, const double* __restrict__ dist_scale,
                                  double elec_scale, double two_s2, float* __restrict__ maps) {
  const long long o = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (o >= G.stride) return;
  const int ix = (int)(o % G.nx), iy = (int)((o / G.nx) % G.ny), iz = (int)(o / ((long long)G.nx * G.ny));
  const double P[3] = {G.ox + G.h * ix, G.oy + G.h * iy, G.oz + G.h * iz};
  for (int t = 0; t < G.n_types + 2; ++t) {
    double v = 0.0;
    for (int j = 0; j < n_sites; ++j) {
      const double* s = sites + 5 * j;
      const double dx = P[0] - s[0], dy = P[1] - s[1], dz = P[2] - s[2];
      const double r2 = dx * dx + dy * dy + dz * dz;
      if (t < G.n_types) {
        const double d = s[4] * dist_scale[t];
        const double c2 = 0.5625 * d * d;
        const double u = r2 + c2;
        const double rho2 = (d * d + c2) / u;
        const double rho6 = rho2 * rho2 * rho2;
        const double rho12 = rho6 * rho6;
        v += s[3] * depth_scale[t] * (rho12 - 2.0 * rho6);
      } else if (t == G.n_types) {
        v += elec_scale * charge[j] / (r2 + 0.5625 * s[4] * s[4]);
      } else {
        v += volume[j] * exp(-r2 / two_s2);
      }
    }
    maps[(long long)t * G.stride + o] = (float)v;
  }
}

// ------------------------------------------------------------ host side
template <class K>
static cudaError_t gprep(K kernel, size_t smem) {
  if (smem > 48 * 1024) return cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  return cudaSuccess;
}

#define MDR_GRID_DISPATCH(KERNEL)                                                                   \
  template <class... A>                                                                             \
  static void gdispatch_##KERNEL(int method, dim3 g, dim3 b, size_t smem, cudaStream_t s, A... args) { \
    switch (method) {                                                                               \
      case MDR_METHOD_BASELINE: KERNEL<MDR_METHOD_BASELINE><<<g, b, smem, s>>>(args...); break;     \
      case MDR_METHOD_TCU: KERNEL<MDR_METHOD_TCU><<<g, b, smem, s>>>(args...); break;               \
      case kGridStrict: KERNEL<kGridStrict><<<g, b, smem, s>>>(args...); break;                     \
      default: KERNEL<MDR_METHOD_TCU_SPLIT><<<g, b, smem, s>>>(args...); break;                     \
    }                                                                                               \
  }                                                                                                 \
  static cudaError_t gprep_##KERNEL(int method, size_t smem) {                                      \
    switch (method) {                                                                               \
      case MDR_METHOD_BASELINE: return gprep(KERNEL<MDR_METHOD_BASELINE>, smem);                    \
      case MDR_METHOD_TCU: return gprep(KERNEL<MDR_METHOD_TCU>, smem);                              \
      case kGridStrict: return gprep(KERNEL<kGridStrict>, smem);                                    \
      default: return gprep(KERNEL<MDR_METHOD_TCU_SPLIT>, smem);                                    \
    }                                                                                               \
  }

MDR_GRID_DISPATCH(grid_score_kernel)
MDR_GRID_DISPATCH(grid_ls_kernel)
MDR_GRID_DISPATCH(grid_lga_init_kernel)
MDR_GRID_DISPATCH(grid_lga_offspring_kernel)
MDR_GRID_DISPATCH(grid_lga_ls_kernel)
MDR_GRID_DISPATCH(grid_lga_polish_kernel)

static size_t gsmem(const LigandView& L, const FlexView& F, int T, int method) {
  return grid_smem_bytes(L.n_atoms, L.n_rot, F.n_tors_atoms, T) + (method == kGridStrict ? grid_strict_bytes(L.n_atoms) : 0);
}

size_t grid_smem_for(const LigandView& L, const FlexView& F, int threads, int method) {
  return gsmem(L, F, threads, method);
}
size_t grid_smem_for(int n_atoms, int n_rot, int n_tors_atoms, int threads) {
  return grid_smem_bytes(n_atoms, n_rot, n_tors_atoms, threads);
}

cudaError_t launch_grid_score(const LigandView& L, const GridView& G, const FlexView& F, const double* genos, int n,
                              int method, int threads, float* energy, float* grad, float* torque, cudaStream_t s) {
  if (n <= 0) return cudaSuccess;
  const size_t sm = gsmem(L, F, threads, method);
  cudaError_t e = gprep_grid_score_kernel(method, sm);
  if (e != cudaSuccess) return e;
  gdispatch_grid_score_kernel(method, n, threads, sm, s, L, G, F, genos, n, energy, grad, torque);
  return cudaGetLastError();
}

cudaError_t launch_grid_local_search(const LigandView& L, const GridView& G, const FlexView& F, const double* starts,
                                     int n, int max_iters, double tol, int method, int threads, double* out_g,
                                     double* out_e, int* out_it, int* out_cv, int* status, cudaStream_t s) {
  if (n <= 0) return cudaSuccess;
  const size_t sm = gsmem(L, F, threads, method);
  cudaError_t e = gprep_grid_ls_kernel(method, sm);
  if (e != cudaSuccess) return e;
  gdispatch_grid_ls_kernel(method, n, threads, sm, s, L, G, F, starts, n, max_iters, tol, out_g, out_e, out_it,
                           out_cv, status);
  return cudaGetLastError();
}

cudaError_t prepare_grid_lga(size_t sm, int method) {
  cudaError_t e = gprep_grid_lga_init_kernel(method, sm);
  if (e == cudaSuccess) e = gprep_grid_lga_offspring_kernel(method, sm);
  if (e == cudaSuccess) e = gprep_grid_lga_ls_kernel(method, sm);
  if (e == cudaSuccess) e = gprep_grid_lga_polish_kernel(method, sm);
  return e;
}

cudaError_t launch_grid_lga(const GridLigands& GL, size_t sm, const GridView& G, const LgaDev& D, int method,
                            int threads, cudaStream_t s, int* n_launches, cudaEvent_t* ls_events) {
  int launches = 0;
  cudaError_t e = cudaSuccess;
  if (ls_events) cudaEventRecord(ls_events[2 * D.gens + 2], s);
  gdispatch_grid_lga_init_kernel(method, D.R * D.P, threads, sm, s, GL, G, D);
  if ((e = launch_lga_init_finalize(D, s)) != cudaSuccess) return e;
  launches += 2;
  for (int gen = 0; gen < D.gens; ++gen) {
    gdispatch_grid_lga_offspring_kernel(method, D.R * D.off, threads, sm, s, GL, G, D, gen);
    if (ls_events) cudaEventRecord(ls_events[2 * gen], s);
    if (D.L > 0) gdispatch_grid_lga_ls_kernel(method, D.R * D.L, threads, sm, s, GL, G, D);
    if (ls_events) cudaEventRecord(ls_events[2 * gen + 1], s);
    if ((e = launch_lga_gen_finalize(D, gen, s)) != cudaSuccess) return e;
    launches += D.L > 0 ? 3 : 2;
  }
  if (ls_events) cudaEventRecord(ls_events[2 * D.gens], s);
  gdispatch_grid_lga_polish_kernel(method, D.R, threads, sm, s, GL, G, D);
  if (ls_events) cudaEventRecord(ls_events[2 * D.gens + 1], s);
  if (ls_events) cudaEventRecord(ls_events[2 * D.gens + 3], s);
  launches += 1;
  if (n_launches) *n_launches = launches;
  return cudaGetLastError();
}

bool sm_grid_read(unsigned* out256, bool reset) {
#if MDR_PHASE_PROF
  if (cudaMemcpyFromSymbol(out256, g_sm_grid, sizeof(unsigned) * 256) != cudaSuccess) return false;
  if (reset) {
    unsigned z[256] = {};
    if (cudaMemcpyToSymbol(g_sm_grid, z, sizeof(z)) != cudaSuccess) return false;
  }
  return true;
#else
  (void)out256;
  (void)reset;
  return false;
#endif
}

cudaError_t launch_grid_build(const GridView& G, const double* sites, int n_sites, const double* charge,
                              const double* volume, const double* depth_scale, const double* dist_scale,
                              double elec_scale, double sigma, float* maps, cudaStream_t s) {
  const long long n = G.stride;
  grid_build_kernel<<<(unsigned)((n + 127) / 128), 128, 0, s>>>(G, sites, n_sites, charge, volume, depth_scale,
                                                                 dist_scale, elec_scale, 2.0 * sigma * sigma, maps);
  return cudaGetLastError();
}

}  // namespace mdr
