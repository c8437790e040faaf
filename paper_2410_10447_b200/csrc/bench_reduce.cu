// bench_reduce.cu — C2 microbench: block float4 sum-reduce-and-broadcast,
// one reduction per thread block of B threads (the paper's test-kernel
// shape), head to head:
//
//   K1a reducefs   AutoDock's REDUCEFLOATSUM x4: per
//                  component a shuffle-down tree, one shared-memory atomicAdd
//                  per warp, __threadfence() x2, __syncthreads() x3.
//   K1b shuffle    strong warp-shuffle baseline: a 6-shuffle transpose-reduce
//                  of the float4 in each warp, one double-buffered smem
//                  exchange, 1 __syncthreads per reduction.
//   K2  wmma_f16   the paper's method: f16 staging in
//                  shared memory, one warp runs ceil(B/64) mma.sync against
//                  P = ones with an f16 accumulator, then Q = I4 blocks; 2
//                  syncs; f16 accuracy (~1e-3).
//   K2p split_tc   the paper's 2-sync structure with the error-compensated
//                  tf32 hi/lo split (fp32 accurate), one warp issues all MMAs.
//   K2s split_warp every warp reduces its own 32 float4 with tf32 hi/lo
//                  m16n8k8 MMAs (no shuffles for the intra-warp part), then
//                  the K1b exchange: 1 sync.
//
// Two modes: chain_steps R > 0 — each block loads one input set and runs a
// dependent chain of R reduce-and-broadcast steps (v += 2^-20 * sum, so
// nothing can be hoisted; on-chip, bound by issue/smem/barriers);
// chain_steps == 0 — streaming: every reduction reads a distinct input set
// from HBM (persistent blocks).
#include <cuda_runtime.h>

#include "dock_launch.h"
#include <cuda_bf16.h>

#include "mdr_device.cuh"

namespace mdr {
namespace bench {

constexpr int kMaxWarps = 32;
constexpr float kFeed = 0x1p-20f;

// Static part (1.1 KB) + a dynamic staging area sized by the kernel that
// needs it (K2: 8*B bytes of f16, K2p/K2s: 16*B bytes of fp32), so the
// shuffle kernels keep full occupancy.
struct Smem {
  float acc[4];                           // K1a accumulator
  __align__(16) float part[2][kMaxWarps][4];  // K1b/K2s double-buffered warp partials
  __align__(16) float result[2][4];       // K2/K2p broadcast
  __half* tile;                           // K2: f16 staging
  float* stage;                           // K2p/K2s: fp32 staging
};
extern __shared__ __align__(16) unsigned char g_dyn[];

__device__ __forceinline__ float4 add_feed(float4 v, float4 s) {
  return make_float4(v.x + kFeed * s.x, v.y + kFeed * s.y, v.z + kFeed * s.z, v.w + kFeed * s.w);
}

// ---------------------------------------------------------------- K1a
__device__ __forceinline__ float reducefs(float value, float* acc) {
  if (threadIdx.x == 0) *acc = 0.0f;
  __threadfence();
  __syncthreads();
#pragma unroll
  for (int off = 16; off >= 1; off >>= 1) value += __shfl_down_sync(kFull, value, off);
  if ((threadIdx.x & 31) == 0) atomicAdd(acc, value);
  __threadfence();
  __syncthreads();
  value = *acc;
  __syncthreads();
  return value;
}

__device__ __forceinline__ float4 k1a(float4 v, Smem& sm, int) {
  float4 s;
  s.x = reducefs(v.x, &sm.acc[0]);
  s.y = reducefs(v.y, &sm.acc[1]);
  s.z = reducefs(v.z, &sm.acc[2]);
  s.w = reducefs(v.w, &sm.acc[3]);
  return s;
}

// ---------------------------------------------------------------- K1b
// 6-shuffle transpose-reduce: lane ends holding component
// k = 2*bit4 + bit3 of its lane id, summed over the warp.
__device__ __forceinline__ float warp_transpose_reduce(float4 v, int lane) {
  const bool hi16 = lane & 16, hi8 = lane & 8;
  float a0 = hi16 ? v.z : v.x, a1 = hi16 ? v.w : v.y;
  const float b0 = hi16 ? v.x : v.z, b1 = hi16 ? v.y : v.w;
  a0 += __shfl_xor_sync(kFull, b0, 16);
  a1 += __shfl_xor_sync(kFull, b1, 16);
  float c = hi8 ? a1 : a0;
  const float d = hi8 ? a0 : a1;
  c += __shfl_xor_sync(kFull, d, 8);
  c += __shfl_xor_sync(kFull, c, 4);
  c += __shfl_xor_sync(kFull, c, 2);
  c += __shfl_xor_sync(kFull, c, 1);
  return c;
}

__device__ __forceinline__ float4 block_exchange(float c_of_lane, Smem& sm, int buf, int lane, int warp, int nw,
                                                 bool lanes_hold_k8) {
  // lanes_hold_k8: component k is in lane 8k (transpose-reduce layout);
  // otherwise in lane 4k (MMA layout)
  if (lanes_hold_k8) {
    if ((lane & 7) == 0) sm.part[buf][warp][lane >> 3] = c_of_lane;
  } else {
    if ((lane & 3) == 0 && lane < 16) sm.part[buf][warp][lane >> 2] = c_of_lane;
  }
  __syncthreads();
  float4 s = make_float4(0.f, 0.f, 0.f, 0.f);
  for (int w = 0; w < nw; ++w) {
    const float4 p = *reinterpret_cast<const float4*>(sm.part[buf][w]);
    s.x += p.x;
    s.y += p.y;
    s.z += p.z;
    s.w += p.w;
  }
  return s;
}

__device__ __forceinline__ float4 k1b(float4 v, Smem& sm, int it) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const float c = warp_transpose_reduce(v, lane);
  return block_exchange(c, sm, it & 1, lane, warp, blockDim.x >> 5, true);
}

// ---------------------------------------------------------------- K2
__device__ __forceinline__ void mma_f16acc(uint32_t (&d)[2], const uint32_t (&a)[4], uint32_t b0, uint32_t b1,
                                           const uint32_t (&c)[2]) {
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f16.f16.f16.f16 {%0,%1}, {%2,%3,%4,%5}, {%6,%7}, {%8,%9};\n"
      : "=r"(d[0]), "=r"(d[1])
      : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1), "r"(c[0]), "r"(c[1]));
}

__device__ __forceinline__ float4 k2(float4 v, Smem& sm, int it) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  __half2* t2 = reinterpret_cast<__half2*>(sm.tile);
  t2[2 * threadIdx.x] = __floats2half2_rn(v.x, v.y);
  t2[2 * threadIdx.x + 1] = __floats2half2_rn(v.z, v.w);
  __syncthreads();
  const int buf = it & 1;
  if (warp == 0) {
    const int mat = lane >> 3, r = lane & 7;
    const int col = r + 8 * (mat >> 1), rowoff = 8 * (mat & 1);
    uint32_t V[2] = {0u, 0u};  // f16 accumulator (the paper's choice)
    const uint32_t ones = 0x3C003C00u;
    for (int c = 0; c < (int)blockDim.x; c += 64) {
      uint32_t a[4];
      ldsm_x4_trans(a, sm.tile + 4 * c + col * 16 + rowoff);
      uint32_t d[2];
      mma_f16acc(d, a, ones, ones, V);
      V[0] = d[0];
      V[1] = d[1];
    }
    // W = Q * V: V rows g (V[0] low half) and g + 8 (V[1] low half)
    const int g = lane >> 2, t = lane & 3;
    const uint32_t x = (V[0] & 0xffffu) | (V[1] << 16);
    const uint32_t y0 = __shfl_sync(kFull, x, 8 * t), y1 = __shfl_sync(kFull, x, 8 * t + 4);
    const uint32_t b0 = (y0 & 0xffffu) | (y1 << 16), b1 = (y0 >> 16) | (y1 & 0xffff0000u);
    const uint32_t qa = ((g & 3) == ((2 * t) & 3) ? 0x3C00u : 0u) | ((g & 3) == ((2 * t + 1) & 3) ? 0x3C000000u : 0u);
    const uint32_t qa4[4] = {qa, qa, qa, qa}, z[2] = {0u, 0u};
    uint32_t W[2];
    mma_f16acc(W, qa4, b0, b1, z);
    if (t == 0 && g < 4) sm.result[buf][g] = __low2float(*reinterpret_cast<__half2*>(&W[0]));
  }
  __syncthreads();
  return *reinterpret_cast<const float4*>(sm.result[buf]);
}

// ---------------------------------------------------------------- K2p
__device__ __forceinline__ float4 k2p(float4 v, Smem& sm, int it) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  reinterpret_cast<float4*>(sm.stage)[threadIdx.x] = v;
  __syncthreads();
  const int buf = it & 1;
  if (warp == 0) {
    // rows 0..3: hi of component g, rows 8..11: lo; k = 8 source threads
    const int g = lane >> 2, t = lane & 3;
    float acc[4] = {0.f, 0.f, 0.f, 0.f};
    const uint32_t one = 0x3f800000u;
    const int comp = g & 3;
    for (int base = 0; base < (int)blockDim.x; base += 8) {
      const float x0 = g < 4 ? sm.stage[(base + t) * 4 + comp] : 0.f;
      const float x1 = g < 4 ? sm.stage[(base + t + 4) * 4 + comp] : 0.f;
      const uint32_t h0 = to_tf32(x0), h1 = to_tf32(x1);
      const uint32_t l0 = to_tf32(x0 - __uint_as_float(h0)), l1 = to_tf32(x1 - __uint_as_float(h1));
      const uint32_t a[4] = {h0, l0, h1, l1};
      mma_tf32_1688(acc, a, one, one);
    }
    if (t == 0 && g < 4) sm.result[buf][g] = acc[0] + acc[2];
  }
  __syncthreads();
  return *reinterpret_cast<const float4*>(sm.result[buf]);
}

// ---------------------------------------------------------------- K2s
__device__ __forceinline__ float4 k2s(float4 v, Smem& sm, int it) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  float* st = sm.stage + warp * 32 * 4;
  reinterpret_cast<float4*>(st)[lane] = v;
  __syncwarp();
  const int g = lane >> 2, t = lane & 3, comp = g & 3;
  float acc[4] = {0.f, 0.f, 0.f, 0.f};
  const uint32_t one = 0x3f800000u;
#pragma unroll
  for (int kb = 0; kb < 4; ++kb) {
    const float x0 = g < 4 ? st[(kb * 8 + t) * 4 + comp] : 0.f;
    const float x1 = g < 4 ? st[(kb * 8 + t + 4) * 4 + comp] : 0.f;
    const uint32_t h0 = to_tf32(x0), h1 = to_tf32(x1);
    const uint32_t l0 = to_tf32(x0 - __uint_as_float(h0)), l1 = to_tf32(x1 - __uint_as_float(h1));
    const uint32_t a[4] = {h0, l0, h1, l1};
    mma_tf32_1688(acc, a, one, one);
  }
  __syncwarp();
  return block_exchange(acc[0] + acc[2], sm, it & 1, lane, warp, blockDim.x >> 5, false);
}

// ---------------------------------------------------------------- K1c
// Two-level shuffle: warp transpose-reduce, then warp 0 folds the per-warp
// partials with shuffles and publishes one float4 (2 syncs, few
// instructions per thread).
__device__ __forceinline__ float4 k1c(float4 v, Smem& sm, int it) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  const int buf = it & 1;
  const float c = warp_transpose_reduce(v, lane);
  if ((lane & 7) == 0) sm.part[buf][warp][lane >> 3] = c;
  __syncthreads();
  if (warp == 0) {
    // lane l: component l & 3 of warps l>>2, (l>>2) + 8, ... (ascending)
    float s = 0.f;
    for (int w = lane >> 2; w < nw; w += 8) s += sm.part[buf][w][lane & 3];
    s += __shfl_xor_sync(kFull, s, 4);
    s += __shfl_xor_sync(kFull, s, 8);
    s += __shfl_xor_sync(kFull, s, 16);
    if (lane < 4) sm.result[buf][lane] = s;
  }
  __syncthreads();
  return *reinterpret_cast<const float4*>(sm.result[buf]);
}

// ---------------------------------------------------------------- K2b
// The paper's 2-sync tensor-core reduction made fp32-accurate: every value
// is split into three bf16 terms (hi + mid + lo carry 24 significant bits,
// bf16 keeps the fp32 exponent range so no scaling is needed), staged in the
// paper's column-major packing, summed by m16n8k16 bf16 MMAs against P =
// ones into fp32 accumulators; the Q fold (4 row groups) is 2 shuffles.
__device__ __forceinline__ void mma_bf16_16816(float (&d)[4], const uint32_t (&a)[4], uint32_t b0, uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
      "{%0,%1,%2,%3};\n"
      : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
      : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}

struct Bf16x3 {
  uint32_t hi[2], mid[2], lo[2];  // (x,y), (z,e) pairs per term
};
__device__ __forceinline__ uint32_t bf2(float a, float b) {
  __nv_bfloat162 h = __floats2bfloat162_rn(a, b);
  return *reinterpret_cast<uint32_t*>(&h);
}
__device__ __forceinline__ void split3(float x, float& h, float& m, float& l) {
  h = __bfloat162float(__float2bfloat16_rn(x));
  const float r = x - h;  // exact
  m = __bfloat162float(__float2bfloat16_rn(r));
  l = r - m;  // exact; rounded to bf16 at packing
}

__device__ __forceinline__ float4 k2b(float4 v, Smem& sm, int it) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int B = blockDim.x;
  __nv_bfloat16* t0 = reinterpret_cast<__nv_bfloat16*>(sm.tile);
  float hx, mx, lx, hy, my, ly, hz, mz, lz, he, me, le;
  split3(v.x, hx, mx, lx);
  split3(v.y, hy, my, ly);
  split3(v.z, hz, mz, lz);
  split3(v.w, he, me, le);
  uint2* s0 = reinterpret_cast<uint2*>(t0);
  uint2* s1 = reinterpret_cast<uint2*>(t0 + 4 * B);
  uint2* s2 = reinterpret_cast<uint2*>(t0 + 8 * B);
  s0[threadIdx.x] = make_uint2(bf2(hx, hy), bf2(hz, he));
  s1[threadIdx.x] = make_uint2(bf2(mx, my), bf2(mz, me));
  s2[threadIdx.x] = make_uint2(bf2(lx, ly), bf2(lz, le));
  __syncthreads();
  const int buf = it & 1;
  if (warp == 0) {
    const int mat = lane >> 3, r = lane & 7;
    const int col = r + 8 * (mat >> 1), rowoff = 8 * (mat & 1);
    const uint32_t ones = 0x3F803F80u;  // bf16 1.0 pairs
    float a0[4] = {0.f, 0.f, 0.f, 0.f}, a1[4] = {0.f, 0.f, 0.f, 0.f}, a2[4] = {0.f, 0.f, 0.f, 0.f};
    for (int c = 0; c < B; c += 64) {
      uint32_t f0[4], f1[4], f2[4];
      ldsm_x4_trans(f0, reinterpret_cast<const __half*>(t0) + 4 * c + col * 16 + rowoff);
      ldsm_x4_trans(f1, reinterpret_cast<const __half*>(t0 + 4 * B) + 4 * c + col * 16 + rowoff);
      ldsm_x4_trans(f2, reinterpret_cast<const __half*>(t0 + 8 * B) + 4 * c + col * 16 + rowoff);
      mma_bf16_16816(a0, f0, ones, ones);
      mma_bf16_16816(a1, f1, ones, ones);
      mma_bf16_16816(a2, f2, ones, ones);
    }
    // V rows g (d0) and g+8 (d2); W_c = V[c] + V[c+4] + V[c+8] + V[c+12]
    const float r0 = (a0[0] + a1[0]) + a2[0], r2 = (a0[2] + a1[2]) + a2[2];
    const float p = r0 + __shfl_down_sync(kFull, r0, 16);
    const float q = r2 + __shfl_down_sync(kFull, r2, 16);
    const int g = lane >> 2, t = lane & 3;
    if (t == 0 && g < 4) sm.result[buf][g] = p + q;
  }
  __syncthreads();
  return *reinterpret_cast<const float4*>(sm.result[buf]);
}

// ---------------------------------------------------------------- kernels
template <int K>
__device__ __forceinline__ float4 reduce_once(float4 v, Smem& sm, int it) {
  if (K == 0) return k1a(v, sm, it);
  if (K == 1) return k1b(v, sm, it);
  if (K == 2) return k2(v, sm, it);
  if (K == 3) return k2p(v, sm, it);
  if (K == 4) return k2s(v, sm, it);
  if (K == 5) return k1c(v, sm, it);
  return k2b(v, sm, it);
}

// cyc (optional): per block, the SM clock cycles of its whole chain
// (clock64 by thread 0 around the loop, after a block barrier), for the
// latency metric (cycles per dependent step).
template <int K>
__global__ void chain_kernel(const float4* __restrict__ in, int steps, float4* __restrict__ out,
                             long long* __restrict__ cyc) {
  __shared__ Smem sm;
  sm.tile = reinterpret_cast<__half*>(g_dyn);
  sm.stage = reinterpret_cast<float*>(g_dyn);
  float4 v = in[(size_t)blockIdx.x * blockDim.x + threadIdx.x];
  float4 s = make_float4(0.f, 0.f, 0.f, 0.f);
  __syncthreads();
  const long long t0 = clock64();
  for (int it = 0; it < steps; ++it) {
    s = reduce_once<K>(v, sm, it);
    v = add_feed(v, s);
  }
  if (threadIdx.x == 0) {
    out[blockIdx.x] = s;
    if (cyc) cyc[blockIdx.x] = clock64() - t0;
  }
}

#ifndef MDR_STREAM_PREFETCH
#define MDR_STREAM_PREFETCH 0  // input sets in flight per thread (0: load at use)
#endif
// Streaming: block b reduces sets b, b + grid, ...; each thread keeps
// MDR_STREAM_PREFETCH sets' float4 loads in flight (the one being reduced
// and the next ones) (the block barriers of the reduction would otherwise
// drain the memory pipe between sets).
template <int K>
__global__ void stream_kernel(const float4* __restrict__ in, int n_red, float4* __restrict__ out) {
  __shared__ Smem sm;
  sm.tile = reinterpret_cast<__half*>(g_dyn);
  sm.stage = reinterpret_cast<float*>(g_dyn);
  constexpr int P = MDR_STREAM_PREFETCH;
  if constexpr (P == 0) {  // load at use
    int it = 0;
    for (int r = blockIdx.x; r < n_red; r += gridDim.x, ++it) {
      const float4 s = reduce_once<K>(__ldcs(&in[(size_t)r * blockDim.x + threadIdx.x]), sm, it);
      if (threadIdx.x == 0) out[r] = s;
    }
    return;
  }
  const float4 zero = make_float4(0.f, 0.f, 0.f, 0.f);
  float4 q[P > 0 ? P : 1];
#pragma unroll
  for (int k = 0; k < P; ++k) {
    const int r = blockIdx.x + k * gridDim.x;
    q[k] = r < n_red ? __ldcs(&in[(size_t)r * blockDim.x + threadIdx.x]) : zero;
  }
  int it = 0;
  for (int r = blockIdx.x; r < n_red; r += gridDim.x, ++it) {
    const float4 v = q[0];
#pragma unroll
    for (int k = 0; k + 1 < P; ++k) q[k] = q[k + 1];
    const int rn = r + P * gridDim.x;
    q[P - 1] = rn < n_red ? __ldcs(&in[(size_t)rn * blockDim.x + threadIdx.x]) : zero;
    const float4 s = reduce_once<K>(v, sm, it);
    if (threadIdx.x == 0) out[r] = s;
  }
}

}  // namespace bench

static const char* kNames[] = {"reducefs_x4 (AutoDock, K1a)", "shuffle_transpose (K1b)", "wmma_f16 (paper, K2)",
                               "split_tf32_block (K2p)", "split_tf32_warp (K2s)", "shuffle_2level (K1c)",
                               "split_bf16x3_mma (K2b)", "tcgen05_batched_tf32x2 (K2t)",
                               "tcgen05_tma_pipelined (K2t2)"};

cudaError_t launch_reduce_bench(int kernel, int block, const float* in, int n_red, int chain_steps, float* out,
                                int blocks_per_sm, cudaStream_t s, long long* cycles) {
  const float4* i4 = reinterpret_cast<const float4*>(in);
  float4* o4 = reinterpret_cast<float4*>(out);
  const size_t dyn = kernel == 2 ? (size_t)8 * block
                     : kernel == 6 ? (size_t)24 * block
                     : (kernel == 3 || kernel == 4) ? (size_t)16 * block : 0;
  if (chain_steps > 0) {
    const int grid = n_red / chain_steps;
#define CH(K) bench::chain_kernel<K><<<grid, block, dyn, s>>>(i4, chain_steps, o4, cycles)
    switch (kernel) {
      case 0: CH(0); break;
      case 1: CH(1); break;
      case 2: CH(2); break;
      case 3: CH(3); break;
      case 4: CH(4); break;
      case 5: CH(5); break;
      default: CH(6); break;
    }
#undef CH
  } else {
    int grid = 148 * blocks_per_sm;
    if (grid > n_red) grid = n_red;
#define ST(K) bench::stream_kernel<K><<<grid, block, dyn, s>>>(i4, n_red, o4)
    switch (kernel) {
      case 0: ST(0); break;
      case 1: ST(1); break;
      case 2: ST(2); break;
      case 3: ST(3); break;
      case 4: ST(4); break;
      case 5: ST(5); break;
      default: ST(6); break;
    }
#undef ST
  }
  return cudaGetLastError();
}

const char* reduce_bench_name(int k) { return (k >= 0 && k < kReduceBenchKernels) ? kNames[k] : "unknown"; }

}  // namespace mdr
