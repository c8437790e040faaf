// tc05_reduce.cu — K2t: many float4 block reductions merged into ONE tensor
// contraction on the 5th-generation tensor cores (tcgen05 + TMEM).
//
// The paper reduces one block's float4 records with a 16x16 WMMA against an
// all-ones matrix.  Here a CTA reduces 32 independent
// reductions at a time: A (M = 128 rows = 32 reductions x 4 components,
// K = the B records of each reduction) is staged in shared memory in the
// canonical K-major no-swizzle UMMA layout (core matrix = 8 rows x 4
// records; the producers scatter each float4 with a bank-conflict-free
// component rotation) and multiplied by an all-ones B (K x 16) into an fp32
// accumulator in TMEM: D[4r + c][*] = sum_t x[r][t][c].
// Error compensation: every fp32 value is split on the CUDA cores into tf32
// hi (mantissa truncated to 10 bits) and lo = x - hi, both staged, both
// multiplied into the same accumulator (kind::tf32), so the result carries
// ~22 significant bits per term and fp32 accumulation (1e-6 of sum|x|).
//
// Pipeline per CTA (persistent over 32-reduction tiles): the 128 threads load
// a 32-record chunk (coalesced 16-byte loads), split it and store hi/lo into
// one of two smem stages; thread 0 issues 8 tcgen05.mma (4 k-steps x hi/lo)
// and commits them to the stage's mbarrier, which the producers wait on
// before refilling that stage.  After the last chunk every warp reads its 32
// TMEM lanes (tcgen05.ld 32x32b) and stores 32 sums.
#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include "dock_launch.h"

namespace mdr {
namespace tc05 {

constexpr int kThreads = 128;
constexpr int kRedPerTile = 32;   // M = 128 rows
constexpr int kChunk = 32;        // records per stage
constexpr int kN = 16;            // ones columns (minimum N for M = 128)
constexpr int kStageBytes = kRedPerTile * kChunk * 16;  // 16 KB per term

struct __align__(16) Smem {
  float hi[2][kRedPerTile * kChunk * 4];  // 2 stages x 16 KB
  float lo[2][kRedPerTile * kChunk * 4];  // 2 stages x 16 KB
  float ones[kN * 8];                     // B: N=16 x K=8, K-major core matrices
  uint64_t mbar[2];
  uint32_t tmem_base;
};

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

// SM100 shared-memory matrix descriptor (cute::UMMA::SmemDescriptor):
// [0,14) start>>4, [16,30) LBO>>4, [32,46) SBO>>4, [46,48) version=1,
// [61,64) layout (0 = SWIZZLE_NONE).
__device__ __forceinline__ uint64_t make_desc(uint32_t addr, uint32_t lbo, uint32_t sbo) {
  uint64_t d = 0;
  d |= (uint64_t)((addr >> 4) & 0x3FFFu);
  d |= (uint64_t)((lbo >> 4) & 0x3FFFu) << 16;
  d |= (uint64_t)((sbo >> 4) & 0x3FFFu) << 32;
  d |= (uint64_t)1 << 46;
  return d;
}

// Instruction descriptor (cute::UMMA::InstrDescriptor) for kind::tf32:
// c_format F32 (bits 4-5 = 1), a/b format TF32 (2), A MN-major (bit 15),
// B K-major, N>>3 at bit 17, M>>4 at bit 24.
__device__ __forceinline__ uint32_t make_idesc() {
  uint32_t d = 0;
  d |= 1u << 4;           // D fp32
  d |= 2u << 7;           // A tf32
  d |= 2u << 10;          // B tf32
  // A and B K-major (bits 15/16 = 0; the MN-major tf32 A variant returned
  // zeros on B200, tools/tc05_probe.cu)
  d |= (uint32_t)(kN >> 3) << 17;
  d |= (uint32_t)(128 >> 4) << 24;
  return d;
}

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(count));
}

__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t phase) {
  const uint32_t a = smem_u32(bar);
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra WAIT_%=;\n"
      "}\n" ::"r"(a),
      "r"(phase));
}

__device__ __forceinline__ void mma_tf32(uint32_t d_tmem, uint64_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "setp.ne.b32 p, %4, 0;\n"
      "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n"
      "}\n" ::"r"(d_tmem),
      "l"(a), "l"(b), "r"(idesc), "r"(acc));
}

__device__ __forceinline__ void commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n" ::"r"(smem_u32(bar)));
}

__device__ __forceinline__ uint32_t trunc_tf32(float x) { return __float_as_uint(x) & 0xFFFFE000u; }

// Component c (0..3, lane-dependent) of x through predicated selects: a
// ternary chain on a lane-varying index compiles to divergent branches.
__device__ __forceinline__ float sel4(float4 x, int c) {
  float a, b, r;
  asm("{\n .reg .pred p;\n setp.ne.b32 p, %3, 0;\n selp.f32 %0, %1, %2, p;\n}\n"
      : "=f"(a) : "f"(x.y), "f"(x.x), "r"(c & 1));
  asm("{\n .reg .pred p;\n setp.ne.b32 p, %3, 0;\n selp.f32 %0, %1, %2, p;\n}\n"
      : "=f"(b) : "f"(x.w), "f"(x.z), "r"(c & 1));
  asm("{\n .reg .pred p;\n setp.ne.b32 p, %3, 0;\n selp.f32 %0, %1, %2, p;\n}\n"
      : "=f"(r) : "f"(b), "f"(a), "r"(c & 2));
  return r;
}

// The 8 float4 this thread stages for chunk `ch` of the tile at r0:
// record t = 16*half + (lane & 15) of reduction r = 2*pair + (lane >> 4).
__device__ __forceinline__ void load_chunk(const float4* __restrict__ in, int B, int n_red, int r0, int ch, int warp,
                                           int lane, float4 (&xr)[8]) {
#pragma unroll
  for (int q = 0; q < 8; ++q) {
    const int combo = warp * 8 + q, pair = combo >> 1, half = combo & 1;
    const int r = 2 * pair + (lane >> 4), t = 16 * half + (lane & 15);
    xr[q] = r0 + r < n_red ? __ldcs(in + (size_t)(r0 + r) * B + ch * kChunk + t) : make_float4(0.f, 0.f, 0.f, 0.f);
  }
}

// Partial7 records (reduce7, reduce.cpp:165-209): 16 reductions per tile,
// 8 rows each (components 0..6 + a zero row).  Warp w stages reductions
// 4w..4w+3 of the chunk: per reduction 32 records x 7 floats = 224 contiguous
// floats, lane l takes floats l + 32q (q < 7), one coalesced 128-byte run
// per step.
__device__ __forceinline__ void load_chunk7(const float* __restrict__ in, int B, int n_red, int r0, int ch, int warp,
                                            int lane, float (&xr)[28]) {
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    const int r = 4 * warp + j;
    const float* src = in + ((size_t)(r0 + r) * B + (size_t)ch * kChunk) * 7;
#pragma unroll
    for (int q = 0; q < 7; ++q) xr[7 * j + q] = r0 + r < n_red ? __ldcs(src + lane + 32 * q) : 0.f;
  }
}

// NC = 4: float4 records, 32 reductions x 4 rows per 128-row tile.
// NC = 7: Partial7 records, 16 reductions x 8 rows (row 7 stays zero).
// A row = rows_per_reduction * r + c sits in the K-major core-matrix layout
// at (row / 8) * 256 + (t / 4) * 32 + (row % 8) * 4 + t % 4 floats.
template <int NC>
__global__ void __launch_bounds__(kThreads, 1)
    reduce_tc05_kernel(const float* __restrict__ in_f, int B, int n_red, float* __restrict__ out) {
  constexpr int kRpt = NC == 4 ? kRedPerTile : kRedPerTile / 2;  // reductions per 128-row tile
  extern __shared__ __align__(1024) unsigned char raw[];
  Smem& sm = *reinterpret_cast<Smem*>(raw);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const float4* in = reinterpret_cast<const float4*>(in_f);

  if (warp == 0) {  // TMEM: 32 columns (D uses 16)
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 32;\n" ::"r"(smem_u32(&sm.tmem_base)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n");
  }
  if (tid == 0) {
    mbar_init(&sm.mbar[0], 1);
    mbar_init(&sm.mbar[1], 1);
    asm volatile("fence.mbarrier_init.release.cluster;\n");
  }
  for (int i = tid; i < kN * 8; i += kThreads) sm.ones[i] = 1.0f;
  if (NC == 7)  // the padding rows (component 7) are never written: zero them once
    for (int i = tid; i < 2 * kRedPerTile * kChunk * 4; i += kThreads) {
      (&sm.hi[0][0])[i] = 0.f;
      (&sm.lo[0][0])[i] = 0.f;
    }
  asm volatile("fence.proxy.async.shared::cta;\n");
  asm volatile("tcgen05.fence::before_thread_sync;\n");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;\n");
  const uint32_t tmem = sm.tmem_base;
  const uint32_t idesc = make_idesc();
  // B = ones, K-major: core matrix = 8 N-rows x 16 B; 2 N-groups (SBO) x 2
  // K-groups (LBO); every element is 1.0 so strides only need to be valid.
  const uint64_t bdesc = make_desc(smem_u32(sm.ones), 128, 256);

  uint32_t phase[2] = {0u, 0u};
  int uses[2] = {0, 0};
  float4 xr[NC == 4 ? 8 : 1];
  float xs[NC == 7 ? 28 : 1];
  bool have = false;
  const int n_tiles = (n_red + kRpt - 1) / kRpt;
  const int chunks = B / kChunk;
  auto load = [&](int r0, int ch) {
    if constexpr (NC == 4)
      load_chunk(in, B, n_red, r0, ch, warp, lane, xr);
    else
      load_chunk7(in_f, B, n_red, r0, ch, warp, lane, xs);
  };
  for (int tile = blockIdx.x; tile < n_tiles; tile += gridDim.x) {
    const int r0 = tile * kRpt;
    for (int ch = 0; ch < chunks; ++ch) {
      const int s = ch & 1;
      if (uses[s] > 0) {  // previous MMAs reading stage s must be done
        mbar_wait(&sm.mbar[s], phase[s]);
        phase[s] ^= 1u;
      }
      if (!have) load(r0, ch);
      have = false;
      if constexpr (NC == 4) {
        // 32 reductions x 32 records = 1024 float4 per chunk, 8 per thread.
        // Lane l holds record t = 16*half + (l & 15) of reduction
        // r = 2*pair + (l >> 4): two coalesced 256-byte runs per warp.  The
        // K-major core-matrix position of component c is
        //   pair*1024 + (t/4)*128 + (4*(l>>4) + c)*16 + (t%4)*4  bytes,
        // and storing component (c0 + s) % 4 at step s (c0 = (l>>2)&3) makes
        // the 32 lanes hit 32 distinct banks.
        const int c0 = (lane >> 2) & 3;
#pragma unroll
        for (int q = 0; q < 8; ++q) {
          const int combo = warp * 8 + q, pair = combo >> 1, half = combo & 1;
          const int t = 16 * half + (lane & 15);
          const float4 x = xr[q];
          const int base = pair * 256 + (t >> 2) * 32 + 4 * (lane >> 4) * 4 + (t & 3);  // in floats
#pragma unroll
          for (int st = 0; st < 4; ++st) {
            const int c = (c0 + st) & 3;
            const float v = sel4(x, c);
            const float h = __uint_as_float(trunc_tf32(v));
            sm.hi[s][base + c * 4] = h;
            sm.lo[s][base + c * 4] = v - h;
          }
        }
      } else {
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          const int r = 4 * warp + j;
#pragma unroll
          for (int q = 0; q < 7; ++q) {
            const int f = lane + 32 * q, t = f / 7, c = f - 7 * t;
            const int at = r * 256 + (t >> 2) * 32 + c * 4 + (t & 3);
            const float v = xs[7 * j + q];
            const float h = __uint_as_float(trunc_tf32(v));
            sm.hi[s][at] = h;
            sm.lo[s][at] = v - h;
          }
        }
      }
      // prefetch the next chunk (this tile's or the next tile's first) so
      // its HBM latency overlaps the barrier and the MMA issue
      if (ch + 1 < chunks) {
        load(r0, ch + 1);
        have = true;
      } else if (tile + (int)gridDim.x < n_tiles) {
        load(r0 + (int)gridDim.x * kRpt, 0);
        have = true;
      }
      asm volatile("fence.proxy.async.shared::cta;\n");
      __syncthreads();
      if (tid == 0) {
        asm volatile("tcgen05.fence::after_thread_sync;\n");
        const uint32_t ah = smem_u32(sm.hi[s]), al = smem_u32(sm.lo[s]);
#pragma unroll
        for (int k = 0; k < kChunk / 8; ++k) {
          // A: K-major, core matrix = 8 rows x 4 records (128 B); next
          // 4-record group +128 B (LBO), next 8 rows +1024 B (SBO); one MMA
          // (K = 8) spans two groups -> +256 B per k-step
          const uint64_t dh = make_desc(ah + k * 256, 128, 1024);
          const uint64_t dl = make_desc(al + k * 256, 128, 1024);
          mma_tf32(tmem, dh, bdesc, idesc, (ch > 0 || k > 0) ? 1u : 0u);
          mma_tf32(tmem, dl, bdesc, idesc, 1u);
        }
        commit(&sm.mbar[s]);
      }
      uses[s]++;
    }
    // all MMAs of this tile have completed once the last stage's barrier flips
    const int last = (chunks - 1) & 1;
    mbar_wait(&sm.mbar[last], phase[last]);
    phase[last] ^= 1u;
    uses[last] = 0;
    if (chunks > 1) {  // the other stage's commit is older: consume its phase too
      const int other = last ^ 1;
      mbar_wait(&sm.mbar[other], phase[other]);
      phase[other] ^= 1u;
      uses[other] = 0;
    }
    asm volatile("tcgen05.fence::after_thread_sync;\n");
    uint32_t v;
    const uint32_t taddr = tmem + ((uint32_t)(warp * 32) << 16);
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x1.b32 {%0}, [%1];\n" : "=r"(v) : "r"(taddr));
    asm volatile("tcgen05.wait::ld.sync.aligned;\n");
    const int row = warp * 32 + lane;
    if constexpr (NC == 4) {  // row = 4 * reduction + component
      if (r0 + (row >> 2) < n_red) out[(size_t)r0 * 4 + row] = __uint_as_float(v);
    } else {  // row = 8 * reduction + component
      const int r = row >> 3, c = row & 7;
      if (c < 7 && r0 + r < n_red) out[(size_t)(r0 + r) * 7 + c] = __uint_as_float(v);
    }
    asm volatile("tcgen05.fence::before_thread_sync;\n");
    __syncthreads();  // D is overwritten by the next tile's first MMA
  }
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 32;\n" ::"r"(tmem));
}


// ---------------------------------------------------------------------------
// K2t2: the same contraction fed by TMA.  Raw 16 KB chunks (32 reductions x
// 32 float4 records) arrive by bulk copies (cp.async.bulk, one per
// reduction: 512 contiguous bytes) into a 6-deep shared-memory ring; thread 0
// keeps the ring full ahead of the consumers (an mbarrier per slot with a
// transaction count for "full", an arrival count of 128 for "empty").  The
// 128 threads transpose / split each chunk from the ring into the tf32
// hi/lo UMMA stages exactly as K2t does, then thread 0 issues the 8 MMAs.
// Up to 96 KB of input is in flight per SM (K2t: one 16 KB chunk per CTA in
// registers), which is what the HBM stream needs.
#ifndef MDR_TC05_RAW
#define MDR_TC05_RAW 3
#endif
#ifndef MDR_TC05_MMA
#define MDR_TC05_MMA 4
#endif
constexpr int kRawStages = MDR_TC05_RAW;
constexpr int kAcc = 4;  // independent TMEM accumulators
#ifndef MDR_TC05_WARPS
#define MDR_TC05_WARPS 16
#endif
constexpr int kTmaWarps = MDR_TC05_WARPS;  // transpose/split warps (4, 8 or 16)
constexpr int kTmaThreads = 32 * kTmaWarps;
constexpr int kMmaStages = MDR_TC05_MMA;
constexpr int kChunkBytes = kRedPerTile * kChunk * 16;  // one 32 x 32 float4 box

struct __align__(128) SmemTma {
  float4 raw[kRawStages][kRedPerTile * kChunk];  // [slot][r * 32 + t]
  float hi[kMmaStages][kRedPerTile * kChunk * 4];
  float lo[kMmaStages][kRedPerTile * kChunk * 4];
  float ones[kN * 8];
  uint64_t full[kRawStages], empty[kRawStages], mbar[kMmaStages];
  uint32_t tmem_base;
};

__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(bytes));
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(smem_u32(bar)));
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(
                   smem_u32(dst)),
               "l"(src), "r"(bytes), "r"(smem_u32(bar))
               : "memory");
}

__device__ __forceinline__ void tma_2d(void* dst, const void* tmap, int x, int y, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];\n" ::
          "r"(smem_u32(dst)),
      "l"(tmap), "r"(x), "r"(y), "r"(smem_u32(bar))
      : "memory");
}

// tmap: 2D tensor map over the input viewed as n_red rows of 4 B floats
// (inner dimension B * 4 floats), box = 32 records (128 floats) x 32 rows;
// rows beyond n_red are zero-filled by the TMA unit.
__global__ void __launch_bounds__(kTmaThreads, 1)
    reduce4_tc05_tma_kernel(const __grid_constant__ CUtensorMap tmap, int B, int n_red, float* __restrict__ out) {
  extern __shared__ __align__(1024) unsigned char raw_smem[];
  SmemTma& sm = *reinterpret_cast<SmemTma*>(raw_smem);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 64;\n" ::"r"(smem_u32(&sm.tmem_base)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n");
  }
  if (tid == 0) {
    for (int i = 0; i < kRawStages; ++i) {
      mbar_init(&sm.full[i], 1);
      mbar_init(&sm.empty[i], kTmaThreads);
    }
    for (int i = 0; i < kMmaStages; ++i) mbar_init(&sm.mbar[i], 1);
    asm volatile("fence.mbarrier_init.release.cluster;\n");
  }
  for (int i = tid; i < kN * 8; i += kTmaThreads) sm.ones[i] = 1.0f;
  asm volatile("fence.proxy.async.shared::cta;\n");
  asm volatile("tcgen05.fence::before_thread_sync;\n");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;\n");
  const uint32_t tmem = sm.tmem_base;
  const uint32_t idesc = make_idesc();
  const uint64_t bdesc = make_desc(smem_u32(sm.ones), 128, 256);
  const int n_tiles = (n_red + kRedPerTile - 1) / kRedPerTile;
  const int chunks = B / kChunk;
  const int my_tiles = blockIdx.x < n_tiles ? (n_tiles - 1 - (int)blockIdx.x) / (int)gridDim.x + 1 : 0;
  const long long total = (long long)my_tiles * chunks;  // chunks this CTA consumes
  long long issued = 0;
  // producer: chunk q of this CTA -> ring slot q % kRawStages (thread 0)
  auto issue = [&](long long q) {
    const int slot = (int)(q % kRawStages);
    if (q >= kRawStages) mbar_wait(&sm.empty[slot], (uint32_t)(((q / kRawStages) - 1) & 1));
    const int tile = (int)blockIdx.x + (int)(q / chunks) * (int)gridDim.x, ch = (int)(q % chunks);
    mbar_expect_tx(&sm.full[slot], (uint32_t)kChunkBytes);  // out-of-range rows arrive zero-filled
    tma_2d(&sm.raw[slot][0], &tmap, ch * kChunk * 4, tile * kRedPerTile, &sm.full[slot]);
  };
  uint32_t phase[kMmaStages] = {};
  int uses[kMmaStages] = {};
  long long g = 0;
  for (int tile = blockIdx.x; tile < n_tiles; tile += gridDim.x) {
    const int r0 = tile * kRedPerTile;
    for (int ch = 0; ch < chunks; ++ch, ++g) {
      if (tid == 0)
        for (; issued < total && issued <= g + kRawStages - 1; ++issued) issue(issued);
      const int slot = (int)(g % kRawStages);
      mbar_wait(&sm.full[slot], (uint32_t)((g / kRawStages) & 1));
      const int s = (int)(g % kMmaStages);
      if (uses[s] > 0) {  // previous MMAs reading stage s must be done
        mbar_wait(&sm.mbar[s], phase[s]);
        phase[s] ^= 1u;
      }
      const int c0 = (lane >> 2) & 3;
#pragma unroll
      for (int q = 0; q < 32 / kTmaWarps; ++q) {
        const int combo = warp * (32 / kTmaWarps) + q, pair = combo >> 1, half = combo & 1;
        const int r = 2 * pair + (lane >> 4), t = 16 * half + (lane & 15);
        const float4 x = sm.raw[slot][r * kChunk + t];
        const int base = pair * 256 + (t >> 2) * 32 + 4 * (lane >> 4) * 4 + (t & 3);  // in floats
#pragma unroll
        for (int st = 0; st < 4; ++st) {
          const int c = (c0 + st) & 3;
          const float v = sel4(x, c);
          const float h = __uint_as_float(trunc_tf32(v));
          sm.hi[s][base + c * 4] = h;
          sm.lo[s][base + c * 4] = v - h;
        }
      }
      mbar_arrive(&sm.empty[slot]);  // this thread is done with the raw slot
      asm volatile("fence.proxy.async.shared::cta;\n");
      __syncthreads();
      if (tid == 0) {
        asm volatile("tcgen05.fence::after_thread_sync;\n");
        const uint32_t ah = smem_u32(sm.hi[s]), al = smem_u32(sm.lo[s]);
#pragma unroll
        for (int k = 0; k < kChunk / 8; ++k) {
          const uint64_t dh = make_desc(ah + k * 256, 128, 1024);
          const uint64_t dl = make_desc(al + k * 256, 128, 1024);
          // kAcc independent accumulators (16 TMEM columns each): the MMAs of
          // consecutive chunks do not serialise on one D
          const uint32_t d = tmem + (uint32_t)((ch % kAcc) * kN);
          mma_tf32(d, dh, bdesc, idesc, (ch >= kAcc || k > 0) ? 1u : 0u);
          mma_tf32(d, dl, bdesc, idesc, 1u);
        }
        commit(&sm.mbar[s]);
      }
      uses[s]++;
    }
    for (int st = 0; st < kMmaStages; ++st)  // every outstanding commit of this tile
      if (uses[st] > 0) {
        mbar_wait(&sm.mbar[st], phase[st]);
        phase[st] ^= 1u;
        uses[st] = 0;
      }
    asm volatile("tcgen05.fence::after_thread_sync;\n");
    if (warp < 4) {  // TMEM lane quadrant w % 4: warps 0..3 read the 128 rows
      float acc = 0.f;
      const int nacc = chunks < kAcc ? chunks : kAcc;
      for (int q = 0; q < nacc; ++q) {  // fixed order: deterministic
        uint32_t v;
        const uint32_t taddr = tmem + ((uint32_t)(warp * 32) << 16) + (uint32_t)(q * kN);
        asm volatile("tcgen05.ld.sync.aligned.32x32b.x1.b32 {%0}, [%1];\n" : "=r"(v) : "r"(taddr));
        asm volatile("tcgen05.wait::ld.sync.aligned;\n");
        acc += __uint_as_float(v);
      }
      const int row = warp * 32 + lane;
      if (r0 + (row >> 2) < n_red) out[(size_t)r0 * 4 + row] = acc;
    }
    asm volatile("tcgen05.fence::before_thread_sync;\n");
    __syncthreads();
  }
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 64;\n" ::"r"(tmem));
}

}  // namespace tc05

template <int NC>
static cudaError_t launch_tc05(const float* in, int B, int n_red, float* out, int ctas_per_sm, cudaStream_t s) {
  if (n_red <= 0) return cudaSuccess;
  const size_t smem = sizeof(tc05::Smem) + 1024;
  cudaError_t e = cudaFuncSetAttribute(tc05::reduce_tc05_kernel<NC>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       (int)smem);
  if (e != cudaSuccess) return e;
  const int rpt = NC == 4 ? tc05::kRedPerTile : tc05::kRedPerTile / 2;
  const int tiles = (n_red + rpt - 1) / rpt;
  int grid = 148 * ctas_per_sm;
  if (grid > tiles) grid = tiles;
  tc05::reduce_tc05_kernel<NC><<<grid, tc05::kThreads, smem, s>>>(in, B, n_red, out);
  return cudaGetLastError();
}

cudaError_t launch_reduce4_tc05(const float* in, int B, int n_red, float* out, int ctas_per_sm, cudaStream_t s) {
  return launch_tc05<4>(in, B, n_red, out, ctas_per_sm, s);
}
cudaError_t launch_reduce7_tc05(const float* in, int B, int n_red, float* out, int ctas_per_sm, cudaStream_t s) {
  return launch_tc05<7>(in, B, n_red, out, ctas_per_sm, s);
}

// cuTensorMapEncodeTiled through the runtime's driver entry point (no -lcuda)
typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                  const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                  CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

cudaError_t launch_reduce4_tc05_tma(const float* in, int B, int n_red, float* out, cudaStream_t s) {
  static EncodeTiledFn encode = nullptr;
  if (!encode) {
    void* fn = nullptr;
    cudaDriverEntryPointQueryResult q;
    cudaError_t e = cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q);
    if (e != cudaSuccess || !fn) return e != cudaSuccess ? e : cudaErrorNotSupported;
    encode = reinterpret_cast<EncodeTiledFn>(fn);
  }
  CUtensorMap tmap;
  const cuuint64_t dims[2] = {(cuuint64_t)B * 4, (cuuint64_t)n_red};
  const cuuint64_t strides[1] = {(cuuint64_t)B * 16};  // bytes between rows
  const cuuint32_t box[2] = {(cuuint32_t)tc05::kChunk * 4, (cuuint32_t)tc05::kRedPerTile};
  const cuuint32_t estr[2] = {1, 1};
  if (encode(&tmap, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<float*>(in), dims, strides, box, estr,
             CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
             CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
    return cudaErrorInvalidValue;
  const size_t smem = sizeof(tc05::SmemTma) + 1024;
  cudaError_t e = cudaFuncSetAttribute(tc05::reduce4_tc05_tma_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       (int)smem);
  if (e != cudaSuccess) return e;
  const int tiles = (n_red + tc05::kRedPerTile - 1) / tc05::kRedPerTile;
  const int grid = tiles < 148 ? tiles : 148;  // one CTA per SM (160 KB of shared memory)
  tc05::reduce4_tc05_tma_kernel<<<grid, tc05::kTmaThreads, smem, s>>>(tmap, B, n_red, out);
  return cudaGetLastError();
}

}  // namespace mdr
