// tc05_probe.cu — standalone probe of the tcgen05 kind::tf32 ones-matrix
// contraction (one CTA, one 128x16x8 MMA), to pin the A-operand layout.
// Build/run on the GPU box:
//   nvcc -gencode arch=compute_100a,code=sm_100a -o /tmp/probe tools/tc05_probe.cu && /tmp/probe
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t su(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint64_t desc(uint32_t addr, uint32_t lbo, uint32_t sbo) {
  return (uint64_t)((addr >> 4) & 0x3FFFu) | ((uint64_t)((lbo >> 4) & 0x3FFFu) << 16) |
         ((uint64_t)((sbo >> 4) & 0x3FFFu) << 32) | ((uint64_t)1 << 46);
}

// mode 0: A MN-major (4 comps contiguous per record, records 16 B apart)
// mode 1: A K-major  (core matrix 8 rows x 4 k, row stride 16 B)
__global__ void probe(int mode, const float* a_in /*128 x 8 logical A[m][k]*/, float* out /*128*/) {
  __shared__ __align__(1024) float A[128 * 8];
  __shared__ __align__(128) float ones[16 * 8];
  __shared__ __align__(8) uint64_t bar;
  __shared__ uint32_t tbase;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 32;" ::"r"(su(&tbase)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (tid == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su(&bar)));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  for (int i = tid; i < 128; i += blockDim.x) ones[i] = 1.0f;
  // place logical A[m][k] (m < 128, k < 8)
  for (int idx = tid; idx < 128 * 8; idx += blockDim.x) {
    const int m = idx / 8, k = idx % 8;
    int off;
    if (mode == 0) {  // MN-major: element (m,k) at (m/4)*SBO + k*16 B + (m%4)*4 B ; SBO = 128 B
      off = (m / 4) * 32 + k * 4 + (m % 4);
    } else {  // K-major: core (mg = m/8, kg = k/4): mg*SBO + kg*LBO + (m%8)*16 B + (k%4)*4 B ; LBO=128 B, SBO=256 B
      off = (m / 8) * 64 + (k / 4) * 32 + (m % 8) * 4 + (k % 4);
    }
    A[off] = a_in[idx];
  }
  asm volatile("fence.proxy.async.shared::cta;");
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tm = tbase;
  if (tid == 0) {
    uint32_t idesc = (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(mode == 0) << 15) | ((16u >> 3) << 17) |
                     ((128u >> 4) << 24);
    const uint64_t ad = mode == 0 ? desc(su(A), 128, 128) : desc(su(A), 128, 256);
    const uint64_t bd = desc(su(ones), 128, 256);
    asm volatile(
        "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
        "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n}\n" ::"r"(tm),
        "l"(ad), "l"(bd), "r"(idesc), "r"(0));
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(su(&bar)));
  }
  asm volatile(
      "{\n.reg .pred p;\nW:\nmbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n@!p bra W;\n}\n" ::"r"(su(&bar)));
  asm volatile("tcgen05.fence::after_thread_sync;");
  uint32_t v0, v1;
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x2.b32 {%0, %1}, [%2];" : "=r"(v0), "=r"(v1) : "r"(tm + ((warp * 32) << 16)));
  asm volatile("tcgen05.wait::ld.sync.aligned;");
  out[tid * 2] = __uint_as_float(v0);
  out[tid * 2 + 1] = __uint_as_float(v1);
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 32;" ::"r"(tm));
}

int main() {
  float h[128 * 8];
  for (int m = 0; m < 128; ++m)
    for (int k = 0; k < 8; ++k) h[m * 8 + k] = (float)(m + 1) + 0.001f * k;  // row sum = 8(m+1) + 0.028
  float *d_in, *d_out;
  cudaMalloc(&d_in, sizeof h);
  cudaMalloc(&d_out, 256 * 4);
  cudaMemcpy(d_in, h, sizeof h, cudaMemcpyHostToDevice);
  for (int mode = 0; mode < 2; ++mode) {
    cudaMemset(d_out, 0, 256 * 4);
    probe<<<1, 128>>>(mode, d_in, d_out);
    cudaError_t e = cudaDeviceSynchronize();
    float o[256];
    cudaMemcpy(o, d_out, sizeof o, cudaMemcpyDeviceToHost);
    printf("mode %d (%s) err=%s\n", mode, mode == 0 ? "A MN-major" : "A K-major", cudaGetErrorString(e));
    int bad = 0;
    for (int m = 0; m < 128; ++m) {
      const float want = 8.0f * (m + 1) + 0.028f;
      if (fabsf(o[2 * m] - want) > 1e-2f * want) ++bad;
      if (m < 6 || m == 127) printf("  row %3d: col0 %.4f col1 %.4f (want %.4f)\n", m, o[2 * m], o[2 * m + 1], want);
    }
    printf("  rows wrong: %d / 128\n", bad);
  }
  return 0;
}
