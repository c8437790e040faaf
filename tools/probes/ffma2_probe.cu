// Throughput probe: scalar FFMA vs packed FFMA2 (fma.rn.f32x2, sm_100a).
// Build: nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o tools/probes/ffma2_probe tools/probes/ffma2_probe.cu
// Each thread runs 8 independent chains; reports FP32 FLOP/s for both forms.
#include <cstdio>
#include <cuda_runtime.h>

__global__ void ffma_kernel(float* out, int iters, float a, float b) {
  float x[16];
#pragma unroll
  for (int k = 0; k < 16; ++k) x[k] = threadIdx.x * 1e-3f + k;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int k = 0; k < 16; ++k) x[k] = fmaf(x[k], a, b);
  }
  float s = 0.f;
#pragma unroll
  for (int k = 0; k < 16; ++k) s += x[k];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

__global__ void ffma2_kernel(float* out, int iters, float a, float b) {
  unsigned long long x[8], A, B;
  asm("mov.b64 %0, {%1, %1};" : "=l"(A) : "f"(a));
  asm("mov.b64 %0, {%1, %1};" : "=l"(B) : "f"(b));
#pragma unroll
  for (int k = 0; k < 8; ++k) {
    float lo = threadIdx.x * 1e-3f + 2 * k, hi = lo + 1.f;
    asm("mov.b64 %0, {%1, %2};" : "=l"(x[k]) : "f"(lo), "f"(hi));
  }
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int k = 0; k < 8; ++k) asm volatile("fma.rn.f32x2 %0, %0, %1, %2;" : "+l"(x[k]) : "l"(A), "l"(B));
  }
  float s = 0.f;
#pragma unroll
  for (int k = 0; k < 8; ++k) {
    float lo, hi;
    asm("mov.b64 {%0, %1}, %2;" : "=f"(lo), "=f"(hi) : "l"(x[k]));
    s += lo + hi;
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

int main() {
  const int blocks = 148 * 8, threads = 256, iters = 1 << 14;
  float* out;
  cudaMalloc(&out, sizeof(float) * blocks * threads);
  cudaEvent_t s, e;
  cudaEventCreate(&s);
  cudaEventCreate(&e);
  for (int rep = 0; rep < 2; ++rep) {
    float ms1, ms2;
    cudaEventRecord(s);
    ffma_kernel<<<blocks, threads>>>(out, iters, 0.999f, 1e-3f);
    cudaEventRecord(e);
    cudaEventSynchronize(e);
    cudaEventElapsedTime(&ms1, s, e);
    cudaEventRecord(s);
    ffma2_kernel<<<blocks, threads>>>(out, iters, 0.999f, 1e-3f);
    cudaEventRecord(e);
    cudaEventSynchronize(e);
    cudaEventElapsedTime(&ms2, s, e);
    const double flops = 2.0 * 16 * (double)iters * blocks * threads;
    printf("FFMA  %.1f TFLOP/s   FFMA2 %.1f TFLOP/s\n", flops / ms1 / 1e9, flops / ms2 / 1e9);
  }
  // latency-bound variant: 1 warp per SMSP, 16 chains
  return 0;
}
