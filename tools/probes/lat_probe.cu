// Dependent-latency probe (one warp): cycles per op for FP64 fma/add, FP32 fma,
// shfl, shared load, FP64 sqrt/div/sincos.  nvcc -arch=sm_100a -O3 lat_probe.cu -o lat_probe
#include <cstdio>
#include <cuda_runtime.h>
#define N 1024
__global__ void k(double* out, float* outf, long long* cyc, double seed) {
  __shared__ double sm[64];
  int lane = threadIdx.x;
  sm[lane] = lane; sm[lane + 32] = lane;
  __syncwarp();
  double a = seed + lane * 1e-9, m = 0.9999999, c = 1e-7;
  float fa = (float)a, fm = 0.9999f, fc = 1e-5f;
  long long t0, t1;
  t0 = clock64(); for (int i = 0; i < N; ++i) a = fma(a, m, c); t1 = clock64(); cyc[0] = t1 - t0;
  t0 = clock64(); for (int i = 0; i < N; ++i) a = a + c; t1 = clock64(); cyc[1] = t1 - t0;
  t0 = clock64(); for (int i = 0; i < N; ++i) fa = fmaf(fa, fm, fc); t1 = clock64(); cyc[2] = t1 - t0;
  t0 = clock64(); for (int i = 0; i < N; ++i) fa = __shfl_xor_sync(0xffffffff, fa, 1) + fc; t1 = clock64(); cyc[3] = t1 - t0;
  int idx = lane;
  t0 = clock64(); for (int i = 0; i < N; ++i) { idx = (int)sm[idx & 63] ; } t1 = clock64(); cyc[4] = t1 - t0;
  t0 = clock64(); for (int i = 0; i < N; ++i) a = sqrt(a) + 1.0; t1 = clock64(); cyc[5] = t1 - t0;
  t0 = clock64(); for (int i = 0; i < N; ++i) a = 3.0 / a + 1.0; t1 = clock64(); cyc[6] = t1 - t0;
  double s, co;
  t0 = clock64(); for (int i = 0; i < N; ++i) { sincos(a, &s, &co); a = s + co; } t1 = clock64(); cyc[7] = t1 - t0;
  t0 = clock64(); for (int i = 0; i < N; ++i) { double y; asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(a)); a = y + 1.0; } t1 = clock64(); cyc[8] = t1 - t0;
  t0 = clock64(); for (int i = 0; i < N; ++i) a = a * m; t1 = clock64(); cyc[9] = t1 - t0;
  t0 = clock64(); for (int i = 0; i < N; ++i) fa = fa + fc; t1 = clock64(); cyc[10] = t1 - t0;
  t0 = clock64(); for (int i = 0; i < N; ++i) a = (double)(float)a + c; t1 = clock64(); cyc[11] = t1 - t0;
  t0 = clock64(); for (int i = 0; i < N; ++i) a = floor(a) + 0.5; t1 = clock64(); cyc[12] = t1 - t0;
  out[lane] = a + idx; outf[lane] = fa;
}
int main() {
  double* o; float* of; long long* c;
  cudaMalloc(&o, 256); cudaMalloc(&of, 256); cudaMallocManaged(&c, 16 * 8);
  for (int r = 0; r < 2; ++r) { k<<<1, 32>>>(o, of, c, 0.5); cudaDeviceSynchronize(); }
  const char* nm[] = {"dfma", "dadd", "ffma", "shfl+fadd", "lds.f64->idx", "dsqrt+dadd", "ddiv+dadd", "sincos+dadd", "rcp64h+dadd", "dmul", "fadd", "f2f64 roundtrip+dadd", "floor+dadd"};
  for (int i = 0; i < 13; ++i) printf("%-22s %.1f cycles\n", nm[i], (double)c[i] / N);
  return 0;
}
