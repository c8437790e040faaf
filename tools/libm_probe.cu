// How often CUDA's double sin/cos/log differ from glibc's on the hot-path
// domains: angles in [-pi, pi) (build_frame, rotate_axis) and the
// Box-Muller terms log(u1), cos(2 pi u2) of RngStream::normal (rng.cpp:47-52).
#include <cmath>
#include <cstdio>
#include <cstdint>
#include <vector>
#include <cuda_runtime.h>

__host__ __device__ inline uint64_t mix64(uint64_t z) {
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
  return z ^ (z >> 31);
}
__host__ __device__ inline double unit(uint64_t n) { return (double)(mix64(n * 0x9e3779b97f4a7c15ull) >> 11) * 0x1p-53; }

__global__ void k(int n, double* s, double* c, double* lg, double* cz) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const double a = -M_PI + 2 * M_PI * unit(4 * (uint64_t)i + 1);
  sincos(a, &s[i], &c[i]);
  const double u1 = ((mix64((4 * (uint64_t)i + 2) * 0x9e3779b97f4a7c15ull) >> 11) + 1) * 0x1p-53;
  lg[i] = log(u1);
  cz[i] = cos(2.0 * M_PI * unit(4 * (uint64_t)i + 3));
}

int main() {
  const int n = 1 << 24;
  double *s, *c, *lg, *cz;
  cudaMallocManaged(&s, n * 8); cudaMallocManaged(&c, n * 8); cudaMallocManaged(&lg, n * 8); cudaMallocManaged(&cz, n * 8);
  k<<<(n + 255) / 256, 256>>>(n, s, c, lg, cz);
  cudaDeviceSynchronize();
  long ms = 0, mc = 0, ml = 0, mz = 0;
  for (int i = 0; i < n; ++i) {
    const double a = -M_PI + 2 * M_PI * unit(4 * (uint64_t)i + 1);
    const double u1 = ((mix64((4 * (uint64_t)i + 2) * 0x9e3779b97f4a7c15ull) >> 11) + 1) * 0x1p-53;
    ms += std::sin(a) != s[i];
    mc += std::cos(a) != c[i];
    ml += std::log(u1) != lg[i];
    mz += std::cos(2.0 * M_PI * unit(4 * (uint64_t)i + 3)) != cz[i];
  }
  printf("n=%d mismatches: sin %ld cos %ld log %ld cos(2pi u) %ld  (rates %.2e %.2e %.2e %.2e)\n", n, ms, mc, ml, mz,
         (double)ms / n, (double)mc / n, (double)ml / n, (double)mz / n);
}
