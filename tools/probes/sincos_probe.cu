// Prints inputs where sincos_fast differs from libdevice sincos.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 --fmad=false -I../../include -I../../paper_2410_10447_b200/csrc sincos_probe.cu -o sincos_probe
#include <cstdio>
#include "mdr_device.cuh"
using namespace mdr;
__global__ void k(unsigned long long* cnt, double* bad) {
  long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  for (int rep = 0; rep < 64; ++rep, i += (long long)gridDim.x * blockDim.x) {
    const uint64_t r1 = mix64(777 + (uint64_t)i + 1);
    double a;
    int cls;
    if (i & 1) {
      const double m = 1.0 + (double)(r1 >> 12) * 0x1p-52;
      a = ldexp((r1 & 2048) ? -m : m, (int)((r1 >> 1) & 63) - 31);
      cls = 1;
    } else {
      a = -kPi + 2.0 * kPi * ((double)(r1 >> 11) * 0x1p-53);
      cls = 0;
    }
    double s1, c1, s2, c2;
    sincos_fast(a, &s1, &c1);
    sincos(a, &s2, &c2);
    if (__double_as_longlong(s1) != __double_as_longlong(s2) || __double_as_longlong(c1) != __double_as_longlong(c2)) {
      unsigned long long k = atomicAdd(&cnt[cls], 1ull);
      if (cls == 0 && k < 8) { bad[6 * k] = a; bad[6*k+1] = s1; bad[6*k+2] = s2; bad[6*k+3] = c1; bad[6*k+4] = c2; }
      if (cls == 1 && k < 8) { bad[48 + 6 * k] = a; bad[48+6*k+1] = s1; bad[48+6*k+2] = s2; bad[48+6*k+3] = c1; bad[48+6*k+4] = c2; }
    }
  }
}
int main() {
  unsigned long long* c; double* b;
  cudaMallocManaged(&c, 16); cudaMallocManaged(&b, 96 * 8);
  c[0] = c[1] = 0;
  k<<<1184, 256>>>(c, b);
  cudaDeviceSynchronize();
  printf("mismatches: angle class %llu, magnitude class %llu (of %d each)\n", c[0], c[1], 1184 * 256 * 32);
  for (int cls = 0; cls < 2; ++cls)
    for (int j = 0; j < 8 && j < (int)c[cls]; ++j) {
      double* r = b + 48 * cls + 6 * j;
      printf("a=%.17g s_fast=%.17g s_lib=%.17g c_fast=%.17g c_lib=%.17g\n", r[0], r[1], r[2], r[3], r[4]);
    }
  return 0;
}
