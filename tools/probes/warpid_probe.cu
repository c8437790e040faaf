// Which hardware warp slot (%warpid; SMSP = warpid % 4) do the warps of
// 128-thread CTAs get?  nvcc -gencode arch=compute_100a,code=sm_100a -O3 warpid_probe.cu -o warpid_probe
#include <cstdio>
__global__ void k(int* out) {
  unsigned w, sm;
  asm volatile("mov.u32 %0, %%warpid;" : "=r"(w));
  asm volatile("mov.u32 %0, %%smid;" : "=r"(sm));
  long long t0 = clock64();
  while (clock64() - t0 < 200000) {}
  if ((threadIdx.x & 31) == 0) {
    out[(blockIdx.x * 4 + threadIdx.x / 32) * 2] = sm;
    out[(blockIdx.x * 4 + threadIdx.x / 32) * 2 + 1] = w;
  }
}
int main() {
  int* o; const int blocks = 450;
  cudaMallocManaged(&o, blocks * 4 * 2 * 4);
  k<<<blocks, 128>>>(o);
  cudaDeviceSynchronize();
  int same = 0, pairs = 0;
  for (int b = 0; b < 12; ++b) {
    printf("block %d: sm %d warps", b, o[b * 8]);
    for (int j = 0; j < 4; ++j) printf(" %d", o[(b * 4 + j) * 2 + 1]);
    printf("\n");
  }
  for (int b = 0; b < blocks; ++b)
    for (int p = 0; p < 2; ++p) {
      ++pairs;
      same += (o[(b * 4 + 2 * p) * 2 + 1] % 4) == (o[(b * 4 + 2 * p + 1) * 2 + 1] % 4);
    }
  printf("warp pairs (2p, 2p+1) on the same warpid%%4: %d of %d\n", same, pairs);
  return 0;
}
