// Does compute-sanitizer racecheck model mbarrier synchronisation?
// Warp 0 writes shared memory and arrives on an mbarrier; warp 1 waits
// (mode 0: try_wait.parity without arriving, the item-pool protocol of
// ls_multi.cu; mode 1: arrives itself and waits on its token) and reads.
// Mode 2: the reverse (warp 1 reads, arrives; warp 0 waits, then writes).
// Mode 3: ten rounds of full / empty ping-pong on two barriers (parity
// waits), warp 0 writing, warp 1 reading.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -o /tmp/mbp mbar_race_probe.cu
// Run:   compute-sanitizer --tool racecheck /tmp/mbp 0 ; ... /tmp/mbp 1
#include <cstdio>
#include <cstdlib>

__device__ __forceinline__ unsigned sa(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }

__device__ __forceinline__ void arrive(unsigned long long* b) {
  unsigned long long st;
  asm volatile("mbarrier.arrive.shared::cta.b64 %0, [%1];" : "=l"(st) : "r"(sa(b)) : "memory");
}
__device__ __forceinline__ void wait_parity(unsigned long long* b, int ph) {
  unsigned ok = 0;
  do {
    asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
                 : "=r"(ok) : "r"(sa(b)), "r"(ph) : "memory");
  } while (!ok);
}

__global__ void k2(int mode, int* out) {
  __shared__ __align__(8) unsigned long long full, empty;
  __shared__ int data[32];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(sa(&full)), "r"(32) : "memory");
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(sa(&empty)), "r"(32) : "memory");
    data[0] = 0;
  }
  __syncthreads();
  if (mode == 2) {
    if (warp == 1) {
      out[lane] = data[lane == 0 ? 0 : 0];
      arrive(&empty);
    } else {
      wait_parity(&empty, 0);
      data[lane] = lane;
    }
    return;
  }
  int acc = 0;
  for (int it = 0; it < 10; ++it) {
    if (warp == 0) {
      if (it > 0) wait_parity(&empty, (it - 1) & 1);
      data[lane] = it * 100 + lane;
      arrive(&full);
    } else {
      wait_parity(&full, it & 1);
      acc += data[31 - lane];
      arrive(&empty);
    }
  }
  if (warp == 1) out[lane] = acc;
}

__global__ void k(int mode, int* out) {
  __shared__ __align__(8) unsigned long long bar;
  __shared__ int data[32];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0)
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(sa(&bar)), "r"(mode ? 64 : 32) : "memory");
  __syncthreads();
  unsigned long long st = 0;
  if (warp == 0) {
    data[lane] = lane * 3 + 1;
    asm volatile("mbarrier.arrive.shared::cta.b64 %0, [%1];" : "=l"(st) : "r"(sa(&bar)) : "memory");
  } else {
    unsigned ok = 0;
    if (mode == 0) {
      do {
        asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
                     : "=r"(ok) : "r"(sa(&bar)), "r"(0) : "memory");
      } while (!ok);
    } else {
      asm volatile("mbarrier.arrive.shared::cta.b64 %0, [%1];" : "=l"(st) : "r"(sa(&bar)) : "memory");
      do {
        asm volatile("{ .reg .pred p; mbarrier.try_wait.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
                     : "=r"(ok) : "r"(sa(&bar)), "l"(st) : "memory");
      } while (!ok);
    }
    out[lane] = data[lane];
  }
}

int main(int argc, char** argv) {
  const int mode = argc > 1 ? atoi(argv[1]) : 0;
  int* d;
  cudaMalloc(&d, 128);
  if (mode >= 2)
    k2<<<1, 64>>>(mode, d);
  else
    k<<<1, 64>>>(mode, d);
  int h[32];
  cudaMemcpy(h, d, 128, cudaMemcpyDeviceToHost);
  printf("mode %d: out[5] = %d (expect 16), %s\n", mode, h[5], cudaGetErrorString(cudaGetLastError()));
  return 0;
}
