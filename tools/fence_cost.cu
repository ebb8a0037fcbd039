// Cost of the system-scope fences in a one-thread barrier kernel (dev tool):
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/fence_cost tools/fence_cost.cu
#include <cstdio>
#include <cuda_runtime.h>
__device__ __forceinline__ void st_release_sys(unsigned* p, unsigned v) {
  asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ unsigned ld_acquire_sys(const unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
template <int MODE>
__global__ void kb(unsigned* flag, unsigned epoch) {
  if (threadIdx.x) return;
  if (MODE & 1) __threadfence_system();
  st_release_sys(flag, epoch);
  while ((int)(ld_acquire_sys(flag) - epoch) < 0) __nanosleep(256);
  if (MODE & 2) __threadfence_system();
}
__global__ void kw(float* x, int n) {  // a writer kernel before the barrier
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) x[i] += 1.f;
}
int main() {
  unsigned* flag; float* x;
  cudaMalloc(&flag, 4); cudaMemset(flag, 0, 4);
  const int n = 1 << 20;
  cudaMalloc(&x, n * 4);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  unsigned ep = 0;
  for (int mode = 0; mode < 4; ++mode) {
    for (int rep = 0; rep < 2; ++rep) {
      cudaDeviceSynchronize();
      cudaEventRecord(a);
      for (int i = 0; i < 100; ++i) {
        kw<<<n / 256, 256>>>(x, n);
        switch (mode) {
          case 0: kb<0><<<1, 32>>>(flag, ++ep); break;
          case 1: kb<1><<<1, 32>>>(flag, ++ep); break;
          case 2: kb<2><<<1, 32>>>(flag, ++ep); break;
          default: kb<3><<<1, 32>>>(flag, ++ep); break;
        }
      }
      cudaEventRecord(b);
      cudaEventSynchronize(b);
      float ms; cudaEventElapsedTime(&ms, a, b);
      if (rep) printf("mode %d (lead fence %d, trail fence %d): %.2f us per writer+barrier\n", mode, mode & 1, (mode >> 1) & 1, ms * 10);
    }
  }
  cudaDeviceSynchronize();
  cudaEventRecord(a);
  for (int i = 0; i < 100; ++i) kw<<<n / 256, 256>>>(x, n);
  cudaEventRecord(b); cudaEventSynchronize(b);
  float ms; cudaEventElapsedTime(&ms, a, b);
  printf("writer alone: %.2f us\n", ms * 10);
  return 0;
}
