// NVLS multicast probe: one device, one multicast object, multimem.st from a kernel
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdint>
#define CK(x) do { CUresult r = (x); if (r != CUDA_SUCCESS) { const char* s; cuGetErrorString(r, &s); printf("FAIL %s: %d %s\n", #x, (int)r, s); return 1; } } while (0)
__global__ void k_mc_store(uint32_t* mc, int n) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n / 4) {
    uint4 v = make_uint4(4 * i, 4 * i + 1, 4 * i + 2, 4 * i + 3);
    asm volatile("multimem.st.relaxed.sys.global.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(mc + 4 * i), "r"(v.x), "r"(v.y), "r"(v.z), "r"(v.w) : "memory");
  }
}
int main() {
  CK(cuInit(0));
  CUdevice dev; CK(cuDeviceGet(&dev, 0));
  CUcontext ctx; CK(cuDevicePrimaryCtxRetain(&ctx, dev)); CK(cuCtxSetCurrent(ctx));
  int mcs = -1; cuDeviceGetAttribute(&mcs, CU_DEVICE_ATTRIBUTE_MULTICAST_SUPPORTED, dev);
  printf("multicast supported %d\n", mcs);
  CUmulticastObjectProp mp = {};
  mp.numDevices = 1; mp.size = 2 << 20; mp.handleTypes = CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR;
  size_t gran = 0; CK(cuMulticastGetGranularity(&gran, &mp, CU_MULTICAST_GRANULARITY_RECOMMENDED));
  printf("granularity %zu\n", gran);
  mp.size = (mp.size + gran - 1) / gran * gran;
  CUmemGenericAllocationHandle mc;
  {
    const unsigned long long hts[3] = {0ull, (unsigned long long)CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR, (unsigned long long)CU_MEM_HANDLE_TYPE_FABRIC};
    for (unsigned nd = 1; nd <= 2; ++nd)
      for (int h = 0; h < 3; ++h) {
        CUmulticastObjectProp q = mp; q.numDevices = nd; q.handleTypes = hts[h];
        CUmemGenericAllocationHandle t;
        CUresult r = cuMulticastCreate(&t, &q);
        const char* es; cuGetErrorString(r, &es);
        printf("cuMulticastCreate numDevices=%u handleTypes=%llu -> %d %s\n", nd, hts[h], (int)r, es);
        if (r == CUDA_SUCCESS) cuMemRelease(t);
      }
  }
  mp.handleTypes = 0;
  CK(cuMulticastCreate(&mc, &mp));
  CK(cuMulticastAddDevice(mc, dev));
  CUmemAllocationProp ap = {};
  ap.type = CU_MEM_ALLOCATION_TYPE_PINNED; ap.location.type = CU_MEM_LOCATION_TYPE_DEVICE; ap.location.id = 0;
  ap.requestedHandleTypes = CU_MEM_HANDLE_TYPE_NONE;
  CUmemGenericAllocationHandle mem; CK(cuMemCreate(&mem, mp.size, &ap, 0));
  CK(cuMulticastBindMem(mc, 0, mem, 0, mp.size, 0));
  CUdeviceptr uva, mva;
  CK(cuMemAddressReserve(&uva, mp.size, gran, 0, 0)); CK(cuMemMap(uva, mp.size, 0, mem, 0));
  CK(cuMemAddressReserve(&mva, mp.size, gran, 0, 0)); CK(cuMemMap(mva, mp.size, 0, mc, 0));
  CUmemAccessDesc ad = {}; ad.location.type = CU_MEM_LOCATION_TYPE_DEVICE; ad.location.id = 0; ad.flags = CU_MEM_ACCESS_FLAGS_PROT_READWRITE;
  CK(cuMemSetAccess(uva, mp.size, &ad, 1)); CK(cuMemSetAccess(mva, mp.size, &ad, 1));
  int n = 1 << 16;
  cudaMemset((void*)uva, 0, n * 4);
  k_mc_store<<<(n / 4 + 255) / 256, 256>>>((uint32_t*)mva, n);
  cudaError_t e = cudaDeviceSynchronize();
  printf("kernel: %s\n", cudaGetErrorString(e));
  static uint32_t h[1 << 16];
  cudaMemcpy(h, (void*)uva, n * 4, cudaMemcpyDeviceToHost);
  int bad = 0; for (int i = 0; i < n; ++i) bad += h[i] != (uint32_t)i;
  printf("multicast store readback: %d mismatches of %d\n", bad, n);
  return 0;
}
