// NVLS multicast probe: which cuMulticastCreate parameters this box accepts, then one
// multimem.red / ld_reduce round trip through a 1-device team.
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <cstring>

__global__ void k_red(float* mc, float* uc, float* out) {
  asm volatile("multimem.red.relaxed.sys.global.add.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(mc), "f"(1.f), "f"(2.f),
               "f"(3.f), "f"(4.f) : "memory");
  asm volatile("fence.proxy.alias;" ::: "memory");
  __threadfence_system();
  float4 v;
  asm volatile("multimem.ld_reduce.relaxed.sys.global.add.v4.f32 {%0, %1, %2, %3}, [%4];"
               : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "l"(mc) : "memory");
  out[0] = v.x; out[1] = v.w; out[2] = uc[0]; out[3] = uc[3];
}

int main() {
  cuInit(0);
  CUdevice dev;
  cuDeviceGet(&dev, 0);
  CUcontext ctx;
  cuDevicePrimaryCtxRetain(&ctx, dev);
  cuCtxSetCurrent(ctx);
  int mcs = 0;
  cuDeviceGetAttribute(&mcs, CU_DEVICE_ATTRIBUTE_MULTICAST_SUPPORTED, dev);
  printf("multicast supported: %d\n", mcs);
  size_t sizes[] = {2u << 20, 512u << 20, (size_t)1536 << 20};
  unsigned types[] = {0, CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR, CU_MEM_HANDLE_TYPE_FABRIC};
  for (int nd = 1; nd <= 2; ++nd)
    for (unsigned t : types)
      for (size_t s : sizes) {
        CUmulticastObjectProp p;
        memset(&p, 0, sizeof(p));
        p.numDevices = nd;
        p.size = s;
        p.handleTypes = t;
        size_t g = 0, gm = 0;
        CUresult rg = cuMulticastGetGranularity(&g, &p, CU_MULTICAST_GRANULARITY_RECOMMENDED);
        cuMulticastGetGranularity(&gm, &p, CU_MULTICAST_GRANULARITY_MINIMUM);
        CUmemGenericAllocationHandle h;
        CUresult r = cuMulticastCreate(&h, &p);
        printf("numDevices=%d handleTypes=%u size=%zu MB: gran rc=%d rec=%zu min=%zu create rc=%d\n", nd, t, s >> 20,
               (int)rg, g, gm, (int)r);
        if (r == CUDA_SUCCESS) cuMemRelease(h);
      }
  // round trip with the first configuration that works
  CUmulticastObjectProp p;
  memset(&p, 0, sizeof(p));
  p.numDevices = 1;
  p.size = 2u << 20;
  p.handleTypes = CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR;
  CUmemGenericAllocationHandle mch;
  CUresult r = cuMulticastCreate(&mch, &p);
  if (r) { p.handleTypes = 0; r = cuMulticastCreate(&mch, &p); }
  printf("create for round trip: %d\n", (int)r);
  if (r) return 0;
  printf("add device: %d\n", (int)cuMulticastAddDevice(mch, dev));
  CUmemAllocationProp ap;
  memset(&ap, 0, sizeof(ap));
  ap.type = CU_MEM_ALLOCATION_TYPE_PINNED;
  ap.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
  ap.location.id = 0;
  CUmemGenericAllocationHandle mem;
  printf("mem create: %d\n", (int)cuMemCreate(&mem, p.size, &ap, 0));
  CUdeviceptr uc, mc;
  CUmemAccessDesc ad;
  memset(&ad, 0, sizeof(ad));
  ad.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
  ad.location.id = 0;
  ad.flags = CU_MEM_ACCESS_FLAGS_PROT_READWRITE;
  printf("reserve uc %d\n", (int)cuMemAddressReserve(&uc, p.size, 2u << 20, 0, 0));
  printf("map uc %d\n", (int)cuMemMap(uc, p.size, 0, mem, 0));
  printf("access uc %d\n", (int)cuMemSetAccess(uc, p.size, &ad, 1));
  printf("bind %d\n", (int)cuMulticastBindMem(mch, 0, mem, 0, p.size, 0));
  printf("reserve mc %d\n", (int)cuMemAddressReserve(&mc, p.size, 2u << 20, 0, 0));
  printf("map mc %d\n", (int)cuMemMap(mc, p.size, 0, mch, 0));
  printf("access mc %d\n", (int)cuMemSetAccess(mc, p.size, &ad, 1));
  cudaMemset((void*)uc, 0, p.size);
  float* out;
  cudaMalloc(&out, 16);
  k_red<<<1, 1>>>((float*)mc, (float*)uc, out);
  cudaError_t e = cudaDeviceSynchronize();
  float h[4];
  cudaMemcpy(h, out, 16, cudaMemcpyDeviceToHost);
  printf("kernel: %s  ld_reduce %.1f %.1f  local %.1f %.1f (expect 1 4 1 4)\n", cudaGetErrorString(e), h[0], h[1],
         h[2], h[3]);
  return 0;
}
