// mma_probe.cu -- tcgen05.mma issue-to-completion cost per instruction shape (SS mode, bf16,
// fp32 accumulate, SW128 K-major operands) on one SM: n back-to-back MMAs, then a commit;
// prints cycles per MMA.  nvcc -gencode arch=compute_100a,code=sm_100a -o mma_probe mma_probe.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint64_t desc(const void* p, uint32_t lbo) {
  uint64_t d = 0;
  d |= (uint64_t)((smem_u32(p) & 0x3FFFF) >> 4);
  d |= (uint64_t)((lbo >> 4) & 0x3FFF) << 16;
  d |= (uint64_t)(1024 >> 4) << 32;
  d |= (uint64_t)1 << 46;
  d |= (uint64_t)2 << 61;
  return d;
}
__host__ __device__ constexpr uint32_t idesc(int M, int N, bool a_mn, bool b_mn) {
  return (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)a_mn << 15) | ((uint32_t)b_mn << 16) | ((uint32_t)(N >> 3) << 17) |
         ((uint32_t)(M >> 4) << 24);
}

__device__ __forceinline__ void mma_elect(uint32_t tm, uint64_t da, uint64_t db, uint32_t id) {
  asm volatile(
      "{\n\t.reg .pred P;\n\telect.sync _|P, 0xffffffff;\n\t"
      "@P tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, 1;\n\t}" ::"r"(tm),
      "l"(da), "l"(db), "r"(id));
}
template <int MODE>
__global__ void probe(int N, int n_mma, int b_mn, long long* out) {
  extern __shared__ __align__(1024) unsigned char raw[];
  unsigned char* sm = (unsigned char*)(((uintptr_t)raw + 1023) & ~(uintptr_t)1023);
  __shared__ uint64_t bar;
  __shared__ uint32_t slot;
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar)));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (threadIdx.x < 32) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(&slot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  for (int i = threadIdx.x; i < 160 * 1024 / 4; i += blockDim.x) ((uint32_t*)sm)[i] = 0x3c003c00u;
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  if (MODE == 0 ? threadIdx.x == 0 : threadIdx.x < 32) {
    const uint32_t tm = slot;
    const uint32_t id = idesc(128, N, false, b_mn != 0);
    const unsigned char* A = sm;
    const unsigned char* B = sm + 64 * 1024;
    for (int rep = 0; rep < 2; ++rep) {
      long long t0 = clock64();
      for (int i = 0; i < n_mma; ++i) {
        uint64_t da = desc(A, 16) + 2 * (i & 3);
        uint64_t db = b_mn ? desc(B, 8192) + 128 * (i & 7) : desc(B, 16) + 2 * (i & 3);
        if (MODE == 0)
          asm volatile(
              "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
              "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(tm),
              "l"(da), "l"(db), "r"(id), "r"(1));
        else
          mma_elect(tm, da, db, id);
      }
      long long t1 = clock64();
      if (MODE == 0 || threadIdx.x == 0) asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(&bar))
                   : "memory");
      uint32_t done = 0;
      while (!done) {
        asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0,1,0,p;\n\t}"
                     : "=r"(done) : "r"(smem_u32(&bar)), "r"((uint32_t)rep));
      }
      long long t2 = clock64();
      if (threadIdx.x == 0) {
        out[2 * rep] = t1 - t0;
        out[2 * rep + 1] = t2 - t0;
      }
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (threadIdx.x < 32) {
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(slot));
  }
}

int main() {
  long long* d;
  cudaMalloc(&d, 64);
  cudaFuncSetAttribute(probe<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, 170 * 1024);
  cudaFuncSetAttribute(probe<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, 170 * 1024);
  const int Ns[] = {64, 128, 256};
  for (int mode = 0; mode < 2; ++mode)
  for (int bm = 0; bm < 2; ++bm)
    for (int N : Ns)
      for (int n : {16, 256}) {
        if (mode == 0) probe<0><<<1, 128, 170 * 1024>>>(N, n, bm, d);
        else probe<1><<<1, 128, 170 * 1024>>>(N, n, bm, d);
        long long h[4];
        cudaMemcpy(h, d, 32, cudaMemcpyDeviceToHost);
        printf("mode %d M=128 N=%3d K=16 b_mn=%d n=%4d: issue %6lld cyc, complete %7lld cyc, %.1f cyc/mma (warm)\n", mode, N, bm, n,
               h[2], h[3], (double)h[3] / n);
      }
  printf("err: %s\n", cudaGetErrorString(cudaDeviceSynchronize()));
  return 0;
}
