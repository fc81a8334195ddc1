// nvls.cuh -- GEMM -> all-reduce fusion over NVLink SHARP (NVLS) multicast memory
// (no reference counterpart -- the reference has no distributed path,
// SPEC.md:12).
//
// The data-parallel gradient buckets of a plan (planner _bucket_allreduce) live in a
// region that every rank maps twice: its own physical copy (unicast address, what the
// parameter updates read) and the team's multicast address (cuMulticastCreate /
// cuMulticastBindMem, runtime.cu NVLS section).  Then:
//   * a weight-gradient GEMM whose output is a bucket member adds its tiles straight into
//     the multicast address from the epilogue (multimem.red.add.v4.f32, gemm_tc.cuh): the
//     switch performs the cross-rank sum and every rank's copy receives it -- no separate
//     collective pass over the gradient, no split-K reduction kernel (every K slice adds);
//   * members produced by other kernels (bias / layernorm / embedding gradients) write
//     their local copy; the bucket's one-shot all-reduce k_nvls_allreduce gives each rank
//     1/R of those spans: multimem.ld_reduce (the switch sums the R copies) followed by
//     multimem.st (broadcast of the sum);
//   * k_nvls_barrier orders the phases across ranks: an arrival multimem.red.release.sys on
//     a flag word in the multicast region, then a wait until the local copy of the flag
//     reaches R x (this barrier's generation).  Per-plan-position slots, so concurrent side
//     branches never share a counter.
// Per step: list start -- zero the red targets (k_nvls_zero) + barrier; bucket -- barrier
// (every rank's reds landed) [+ all-reduce of the non-GEMM spans + barrier] as a side
// branch joined before the first reader (T_JOIN), like the NCCL buckets it replaces.
//
// Two transports, one protocol (RedMode):
//   RED_MC  -- NVLS multicast object (cuMulticastCreate): one multimem op per 16 bytes, the
//              switch reduces / broadcasts;
//   RED_P2P -- no multicast object available (single-GPU containers report
//              CUDA_ERROR_INVALID_VALUE from cuMulticastCreate, probes/nvls_probe.cu): every
//              rank's region is opened by its peers through CUDA IPC and the same kernels
//              add into / load from each peer's copy over NVLink (red.global.add.v4.f32 per
//              peer, rank-ordered sums in the one-shot all-reduce).  With a single rank
//              this is the path the GPU tests run.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

namespace coex {

constexpr int kNvlsSlots = 1024;          // barrier flag words at the start of the region
constexpr size_t kNvlsFlagBytes = 4096;   // kNvlsSlots x u32
constexpr int kMaxPeers = 8;              // ranks of one NVLink domain (one box)
enum RedMode { RED_NONE = 0, RED_MC = 1, RED_P2P = 2 };

__device__ __forceinline__ void mc_red_add_v4(float* mc, float4 v) {
  asm volatile("multimem.red.relaxed.sys.global.add.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(mc), "f"(v.x), "f"(v.y),
               "f"(v.z), "f"(v.w)
               : "memory");
}
__device__ __forceinline__ void mc_red_add(float* mc, float v) {
  asm volatile("multimem.red.relaxed.sys.global.add.f32 [%0], %1;" ::"l"(mc), "f"(v) : "memory");
}
__device__ __forceinline__ void p2p_red_add_v4(float* q, float4 v) {
  asm volatile("red.relaxed.sys.global.add.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(q), "f"(v.x), "f"(v.y), "f"(v.z),
               "f"(v.w)
               : "memory");
}
__device__ __forceinline__ void p2p_red_add(float* q, float v) {
  asm volatile("red.relaxed.sys.global.add.f32 [%0], %1;" ::"l"(q), "f"(v) : "memory");
}

// The epilogue's reduction target(s) of a GEMM output element: byte distances from the
// local copy to the multicast alias (RED_MC, delta[0]) or to every rank's copy (RED_P2P).
struct RedTarget {
  int mode;
  int npeers;
  long long delta[kMaxPeers];
};
__device__ __forceinline__ void red_store4(const RedTarget& t, float* dst, float4 v, bool vec, int nvalid) {
  if (t.mode == RED_MC) {
    float* q = (float*)((char*)dst + t.delta[0]);
    if (vec) {
      mc_red_add_v4(q, v);
    } else {
      mc_red_add(q, v.x);
      if (nvalid > 1) mc_red_add(q + 1, v.y);
      if (nvalid > 2) mc_red_add(q + 2, v.z);
      if (nvalid > 3) mc_red_add(q + 3, v.w);
    }
    return;
  }
  for (int r = 0; r < t.npeers; ++r) {
    float* q = (float*)((char*)dst + t.delta[r]);
    if (vec) {
      p2p_red_add_v4(q, v);
    } else {
      p2p_red_add(q, v.x);
      if (nvalid > 1) p2p_red_add(q + 1, v.y);
      if (nvalid > 2) p2p_red_add(q + 2, v.z);
      if (nvalid > 3) p2p_red_add(q + 3, v.w);
    }
  }
}

struct NvlsBarrierParams {
  DevState* ds;
  int mode;
  int world;
  unsigned int* flag_arrive[kMaxPeers];   // RED_MC: [0] = multicast alias; RED_P2P: every rank's copy
  unsigned int* flag_local;               // this rank's copy
  unsigned int* gen;                      // local generation counter of the slot (ordinary device memory)
};

// One thread: arrive on every rank's copy, then wait for the team.  A device-side bound
// (20 s) turns a lost peer into COEX_CUDA_ERROR instead of a hung GPU.
__global__ void __launch_bounds__(32) k_nvls_barrier(NvlsBarrierParams p) {
  COEX_PDL_ENTER();
  stamp(p.ds, SK_NVLS);
  if (threadIdx.x != 0) return;
  const unsigned int g = *p.gen + 1u;
  *p.gen = g;
  asm volatile("fence.proxy.alias;" ::: "memory");
  asm volatile("fence.acq_rel.sys;" ::: "memory");
  if (p.mode == RED_MC) {
    asm volatile("multimem.red.release.sys.global.add.u32 [%0], %1;" ::"l"(p.flag_arrive[0]), "r"(1u) : "memory");
  } else {
    for (int r = 0; r < p.world; ++r)
      asm volatile("red.release.sys.global.add.u32 [%0], %1;" ::"l"(p.flag_arrive[r]), "r"(1u) : "memory");
  }
  const unsigned int target = g * (unsigned int)p.world;
  const unsigned long long t0 = globaltimer();
  int polls = 0;
  for (;;) {
    unsigned int v;
    asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(p.flag_local) : "memory");
    if ((int)(v - target) >= 0) break;
    if (++polls > 32) {
      __nanosleep(100);
      if (globaltimer() - t0 > 20000000000ull) {
        p.ds->status = 8;                 // COEX_CUDA_ERROR: a peer never arrived
        p.ds->cancelled = 1;
        break;
      }
    }
  }
  asm volatile("fence.proxy.alias;" ::: "memory");
}

struct NvlsSpan {
  long long off;              // float offset from the region base
  long long n;                // floats
};
constexpr int kNvlsMaxSpans = 100;

struct NvlsAllReduceParams {
  DevState* ds;
  int mode;
  int nspans;
  int rank, world;
  float scale;                // 1 (sum) or 1 / world (average)
  float* base[kMaxPeers];     // RED_MC: [0] = multicast base; RED_P2P: every rank's region base
  NvlsSpan spans[kNvlsMaxSpans];
};

// One-shot all-reduce of the bucket spans the GEMM epilogues did not already reduce:
// rank r owns 16-byte groups g with g % world == r of every span.  RED_MC:
// multimem.ld_reduce sums the R copies in the switch, multimem.st writes the sum to all of
// them; RED_P2P: the owner loads the group from every rank's copy (rank order, so every
// rank sees the same rounding), stores the sum into every copy.
__global__ void __launch_bounds__(256) k_nvls_allreduce(const __grid_constant__ NvlsAllReduceParams p) {
  COEX_PDL_ENTER();
  stamp(p.ds, SK_NVLS);
  const long long tid = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  const long long nth = (long long)gridDim.x * blockDim.x;
  for (int s = 0; s < p.nspans; ++s) {
    const long long off = p.spans[s].off, n = p.spans[s].n;
    const long long groups = n / 4;                 // span offsets are 16-byte aligned
    for (long long g = tid * p.world + p.rank; g < groups; g += nth * p.world) {
      float4 v;
      if (p.mode == RED_MC) {
        asm volatile("multimem.ld_reduce.relaxed.sys.global.add.v4.f32 {%0, %1, %2, %3}, [%4];"
                     : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w)
                     : "l"(p.base[0] + off + 4 * g)
                     : "memory");
      } else {
        v = __ldcv((const float4*)(p.base[0] + off) + g);
        for (int r = 1; r < p.world; ++r) {
          const float4 u = __ldcv((const float4*)(p.base[r] + off) + g);
          v.x += u.x; v.y += u.y; v.z += u.z; v.w += u.w;
        }
      }
      v.x *= p.scale; v.y *= p.scale; v.z *= p.scale; v.w *= p.scale;
      if (p.mode == RED_MC) {
        asm volatile("multimem.st.relaxed.sys.global.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(p.base[0] + off + 4 * g),
                     "f"(v.x), "f"(v.y), "f"(v.z), "f"(v.w)
                     : "memory");
      } else {
        for (int r = 0; r < p.world; ++r) __stcg((float4*)(p.base[r] + off) + g, v);
      }
    }
    if (p.rank == 0) {                              // ragged tail: rank 0
      for (long long i = groups * 4 + tid; i < n; i += nth) {
        float v;
        if (p.mode == RED_MC) {
          asm volatile("multimem.ld_reduce.relaxed.sys.global.add.f32 %0, [%1];" : "=f"(v) : "l"(p.base[0] + off + i) : "memory");
        } else {
          v = __ldcv(p.base[0] + off + i);
          for (int r = 1; r < p.world; ++r) v += __ldcv(p.base[r] + off + i);
        }
        v *= p.scale;
        if (p.mode == RED_MC) {
          asm volatile("multimem.st.relaxed.sys.global.f32 [%0], %1;" ::"l"(p.base[0] + off + i), "f"(v) : "memory");
        } else {
          for (int r = 0; r < p.world; ++r) __stcg(p.base[r] + off + i, v);
        }
      }
    }
  }
}

struct NvlsZeroParams {
  DevState* ds;
  float4* p;                  // local copy, 16-byte aligned
  long long n4;
};
__global__ void __launch_bounds__(256) k_nvls_zero(NvlsZeroParams q) {
  COEX_PDL_ENTER();
  stamp(q.ds, SK_NVLS);
  const float4 z = make_float4(0.f, 0.f, 0.f, 0.f);
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < q.n4; i += (long long)gridDim.x * blockDim.x)
    q.p[i] = z;
}

}  // namespace coex
