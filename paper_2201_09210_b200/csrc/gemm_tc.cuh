// gemm_tc.cuh -- MATMUL on the 5th-generation tensor cores (tcgen05) for the
// bf16 precision mode: C[M,N] (fp32) = A[M,K] . B[K,N], operands rounded to
// bf16, fp32 accumulation in TMEM (reference op: tensor.py:228-236; tolerance
// 2e-2 relative per BASELINE.json north_star).
//
// Two kernels per MatMul node:
//   k_cvt_bf16  -- fp32 operand (read through its cell, optionally stored
//                  transposed) -> bf16 K-major copy with a 16-byte-multiple row
//                  pitch (the TMA source); B is written as B^T [N][K].
//   k_gemm_tc   -- warp-specialised tcgen05 GEMM, one 128 x BN tile per CTA:
//                  warp 0 = TMA producer (cp.async.bulk.tensor, SWIZZLE_128B),
//                  warp 1 = TMEM allocator + single-thread MMA issuer
//                  (tcgen05.mma.cta_group::1.kind::f16, M=128, N=BN, K=16),
//                  warps 2-5 = epilogue (tcgen05.ld 32x32b -> fp32 stores).
//                  4-stage smem ring with full/empty mbarriers; tcgen05.commit
//                  frees a stage when its MMAs retire.
#pragma once
#include <cuda.h>
#include <cuda_bf16.h>

#include "kernels.cuh"

namespace coex {

constexpr int TC_BM = 128;
constexpr int TC_BN = 256;          // 128 x 256 tile: 85 FLOP per operand byte (L2-bandwidth headroom)
constexpr int TC_BK = 64;          // 64 bf16 = 128 B = one SWIZZLE_128B row
constexpr int TC_THREADS = 192;
constexpr int TC_A_BYTES = TC_BM * TC_BK * 2;
constexpr int TC_GROUP_M = 16;      // tile rasterisation: 16 M-tiles sweep N together (L2 reuse)
constexpr int TC_EPI_LD = 36;       // epilogue staging row pitch (floats): 32 columns + 16-byte pad
constexpr int TC_EPI_BYTES = 4 * 32 * TC_EPI_LD * 4;   // four epilogue warps x 32 rows
// Narrow-N variants (convolution GEMMs have N = Cout in 64..512): BN in {64, 128, 256};
// the stage count grows as the B tile shrinks so every variant keeps ~192 KB in flight.
// DUO: a shallow-pipeline variant small enough for two CTAs per SM (BN <= 128; two TMEM
// accumulator pairs fit the 512 columns) -- for short-K GEMMs on under two waves of tiles,
// where per-tile latency rather than operand bandwidth bounds the launch.
template <int BN, bool DUO = false> struct TcCfg {
  static constexpr int STAGES = DUO ? (BN == 64 ? 3 : 2) : BN == 256 ? 4 : BN == 128 ? 6 : 8;
  static constexpr int B_BYTES = BN * TC_BK * 2;
  static constexpr int SMEM = STAGES * (TC_A_BYTES + B_BYTES) + 1024 /*align*/ + 256 /*barriers, tmem slot*/ +
                               TC_EPI_BYTES;
};
constexpr int TC_STAGES = TcCfg<TC_BN>::STAGES;
constexpr int TC_B_BYTES = TcCfg<TC_BN>::B_BYTES;
constexpr int TC_SMEM = TcCfg<TC_BN>::SMEM;

struct CvtParams {
  DevState* ds;
  In src[2];                 // fp32 operands
  long long rows[2];         // rows of the K-major output (M for A, N for B)
  long long K;
  long long ld;              // padded K pitch (elements, multiple of 8)
  int trans[2];              // 1: element (r, k) is src[k * rows + r]; 0: src[r * K + k]
  __nv_bfloat16* dst[2];
  long long Kb, ldb;         // operand 1's row length / pitch when own_b is set
  int own_b;                 // 1: operand 1 has its own K (Kb, may be 0) and pitch (ldb)
};

// Operand conversion: grid.y selects the operand.  Direct operands stream rows
// (coalesced on both sides); transposed operands go through a 32x33 shared-memory
// tile so both the strided read and the K-major write stay coalesced.
__global__ void __launch_bounds__(256) k_cvt_bf16(CvtParams p) {
  COEX_PDL_ENTER();
  stamp(p.ds, SK_CVT);
  // operand select without dynamic indexing of the parameter arrays (that would copy the
  // whole parameter block to local memory in every thread)
  const bool w1 = blockIdx.y != 0;
  const float* s = res<float>(w1 ? p.src[1] : p.src[0]);
  __nv_bfloat16* d = w1 ? p.dst[1] : p.dst[0];
  const bool own = w1 && p.own_b;
  const long long R = w1 ? p.rows[1] : p.rows[0], K = own ? p.Kb : p.K, ld = own ? p.ldb : p.ld;
  if (!(w1 ? p.trans[1] : p.trans[0])) {
    // flattened over 8-element units of every row: 8 consecutive k per thread, one 16-byte store
    const long long per_row = ld / 8, total = R * per_row;
    const bool vec = (K % 4) == 0 && ld == K && ((uintptr_t)s & 15) == 0;
    for (long long u = (long long)blockIdx.x * blockDim.x + threadIdx.x; u < total;
         u += (long long)gridDim.x * blockDim.x) {
      const long long r = u / per_row, k = (u - r * per_row) * 8;
      const float* src = s + r * K;
      uint4 o;
      if (vec) {
        const float4 a = *(const float4*)(src + k), b = *(const float4*)(src + k + 4);
        __nv_bfloat162 v0 = __floats2bfloat162_rn(a.x, a.y), v1 = __floats2bfloat162_rn(a.z, a.w);
        __nv_bfloat162 v2 = __floats2bfloat162_rn(b.x, b.y), v3 = __floats2bfloat162_rn(b.z, b.w);
        o.x = *(uint32_t*)&v0; o.y = *(uint32_t*)&v1; o.z = *(uint32_t*)&v2; o.w = *(uint32_t*)&v3;
      } else {
        __align__(16) __nv_bfloat16 v[8];
#pragma unroll
        for (int j = 0; j < 8; ++j) v[j] = __float2bfloat16_rn(k + j < K ? src[k + j] : 0.f);
        o = *(const uint4*)v;
      }
      *(uint4*)(d + r * ld + k) = o;
    }
    return;
  }
  // element (r, k) = s[k * R + r]: tiles of 32 k x 32 r
  __shared__ float tile[32][33];
  const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;   // 32 x 8
  const long long tr = (R + 31) / 32, tk = (ld + 31) / 32;
  for (long long t = blockIdx.x; t < tr * tk; t += gridDim.x) {
    const long long r0 = (t % tr) * 32, k0 = (t / tr) * 32;
    for (int j = ty; j < 32; j += 8) {
      const long long k = k0 + j, r = r0 + tx;
      tile[j][tx] = (k < K && r < R) ? s[k * R + r] : 0.f;
    }
    __syncthreads();
    for (int j = ty; j < 32; j += 8) {
      const long long r = r0 + j, k = k0 + tx;
      if (r < R && k < ld) d[r * ld + k] = __float2bfloat16_rn(tile[tx][j]);
    }
    __syncthreads();
  }
}

// Implicit-GEMM convolution geometry (AMODE 2 / 3): the A operand is gathered straight from
// the bf16 NHWC input by 4-D TMA boxes {64 channels, bw*s, bh*s, bn} with element strides
// {1, s, s, 1} -- one box per (tap, 64-channel chunk) and pixel block; padding = TMA
// out-of-bounds zero fill.  Pixel (n, oy, ox) of the GEMM grid reads input
// (n, oy*s + off_y + ty, ox*s + off_x + tx) for tap (ty, tx) = (tap / taps_x, tap % taps_x).
// conv2d_t runs as `phases` sub-pixel convolutions (stride 1, per-phase offsets, phase weights
// stacked in B), the epilogue scattering GEMM row (n, h, w) of phase (py, px) to output row
// (n, so*h + py, so*w + px).
struct TcConv {
  int C;                     // input channels (multiple of 64)
  int taps_x;                // taps per kernel row in the K ordering (tap, channel)
  int s;                     // element stride of the gather
  int Hg, Wg;                // GEMM pixel grid
  int bw, bh, bn;            // pixel block of one box (bw * bh * bn = 128 (AMODE 2) or 64 (AMODE 3))
  int phases;                // 1, or so*so for the sub-pixel conv2d_t
  int so, Ho, Wo;            // output grid of the scatter epilogue (phases > 1)
  long long b_rows;          // B rows per phase (phase p reads B rows p * b_rows ...)
  int off_y[4], off_x[4];    // lower offsets (phases == 1: index 0)
  int pad, bord;             // phases > 1: conv2d_t padding and the bf16 copy's zero border
};

// lower input offset of output phase q (sub-pixel conv2d_t): taps ky = ky0 + (T-1-j)*so,
// ky0 = (q + pad) mod so, input row = h + (q + pad - ky0)/so - (T-1) + j (+ border)
__device__ __forceinline__ int phase_off(const TcConv& g, int q) {
  const int k0 = (q + g.pad) % g.so;
  return (q + g.pad - k0) / g.so - (g.taps_x - 1) + g.bord;
}

struct TcGemmParams {
  CUtensorMap tmA;           // bf16 [M][ld], box {64, 128}, SWIZZLE_128B (AMODE 2/3: 4-D NHWC map)
  CUtensorMap tmB;           // bf16 [N][ld], box {64, BN}
  DevState* ds;
  In a, b;                   // original operands (ping-pong output choice only)
  long long M, N, K;
  Out out;
  float* raw;                // non-null: write here (no publication) -- scratch / split-K slices
  int splits;                // split-K: CTA (tile, split) covers k-blocks of its slice, raw + split*M*N
  TcConv cv;
  int batch;                 // batched GEMM (bmm): 3-D tensor maps {inner, rows, batch}; C + b * c_bstride
  long long c_bstride;
  // causal attention structure (planner-proven, see planner.py _tri_flags):
  //   tri_out: only the lower triangle (col <= row) of C is ever read -> tiles strictly above
  //            the diagonal are skipped (no MMA, no store);
  //   tri_a:   A is lower- (1) / upper- (2) triangular in (m, k) -> K blocks outside are zero
  int tri_out, tri_a;
  In bias;                   // has_bias: C[m][n] += bias[n] in the epilogue (fused bias_add)
  int has_bias;
  // GEMM -> all-reduce fusion (nvls.cuh): mode != RED_NONE -- the epilogue adds every tile
  // into the team's copies (multimem.red or per-peer red) instead of storing it
  RedTarget red;
};

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  const uint32_t a = smem_u32(bar);
  uint32_t done = 0;
  while (!done) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t}"
        : "=r"(done)
        : "r"(a), "r"(parity)
        : "memory");
  }
}
__device__ __forceinline__ void tma_load_2d(void* dst, const CUtensorMap* map, uint64_t* bar, int c0, int c1) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], [%2];" ::
          "r"(smem_u32(dst)),
      "l"((uint64_t)map), "r"(smem_u32(bar)), "r"(c0), "r"(c1)
      : "memory");
}

// SMEM matrix descriptor, K-major, SWIZZLE_128B (cute UMMA::SmemDescriptor):
// start>>4 [0,14), LBO=1 [16,30), SBO=1024>>4 [32,46), version=1 [46,48), layout=2 [61,64).
__device__ __forceinline__ uint64_t smem_desc_k_sw128(const void* p) {
  uint64_t d = 0;
  d |= (uint64_t)((smem_u32(p) & 0x3FFFF) >> 4);
  d |= (uint64_t)1 << 16;
  d |= (uint64_t)(1024 >> 4) << 32;
  d |= (uint64_t)1 << 46;
  d |= (uint64_t)2 << 61;
  return d;
}

// SMEM matrix descriptor, MN-major, SWIZZLE_128B: the tile is a stack of TMA boxes of 64
// MN-elements x 64 K-rows (8 KB each, 128-B rows); canonical layout ((8,n),(8,k)) in 16-byte
// units with LBO = 8192 B (next 64 MN-elements), SBO = 1024 B (next 8 K-rows).
__device__ __forceinline__ uint64_t smem_desc_mn_sw128(const void* p) {
  uint64_t d = 0;
  d |= (uint64_t)((smem_u32(p) & 0x3FFFF) >> 4);
  d |= (uint64_t)(8192 >> 4) << 16;
  d |= (uint64_t)(1024 >> 4) << 32;
  d |= (uint64_t)1 << 46;
  d |= (uint64_t)2 << 61;
  return d;
}

// Instruction descriptor kind::f16: D=F32 (bit 4), A=BF16 (bits 7-9), B=BF16 (bits 10-12),
// K-major A/B, N>>3 at [17,23), M>>4 at [24,29).
__host__ __device__ constexpr uint32_t idesc_bf16_f32(int M, int N, bool a_mn = false, bool b_mn = false) {
  return (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(a_mn ? 1 : 0) << 15) | ((uint32_t)(b_mn ? 1 : 0) << 16) |
         ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
}

__device__ __forceinline__ void tma_load_3d(void* dst, const CUtensorMap* map, uint64_t* bar, int c0, int c1, int c2) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4, %5}], [%2];" ::
          "r"(smem_u32(dst)),
      "l"((uint64_t)map), "r"(smem_u32(bar)), "r"(c0), "r"(c1), "r"(c2)
      : "memory");
}

__device__ __forceinline__ void tma_load_4d(void* dst, const CUtensorMap* map, uint64_t* bar, int c0, int c1, int c2,
                                            int c3) {
  asm volatile(
      "cp.async.bulk.tensor.4d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4, %5, %6}], [%2];" ::
          "r"(smem_u32(dst)),
      "l"((uint64_t)map), "r"(smem_u32(bar)), "r"(c0), "r"(c1), "r"(c2), "r"(c3)
      : "memory");
}

// pixel index -> (n, oy, ox) of the GEMM grid
__device__ __forceinline__ void conv_pix(const TcConv& g, long long pix, int& n, int& oy, int& ox) {
  ox = (int)(pix % g.Wg);
  const long long t = pix / g.Wg;
  oy = (int)(t % g.Hg);
  n = (int)(t / g.Hg);
}

// tcgen05.commit from one elected lane of a converged warp
__device__ __forceinline__ void tc_commit_elect(uint64_t* bar) {
  asm volatile(
      "{\n\t.reg .pred e;\n\telect.sync _|e, 0xffffffff;\n\t"
      "@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n\t}" ::"r"(smem_u32(bar))
      : "memory");
}

__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}

// Persistent warp-specialised GEMM.  Work items = (output tile, K slice), strided over the
// grid; three pipelines: the smem ring (TMA -> MMA, `full`/`empty`), two TMEM accumulator
// buffers (MMA -> epilogue, `tfull`/`tempty`) so the epilogue of item i overlaps the MMAs of
// item i+1, and the static round-robin item schedule shared by all roles.
// AMODE: 0 = A K-major 2-D, 1 = A MN-major 2-D ([K][M] rows, e.g. an im2col matrix used as
// A^T), 2 = implicit convolution, A K-major (conv2d / sub-pixel conv2d_t), 3 = implicit
// convolution, A MN-major (weight gradient: M = (tap, channel), K = pixels).  B_MN: B stored
// [K][N].  MN-major operands are loaded as 64 x 64 boxes and consumed through MN-major
// descriptors, so no transposition pass is needed.
// RED: the epilogue adds into the data-parallel gradient region (nvls.cuh) instead of
// storing -- a separate instantiation so the plain epilogue's code is untouched
template <int BN, int AMODE, bool B_MN, bool DUO = false, bool RED = false>
__global__ void __launch_bounds__(TC_THREADS, DUO ? 2 : 1) k_gemm_tc(const __grid_constant__ TcGemmParams p) {
  COEX_PDL_ENTER();
  constexpr int STAGES = TcCfg<BN, DUO>::STAGES;
  constexpr int B_BYTES = TcCfg<BN, DUO>::B_BYTES;
  constexpr uint32_t TMEM_COLS = 2 * BN;            // two accumulator buffers
  constexpr bool A_MN = AMODE == 1 || AMODE == 3;
  stamp(p.ds, SK_MATMUL);
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  unsigned char* smem = (unsigned char*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  unsigned char* sA = smem;
  unsigned char* sB = smem + STAGES * TC_A_BYTES;
  uint64_t* full = (uint64_t*)(sB + STAGES * B_BYTES);
  uint64_t* empty = full + STAGES;
  uint64_t* tfull = empty + STAGES;                 // [2]
  uint64_t* tempty = tfull + 2;                     // [2]
  uint32_t* tmem_slot = (uint32_t*)(tempty + 2);

  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  const long long tiles_n = (p.N + BN - 1) / BN;
  const long long tiles_m = (p.M + TC_BM - 1) / TC_BM;
  const int splits = p.splits > 1 ? p.splits : 1;
  const int phases = AMODE == 2 ? p.cv.phases : 1;
  const int nbat = p.batch > 1 ? p.batch : 1;
  const long long items = tiles_m * tiles_n * splits * phases * nbat;
  const int nk_all = (int)((p.K + TC_BK - 1) / TC_BK);
  const long long group = (long long)TC_GROUP_M * tiles_n;

  // item -> (m0, n0, split, first k-block, k-block count); grouped rasterisation of tiles
  auto decode = [&](long long it, int& m0, int& n0, int& split, int& kb0, int& nk) {
    split = (int)(it % splits);
    const long long t = ((it / splits) / phases) % (tiles_m * tiles_n);
    const long long first_m = (t / group) * TC_GROUP_M;
    const long long gm = min((long long)TC_GROUP_M, tiles_m - first_m);
    m0 = (int)((first_m + (t % group) % gm) * TC_BM);
    n0 = (int)(((t % group) / gm) * BN);
    kb0 = (int)((long long)nk_all * split / splits);
    nk = (int)((long long)nk_all * (split + 1) / splits) - kb0;
    if (p.tri_out && n0 >= m0 + TC_BM) nk = -1;               // tile above the diagonal: skipped
    else if (p.tri_a == 1) {                                  // A[m][k] == 0 for k > m
      const int hi = (m0 + TC_BM + TC_BK - 1) / TC_BK;
      if (kb0 + nk > hi) nk = hi - kb0 > 0 ? hi - kb0 : 0;
    } else if (p.tri_a == 2) {                                // A[m][k] == 0 for k < m
      const int lo = m0 / TC_BK, end = kb0 + nk;
      if (kb0 < lo) {
        kb0 = lo < end ? lo : end;
        nk = end - kb0;
      }
    }
  };

  float* Cout = nullptr;
  if (p.raw == nullptr) {
    Cout = pick_out<float>(p.out, res<float>(p.a), res<float>(p.b));
    publish_early(p.out, Cout);
  }
  count_op(p.ds);

  if (warp == 0 && lane == 0) {
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int a = 0; a < 2; ++a) {
      mbar_init(&tfull[a], 1);
      mbar_init(&tempty[a], 4);                     // one arrival per epilogue warp
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"((uint64_t)&p.tmA) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"((uint64_t)&p.tmB) : "memory");
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                 "r"(TMEM_COLS)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = *tmem_slot;

  if (warp == 0) {
    if (lane == 0) {                                // ===== TMA producer
      long long kbg = 0;                            // k-blocks issued by this CTA (ring position)
      for (long long it = blockIdx.x; it < items; it += gridDim.x) {
        int m0, n0, split, kb0, nk;
        decode(it, m0, n0, split, kb0, nk);
        const int cph = (int)((it / splits) % phases);     // sub-pixel phase of this item
        const int bi = (int)(((it / splits) / phases) / (tiles_m * tiles_n));   // batch of this item
        for (int kb = 0; kb < nk; ++kb, ++kbg) {
          const int s = (int)(kbg % STAGES);
          const uint32_t ph = (uint32_t)((kbg / STAGES) & 1);
          mbar_wait(&empty[s], ph ^ 1u);
          mbar_expect_tx(&full[s], TC_A_BYTES + B_BYTES);
          const int kk = (kb0 + kb) * TC_BK;
          if constexpr (AMODE == 2) {                 // (tap, channel chunk) x 128-pixel block
            const int tap = kk / p.cv.C, c0 = kk - tap * p.cv.C;
            const int ty = tap / p.cv.taps_x, tx = tap - ty * p.cv.taps_x;
            int pn, oy, ox;
            conv_pix(p.cv, m0, pn, oy, ox);
            int offy = p.cv.off_y[0], offx = p.cv.off_x[0];
            if (phases > 1) {
              offy = phase_off(p.cv, cph / p.cv.so);
              offx = phase_off(p.cv, cph % p.cv.so);
            }
            tma_load_4d(sA + s * TC_A_BYTES, &p.tmA, &full[s], c0, ox * p.cv.s + offx + tx, oy * p.cv.s + offy + ty, pn);
          } else if constexpr (AMODE == 3) {          // 64-pixel block x two (tap, channel) halves
            int pn, oy, ox;
            conv_pix(p.cv, kk, pn, oy, ox);
#pragma unroll
            for (int h = 0; h < TC_BM / 64; ++h) {
              const int mm = m0 + 64 * h;
              const int tap = mm / p.cv.C, c0 = mm - tap * p.cv.C;
              const int ty = tap / p.cv.taps_x, tx = tap - ty * p.cv.taps_x;
              tma_load_4d(sA + s * TC_A_BYTES + h * 8192, &p.tmA, &full[s], c0, ox * p.cv.s + p.cv.off_x[0] + tx,
                          oy * p.cv.s + p.cv.off_y[0] + ty, pn);
            }
          } else if constexpr (A_MN) {
#pragma unroll
            for (int h = 0; h < TC_BM / 64; ++h) {
              if (nbat > 1) tma_load_3d(sA + s * TC_A_BYTES + h * 8192, &p.tmA, &full[s], m0 + 64 * h, kk, bi);
              else tma_load_2d(sA + s * TC_A_BYTES + h * 8192, &p.tmA, &full[s], m0 + 64 * h, kk);
            }
          } else {
            if (nbat > 1) tma_load_3d(sA + s * TC_A_BYTES, &p.tmA, &full[s], kk, m0, bi);
            else tma_load_2d(sA + s * TC_A_BYTES, &p.tmA, &full[s], kk, m0);
          }
          const int brow = (int)(cph * p.cv.b_rows) + kk;
          if constexpr (B_MN) {
#pragma unroll
            for (int h = 0; h < BN / 64; ++h) {
              if (nbat > 1) tma_load_3d(sB + s * B_BYTES + h * 8192, &p.tmB, &full[s], n0 + 64 * h, brow, bi);
              else tma_load_2d(sB + s * B_BYTES + h * 8192, &p.tmB, &full[s], n0 + 64 * h, brow);
            }
          } else {
            if (nbat > 1) tma_load_3d(sB + s * B_BYTES, &p.tmB, &full[s], brow, n0, bi);
            else tma_load_2d(sB + s * B_BYTES, &p.tmB, &full[s], brow, n0);
          }
        }
      }
    }
  } else if (warp == 1) {
    {                                               // ===== MMA issuer: the whole warp runs the
      // loop (descriptors stay warp-uniform, on the uniform datapath) and one elected lane
      // issues each tcgen05.mma / commit -- a single-lane issuer pays ~82 cycles per MMA, more
      // than the tensor pipe's own 64 cycles at BN = 128 (probes/mma_probe.cu)
      constexpr uint32_t idesc = idesc_bf16_f32(TC_BM, BN, A_MN, B_MN);
      long long kbg = 0;
      int li = 0;                                   // local item index
      for (long long it = blockIdx.x; it < items; it += gridDim.x, ++li) {
        int m0, n0, split, kb0, nk;
        decode(it, m0, n0, split, kb0, nk);
        const int a = li & 1;
        const uint32_t aph = (uint32_t)((li >> 1) & 1);
        mbar_wait(&tempty[a], aph ^ 1u);            // epilogue drained this accumulator
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        const uint32_t acc_addr = tmem + (uint32_t)(a * BN);
        for (int kb = 0; kb < nk; ++kb, ++kbg) {
          const int s = (int)(kbg % STAGES);
          const uint32_t ph = (uint32_t)((kbg / STAGES) & 1);
          mbar_wait(&full[s], ph);
          asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
          const uint64_t da = A_MN ? smem_desc_mn_sw128(sA + s * TC_A_BYTES) : smem_desc_k_sw128(sA + s * TC_A_BYTES);
          const uint64_t db = B_MN ? smem_desc_mn_sw128(sB + s * B_BYTES) : smem_desc_k_sw128(sB + s * B_BYTES);
          // one K=16 step: K-major advances 32 B inside the 128-B swizzle atom; MN-major
          // advances two 8-row groups (2 x 1024 B)
          constexpr uint64_t stepA = A_MN ? 128 : 2, stepB = B_MN ? 128 : 2;
#pragma unroll
          for (int k = 0; k < TC_BK / 16; ++k) {
            const uint32_t acc = (kb > 0 || k > 0) ? 1u : 0u;
            asm volatile(
                "{\n\t.reg .pred p, e;\n\t"
                "elect.sync _|e, 0xffffffff;\n\t"
                "setp.ne.b32 p, %4, 0;\n\t"
                "@e tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(acc_addr),
                "l"(da + stepA * k), "l"(db + stepB * k), "r"(idesc), "r"(acc)
                : "memory");
          }
          tc_commit_elect(&empty[s]);
        }
        if (nk > 0)
          tc_commit_elect(&tfull[a]);
        else if (lane == 0)
          mbar_arrive(&tfull[a]);                   // empty K slice: the epilogue writes zeros
        __syncwarp();
      }
    }
  } else {                                          // ===== epilogue: warps 2..5
    // TMEM -> registers -> per-warp smem transpose -> coalesced row-segment stores:
    // each 32-column chunk of the warp's 32 rows leaves as 128-byte row segments.
    const int lane_base = 32 * (warp % 4);          // TMEM lanes of this warp
    float* stage = (float*)(tmem_slot + 4) + (warp - 2) * (32 * TC_EPI_LD);
    const bool vec_ok = (p.N % 4) == 0;
    const float* bias = p.has_bias ? res<float>(p.bias) : nullptr;
    int li = 0;
    for (long long it = blockIdx.x; it < items; it += gridDim.x, ++li) {
      int m0, n0, split, kb0, nk;
      decode(it, m0, n0, split, kb0, nk);
      const int a = li & 1;
      const uint32_t aph = (uint32_t)((li >> 1) & 1);
      const int bi = (int)(((it / splits) / phases) / (tiles_m * tiles_n));
      float* C = (p.raw != nullptr ? p.raw + (long long)split * p.M * p.N : Cout) + (long long)bi * p.c_bstride;
      const int cph = (int)((it / splits) % phases);
      mbar_wait(&tfull[a], aph);
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      // TMEM loads software-pipelined one 32-column chunk ahead: chunk c+32 streams out of
      // TMEM while chunk c goes through the smem transpose and the global stores
      auto tload = [&](uint32_t (&r)[32], int c) {
        if (nk > 0) {
          const uint32_t taddr = tmem + ((uint32_t)lane_base << 16) + (uint32_t)(a * BN + c);
          asm volatile(
              "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
              "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
              : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
                "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]),
                "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]),
                "=r"(r[23]), "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]),
                "=r"(r[30]), "=r"(r[31])
              : "r"(taddr));
        } else {
#pragma unroll
          for (int i = 0; i < 32; ++i) r[i] = 0u;
        }
      };
      auto tstore = [&](const uint32_t (&r)[32], int c) {
        if (n0 + c >= p.N) return;                   // chunk entirely past the last column
        float* srow = stage + lane * TC_EPI_LD;
#pragma unroll
        for (int i = 0; i < 32; i += 4)
          *(float4*)(srow + i) = make_float4(__uint_as_float(r[i]), __uint_as_float(r[i + 1]),
                                             __uint_as_float(r[i + 2]), __uint_as_float(r[i + 3]));
        __syncwarp();
        const int sub = lane >> 3, col = (lane & 7) * 4;   // 4 rows x 8 float4 per instruction
        const long long gcol = (long long)n0 + c + col;
        // fused bias_add: this lane's four columns, loaded once per chunk (not per row)
        float4 bv = make_float4(0.f, 0.f, 0.f, 0.f);
        if (bias != nullptr && gcol < p.N) {
          if (vec_ok && gcol + 4 <= p.N) {
            bv = __ldg((const float4*)(bias + gcol));
          } else {
            bv.x = __ldg(bias + gcol);
            if (gcol + 1 < p.N) bv.y = __ldg(bias + gcol + 1);
            if (gcol + 2 < p.N) bv.z = __ldg(bias + gcol + 2);
            if (gcol + 3 < p.N) bv.w = __ldg(bias + gcol + 3);
          }
        }
#pragma unroll
        for (int q = 0; q < 8; ++q) {
          const int rr = q * 4 + sub;
          const long long grow = (long long)m0 + lane_base + rr;
          if (grow < p.M && gcol < p.N) {
            float4 v = *(const float4*)(stage + rr * TC_EPI_LD + col);
            long long orow = grow;
            if (AMODE == 2 && phases > 1) {          // sub-pixel conv2d_t: scatter to the output grid
              int pn, hy, wx;
              conv_pix(p.cv, grow, pn, hy, wx);
              const int py = cph / p.cv.so, px = cph - py * p.cv.so;
              orow = ((long long)pn * p.cv.Ho + (long long)hy * p.cv.so + py) * p.cv.Wo + (long long)wx * p.cv.so + px;
            }
            float* dst = C + orow * p.N + gcol;
            v.x += bv.x; v.y += bv.y; v.z += bv.z; v.w += bv.w;
            if constexpr (RED) {                     // gradient bucket member: reduce across ranks
              const int nv = (int)(p.N - gcol < 4 ? p.N - gcol : 4);
              red_store4(p.red, dst, v, vec_ok && gcol + 4 <= p.N, nv);
            } else if (vec_ok && gcol + 4 <= p.N) {
              *(float4*)dst = v;
            } else {
              dst[0] = v.x;
              if (gcol + 1 < p.N) dst[1] = v.y;
              if (gcol + 2 < p.N) dst[2] = v.z;
              if (gcol + 3 < p.N) dst[3] = v.w;
            }
          }
        }
        __syncwarp();
      };
      if (nk >= 0) {
        uint32_t ra[32], rb[32];
        tload(ra, 0);
        asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll 1
        for (int c = 0; c < BN; c += 64) {
          if (c + 32 < BN) tload(rb, c + 32);
          tstore(ra, c);
          asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
          if (c + 32 < BN) {
            if (c + 64 < BN) tload(ra, c + 64);
            tstore(rb, c + 32);
            asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
          }
        }
      }
      asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
      __syncwarp();
      if (lane == 0) mbar_arrive(&tempty[a]);       // accumulator buffer free for item li + 2
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 1) {
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(TMEM_COLS) : "memory");
  }
  if (p.raw == nullptr) publish_late(p.out, Cout);
}

// Split-K reduction: out[i] = sum of the S fp32 slices in slice order (deterministic).
struct SplitReduceParams {
  DevState* ds;
  const float* ws;
  long long n;               // M * N
  int splits;
  In a, b;                   // node operands (ping-pong output choice only)
  Out out;
  In bias;                   // has_bias: out[m][c] += bias[c] (fused bias_add), ncols = N
  int has_bias;
  long long ncols;
};
__global__ void __launch_bounds__(256) k_splitk_reduce(SplitReduceParams p) {
  COEX_PDL_ENTER();
  stamp(p.ds, SK_SPLITK);
  float* o = pick_out<float>(p.out, res<float>(p.a), p.b.cell || p.b.direct ? res<float>(p.b) : nullptr);
  publish_early(p.out, o);
  const float* bias = p.has_bias ? res<float>(p.bias) : nullptr;
  // slices start 16-byte aligned only when 4 | n; the bias's column groups need 4 | ncols
  const long long n4 = ((p.n % 4) == 0 && (bias == nullptr || p.ncols % 4 == 0)) ? p.n / 4 : 0;
  const long long stride = (long long)gridDim.x * blockDim.x;
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n4; i += stride) {
    float4 acc = ((const float4*)p.ws)[i];
    for (int s = 1; s < p.splits; ++s) {
      const float4 v = ((const float4*)(p.ws + (long long)s * p.n))[i];
      acc.x += v.x; acc.y += v.y; acc.z += v.z; acc.w += v.w;
    }
    if (bias != nullptr) {
      const float4 bv = *(const float4*)(bias + (i * 4) % p.ncols);
      acc.x += bv.x; acc.y += bv.y; acc.z += bv.z; acc.w += bv.w;
    }
    ((float4*)o)[i] = acc;
  }
  for (long long i = n4 * 4 + (long long)blockIdx.x * blockDim.x + threadIdx.x; i < p.n; i += stride) {
    float acc = p.ws[i];
    for (int s = 1; s < p.splits; ++s) acc += p.ws[(long long)s * p.n + i];
    if (bias != nullptr) acc += bias[i % p.ncols];
    o[i] = acc;
  }
  publish_late(p.out, o);
}

}  // namespace coex
