// gemm_tf32.cuh -- MATMUL of the fp32 precision mode on the tcgen05 tensor cores: 3xTF32.
//
// C[M,N] (fp32) = A[M,K] . B[K,N] (reference op: tensor.py:228-236) with the fp32 contract
// (<= 1e-5 relative, north_star).  A single TF32 product keeps 10 mantissa bits (~5e-4
// relative per product) -- not enough -- so every operand is split once into a TF32-exact
// high part and the fp32 remainder, x = hi + lo with hi = x with the low 13 mantissa bits
// cleared (exact in TF32 whatever rounding the tensor core applies to its inputs) and
// lo = x - hi (exact in fp32; its own TF32 rounding costs ~2^-22 of x).  The GEMM then
// accumulates  A_hi.B_hi + A_hi.B_lo + A_lo.B_hi  in the fp32 TMEM accumulator (the dropped
// A_lo.B_lo term is ~2^-22 relative): three tcgen05.mma kind::tf32 per K step.
//
// Measured (tools/tf32_err.py, B200): 2.1e-6 relative per op for K <= 3072 -- a floor set by
// the tensor core's own fp32 accumulation (adding the A_lo.B_lo term does not move it),
// growing with the accumulation length (2.3e-5 at K = 50257 in one chain, 7.5e-6 with chains
// of <= 1024: COEX_TF32_MAXK splits K).  FFMA: 5e-7.  The fp32 mode therefore keeps the SIMT
// kernel by default (the 1e-5 end-to-end gradient bar fails by ~2x with this path);
// COEX_TF32=1 selects it (~190-260 TFLOP/s vs the FFMA kernel's SIMT rate).
//
//   k_cvt_tf32   fp32 operand (as stored, or transposed through a 32 x 33 shared tile) ->
//                hi / lo planes [2][rows][pitch4(K)], K-major (B is written as B^T [N][K]).
//   k_gemm_tf32  the warp-specialised persistent GEMM of gemm_tc.cuh (TMA producer warp, MMA
//                warp with elect.sync issue, four epilogue warps, double-buffered TMEM
//                accumulators), operands as 3-D tensor maps {K, rows, plane}: one stage holds
//                A_hi, A_lo, B_hi, B_lo boxes of 32 fp32 (128 B, SWIZZLE_128B) x rows.
// Split-K slices are reduced by k_splitk_reduce like the bf16 path.
#pragma once
#include "gemm_tc.cuh"

namespace coex {

constexpr int TF_BK = 32;                       // fp32 / tf32 elements per 128-byte K block

template <int BN> struct TfCfg {
  static constexpr int STAGES = BN == 128 ? 3 : 4;
  static constexpr int A_BYTES = TC_BM * TF_BK * 4;   // one plane: 16 KB
  static constexpr int B_BYTES = BN * TF_BK * 4;
  static constexpr int STAGE_BYTES = 2 * (A_BYTES + B_BYTES);
  static constexpr int SMEM = STAGES * STAGE_BYTES + 1024 + 256 + TC_EPI_BYTES;
};

// K-major pitch of the tf32 planes (16-byte rows)
inline long long tf32_pitch(long long K) { return (K + 3) / 4 * 4; }

struct TfCvtParams {
  DevState* ds;
  In src[2];
  long long rows[2];          // output rows (M for A, N for B)
  long long K, ld;            // logical K and the planes' pitch
  int trans[2];               // 1: element (r, k) = src[k * rows + r]; 0: src[r * K + k]
  float* dst[2];              // hi plane; the lo plane follows at + rows * ld
};

__device__ __forceinline__ void tf32_split(float x, float& hi, float& lo) {
  hi = __uint_as_float(__float_as_uint(x) & 0xFFFFE000u);
  lo = x - hi;
}

__global__ void __launch_bounds__(256) k_cvt_tf32(TfCvtParams p) {
  COEX_PDL_ENTER();
  stamp(p.ds, SK_CVT);
  const bool w1 = blockIdx.y != 0;
  const float* s = res<float>(w1 ? p.src[1] : p.src[0]);
  float* hi = w1 ? p.dst[1] : p.dst[0];
  const long long R = w1 ? p.rows[1] : p.rows[0], K = p.K, ld = p.ld;
  float* lo = hi + R * ld;
  if (!(w1 ? p.trans[1] : p.trans[0])) {
    // 4 consecutive k per thread (one 16-byte store per plane)
    const long long per_row = ld / 4, total = R * per_row;
    const bool vec = (K % 4) == 0 && ld == K && ((uintptr_t)s & 15) == 0;
    for (long long u = (long long)blockIdx.x * blockDim.x + threadIdx.x; u < total;
         u += (long long)gridDim.x * blockDim.x) {
      const long long r = u / per_row, k = (u - r * per_row) * 4;
      float4 v;
      if (vec) {
        v = *(const float4*)(s + r * K + k);
      } else {
        v.x = k < K ? s[r * K + k] : 0.f;
        v.y = k + 1 < K ? s[r * K + k + 1] : 0.f;
        v.z = k + 2 < K ? s[r * K + k + 2] : 0.f;
        v.w = k + 3 < K ? s[r * K + k + 3] : 0.f;
      }
      float4 h, l;
      tf32_split(v.x, h.x, l.x);
      tf32_split(v.y, h.y, l.y);
      tf32_split(v.z, h.z, l.z);
      tf32_split(v.w, h.w, l.w);
      *(float4*)(hi + r * ld + k) = h;
      *(float4*)(lo + r * ld + k) = l;
    }
    return;
  }
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
      if (r < R && k < ld) {
        float h, l;
        tf32_split(tile[tx][j], h, l);
        hi[r * ld + k] = h;
        lo[r * ld + k] = l;
      }
    }
    __syncthreads();
  }
}

// Instruction descriptor kind::tf32: D=F32 (bit 4), A=TF32 (2 at bits 7-9), B=TF32 (2 at bits
// 10-12), K-major A/B, N>>3 at [17,23), M>>4 at [24,29).
__host__ __device__ constexpr uint32_t idesc_tf32_f32(int M, int N) {
  return (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
}

__device__ __forceinline__ void tf32_mma(uint32_t d, uint64_t da, uint64_t db, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p, e;\n\t"
      "elect.sync _|e, 0xffffffff;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}" ::"r"(d),
      "l"(da), "l"(db), "r"(idesc), "r"(acc)
      : "memory");
}

// tmA: {ld, M, 2} fp32 (hi / lo planes), box {32, 128, 1}; tmB: {ld, N, 2}, box {32, BN, 1}.
template <int BN>
__global__ void __launch_bounds__(TC_THREADS, 1) k_gemm_tf32(const __grid_constant__ TcGemmParams p) {
  COEX_PDL_ENTER();
  using Cfg = TfCfg<BN>;
  constexpr int STAGES = Cfg::STAGES;
  constexpr uint32_t TMEM_COLS = 2 * BN;
  stamp(p.ds, SK_MATMUL);
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  unsigned char* smem = (unsigned char*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  uint64_t* full = (uint64_t*)(smem + STAGES * Cfg::STAGE_BYTES);
  uint64_t* empty = full + STAGES;
  uint64_t* tfull = empty + STAGES;
  uint64_t* tempty = tfull + 2;
  uint32_t* tmem_slot = (uint32_t*)(tempty + 2);
  auto sAh = [&](int s) { return smem + s * Cfg::STAGE_BYTES; };
  auto sAl = [&](int s) { return smem + s * Cfg::STAGE_BYTES + Cfg::A_BYTES; };
  auto sBh = [&](int s) { return smem + s * Cfg::STAGE_BYTES + 2 * Cfg::A_BYTES; };
  auto sBl = [&](int s) { return smem + s * Cfg::STAGE_BYTES + 2 * Cfg::A_BYTES + Cfg::B_BYTES; };

  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  const long long tiles_n = (p.N + BN - 1) / BN;
  const long long tiles_m = (p.M + TC_BM - 1) / TC_BM;
  const int splits = p.splits > 1 ? p.splits : 1;
  const long long items = tiles_m * tiles_n * splits;
  const int nk_all = (int)((p.K + TF_BK - 1) / TF_BK);
  const long long group = (long long)TC_GROUP_M * tiles_n;
  auto decode = [&](long long it, int& m0, int& n0, int& split, int& kb0, int& nk) {
    split = (int)(it % splits);
    const long long t = it / splits;
    const long long first_m = (t / group) * TC_GROUP_M;
    const long long gm = min((long long)TC_GROUP_M, tiles_m - first_m);
    m0 = (int)((first_m + (t % group) % gm) * TC_BM);
    n0 = (int)(((t % group) / gm) * BN);
    kb0 = (int)((long long)nk_all * split / splits);
    nk = (int)((long long)nk_all * (split + 1) / splits) - kb0;
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
      mbar_init(&tempty[a], 4);
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
      long long kbg = 0;
      for (long long it = blockIdx.x; it < items; it += gridDim.x) {
        int m0, n0, split, kb0, nk;
        decode(it, m0, n0, split, kb0, nk);
        for (int kb = 0; kb < nk; ++kb, ++kbg) {
          const int s = (int)(kbg % STAGES);
          const uint32_t ph = (uint32_t)((kbg / STAGES) & 1);
          mbar_wait(&empty[s], ph ^ 1u);
          mbar_expect_tx(&full[s], Cfg::STAGE_BYTES);
          const int kk = (kb0 + kb) * TF_BK;
          tma_load_3d(sAh(s), &p.tmA, &full[s], kk, m0, 0);
          tma_load_3d(sAl(s), &p.tmA, &full[s], kk, m0, 1);
          tma_load_3d(sBh(s), &p.tmB, &full[s], kk, n0, 0);
          tma_load_3d(sBl(s), &p.tmB, &full[s], kk, n0, 1);
        }
      }
    }
  } else if (warp == 1) {                           // ===== MMA issuer (whole warp, elected lane)
    constexpr uint32_t idesc = idesc_tf32_f32(TC_BM, BN);
    long long kbg = 0;
    int li = 0;
    for (long long it = blockIdx.x; it < items; it += gridDim.x, ++li) {
      int m0, n0, split, kb0, nk;
      decode(it, m0, n0, split, kb0, nk);
      const int a = li & 1;
      mbar_wait(&tempty[a], (uint32_t)((li >> 1) & 1) ^ 1u);
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      const uint32_t acc_addr = tmem + (uint32_t)(a * BN);
      for (int kb = 0; kb < nk; ++kb, ++kbg) {
        const int s = (int)(kbg % STAGES);
        mbar_wait(&full[s], (uint32_t)((kbg / STAGES) & 1));
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        const uint64_t ah = smem_desc_k_sw128(sAh(s)), al = smem_desc_k_sw128(sAl(s));
        const uint64_t bh = smem_desc_k_sw128(sBh(s)), bl = smem_desc_k_sw128(sBl(s));
#pragma unroll
        for (int k = 0; k < TF_BK / 8; ++k) {      // K = 8 per MMA: 32 B inside the swizzle atom
          const uint32_t acc = (kb > 0 || k > 0) ? 1u : 0u;
          tf32_mma(acc_addr, al + 2 * k, bh + 2 * k, idesc, acc);   // small terms first
          tf32_mma(acc_addr, ah + 2 * k, bl + 2 * k, idesc, 1u);
          tf32_mma(acc_addr, ah + 2 * k, bh + 2 * k, idesc, 1u);
        }
        tc_commit_elect(&empty[s]);
      }
      if (nk > 0)
        tc_commit_elect(&tfull[a]);
      else if (lane == 0)
        mbar_arrive(&tfull[a]);
      __syncwarp();
    }
  } else {                                          // ===== epilogue: warps 2..5
    const int lane_base = 32 * (warp % 4);
    float* stage = (float*)(tmem_slot + 4) + (warp - 2) * (32 * TC_EPI_LD);
    const bool vec_ok = (p.N % 4) == 0;
    int li = 0;
    for (long long it = blockIdx.x; it < items; it += gridDim.x, ++li) {
      int m0, n0, split, kb0, nk;
      decode(it, m0, n0, split, kb0, nk);
      const int a = li & 1;
      float* C = p.raw != nullptr ? p.raw + (long long)split * p.M * p.N : Cout;
      mbar_wait(&tfull[a], (uint32_t)((li >> 1) & 1));
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
#pragma unroll 1
      for (int c = 0; c < BN; c += 32) {
        uint32_t r[32];
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
          asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
        } else {
#pragma unroll
          for (int i = 0; i < 32; ++i) r[i] = 0u;
        }
        if (n0 + c >= p.N) continue;
        float* srow = stage + lane * TC_EPI_LD;
#pragma unroll
        for (int i = 0; i < 32; i += 4)
          *(float4*)(srow + i) = make_float4(__uint_as_float(r[i]), __uint_as_float(r[i + 1]),
                                             __uint_as_float(r[i + 2]), __uint_as_float(r[i + 3]));
        __syncwarp();
        const int sub = lane >> 3, col = (lane & 7) * 4;
        const long long gcol = (long long)n0 + c + col;
#pragma unroll
        for (int q = 0; q < 8; ++q) {
          const int rr = q * 4 + sub;
          const long long grow = (long long)m0 + lane_base + rr;
          if (grow < p.M && gcol < p.N) {
            const float4 v = *(const float4*)(stage + rr * TC_EPI_LD + col);
            float* dst = C + grow * p.N + gcol;
            if (vec_ok && gcol + 4 <= p.N) {
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
      }
      asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
      __syncwarp();
      if (lane == 0) mbar_arrive(&tempty[a]);
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

}  // namespace coex
