// attn_tc.cuh -- fused causal attention on the tcgen05 tensor cores (bf16 precision mode).
//
// The planner (planner.py _attn_groups) recognises one layer's hand-written attention in the
// step program -- forward  S = bmm_nt(q, k), P = causal_softmax(S, scale), O = bmm(P, v);
// backward dP = bmm_nt(dO, v), dS = softmax_grad(P, dP, scale), dQ = bmm(dS, k),
// dK = bmm_tn(dS, q), dV = bmm_tn(P, dO) (oracle/kernels.py transformer_kernel; extension op
// set) -- and runs it as flash attention: the [B*H, T, T] scores and
// probabilities never reach HBM.
//
//   k_fa_fwd    one CTA per (head, 128-query block), 128 threads = 128 query rows = 128 TMEM
//               lanes.  Per 128-key block: K / V tiles fp32 -> bf16 into 128-B-swizzled
//               shared memory (SIMT, coalesced), S = Q.K^T by one tcgen05.mma thread into TMEM,
//               online softmax from TMEM (tcgen05.ld, exp2, causal mask on the diagonal
//               block), P (bf16) to shared memory, P.V by tcgen05.mma into TMEM, rescaled
//               accumulation of O in registers.  Writes O and the per-row log2-sum-exp.
//   k_fa_delta  delta = rowsum(dO * O) (the softmax-gradient row dot, dO.O = sum_j dP*P).
//   k_fa_bwd_kv one CTA per (head, 128-key block), 256 threads: per query block at or after
//               it, S and dP on the tensor cores, P = exp2(S*scale*log2e - lse) and
//               dS = scale * P * (dP - delta) in registers, both to shared memory; dV += P^T.dO
//               and dK += dS^T.Q accumulate in TMEM (the same shared tile serves K-major and
//               MN-major operands -- only the descriptor differs).
//   k_fa_bwd_q  one CTA per (head, 128-query block): S, dP, dS again and dQ += dS.K in TMEM.
//
// Head dim 64 and T a multiple of 128.  Operands rounded to bf16 exactly where the unfused
// bf16 path rounds them (every GEMM operand), accumulation fp32 (tolerance 2e-2, north_star).
#pragma once
#include "gemm_tc.cuh"

namespace coex {

constexpr int FA_BLK = 128;                   // query rows / keys per block
constexpr int FA_D = 64;                      // head dim
constexpr int FA_TILE = FA_BLK * FA_D * 2;    // one bf16 [128][64] 128-B-swizzled tile: 16 KB
constexpr float FA_LOG2E = 1.4426950408889634f;

struct FaParams {
  DevState* ds;
  In q, k, v, o, dout;       // fp32 [BH][T][64] (element (bh, t, e) at bh*T*64 + t*64 + e)
  int BH, T;
  float scale;               // logits = scale * q.k
  float* lse;                // [BH][T] log2-domain row log-sum-exp of scale*q.k (fwd -> bwd)
  float* delta;              // [BH][T] rowsum(dO * O)
  Out out, out2, out3;       // fwd: O | bwd_kv: dK (out2), dV (out3) | bwd_q: dQ (out)
  In pa, pb;                 // ping-pong output choice of the node being written
};

// 128-B swizzle of a [rows][64 bf16] tile: 16-byte chunk c of row r at chunk c ^ (r & 7)
__device__ __forceinline__ uint32_t fa_sw(int r, int c) { return (uint32_t)(r * 128 + ((c ^ (r & 7)) << 4)); }

// SW128 smem descriptor with an explicit leading-byte offset (MN-major: the stride between
// 64-element MN blocks; K-major: unused) and SBO = 1024 (8 rows)
__device__ __forceinline__ uint64_t fa_desc(const void* p, uint32_t lbo) {
  uint64_t d = 0;
  d |= (uint64_t)((smem_u32(p) & 0x3FFFF) >> 4);
  d |= (uint64_t)((lbo >> 4) & 0x3FFF) << 16;
  d |= (uint64_t)(1024 >> 4) << 32;
  d |= (uint64_t)1 << 46;
  d |= (uint64_t)2 << 61;
  return d;
}

__device__ __forceinline__ void fa_mma(uint32_t d_tmem, uint64_t da, uint64_t db, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(d_tmem),
      "l"(da), "l"(db), "r"(idesc), "r"(acc)
      : "memory");
}
__device__ __forceinline__ void fa_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(bar))
               : "memory");
}
__device__ __forceinline__ void fa_ld32(uint32_t taddr, float (&v)[32]) {
  uint32_t r[32];
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
      "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]), "=r"(r[8]),
        "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]), "=r"(r[16]),
        "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]),
        "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
      : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
  for (int i = 0; i < 32; ++i) v[i] = __uint_as_float(r[i]);
}

// rows [t0, t0 + 128) of a fp32 [T][64] matrix -> bf16 swizzled tile; NT threads, coalesced
// (8 consecutive threads cover one 256-byte row)
template <int NT>
__device__ __forceinline__ void fa_load(unsigned char* dst, const float* src, int t0) {
#pragma unroll 4
  for (int u = threadIdx.x % NT; u < FA_BLK * 8; u += NT) {     // (loader warpgroup: its own index)
    const int r = u >> 3, c = u & 7;
    const float* s = src + (long long)(t0 + r) * FA_D + c * 8;
    const float4 a = *(const float4*)s, b = *(const float4*)(s + 4);
    __nv_bfloat162 v0 = __floats2bfloat162_rn(a.x, a.y), v1 = __floats2bfloat162_rn(a.z, a.w);
    __nv_bfloat162 v2 = __floats2bfloat162_rn(b.x, b.y), v3 = __floats2bfloat162_rn(b.z, b.w);
    uint4 o;
    o.x = *(uint32_t*)&v0; o.y = *(uint32_t*)&v1; o.z = *(uint32_t*)&v2; o.w = *(uint32_t*)&v3;
    *(uint4*)(dst + fa_sw(r, c)) = o;
  }
}

// 32 consecutive keys [k0, k0 + 32) of one row r of a [128][128] bf16 probability-type tile
// stored as two K-major [128][64] swizzled sub-tiles (keys 0-63 | 64-127)
__device__ __forceinline__ void fa_store_row32(unsigned char* tile, int r, int k0, const float (&v)[32]) {
  unsigned char* sub = tile + (k0 >> 6) * FA_TILE;
  const int cbase = (k0 & 63) >> 3;
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    uint4 o;
    __nv_bfloat162 w0 = __floats2bfloat162_rn(v[8 * q + 0], v[8 * q + 1]);
    __nv_bfloat162 w1 = __floats2bfloat162_rn(v[8 * q + 2], v[8 * q + 3]);
    __nv_bfloat162 w2 = __floats2bfloat162_rn(v[8 * q + 4], v[8 * q + 5]);
    __nv_bfloat162 w3 = __floats2bfloat162_rn(v[8 * q + 6], v[8 * q + 7]);
    o.x = *(uint32_t*)&w0; o.y = *(uint32_t*)&w1; o.z = *(uint32_t*)&w2; o.w = *(uint32_t*)&w3;
    *(uint4*)(sub + fa_sw(r, cbase + q)) = o;
  }
}

__device__ __forceinline__ void fa_proxy_fence() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

// K-major A [128 rows][64 K] x K-major B [N rows][64 K] over K = 64 (4 steps of 16)
__device__ __forceinline__ void fa_mma_k64(uint32_t d, const unsigned char* a, const unsigned char* b, uint32_t idesc,
                                           bool acc0) {
#pragma unroll
  for (int k = 0; k < FA_D / 16; ++k)
    fa_mma(d, fa_desc(a, 16) + 2 * k, fa_desc(b, 16) + 2 * k, idesc, (acc0 || k > 0) ? 1u : 0u);
}

// named barrier over `count` threads (id 0 is __syncthreads)
__device__ __forceinline__ void fa_bar(int id, int count) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(count) : "memory");
}
__device__ __forceinline__ void fa_tmem_alloc(uint32_t* slot, uint32_t cols) {
  asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(slot)), "r"(cols)
               : "memory");
  asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
}
__device__ __forceinline__ void fa_tmem_free(uint32_t tmem, uint32_t cols) {
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(cols) : "memory");
}
// loader side of a tile hand-off: the 128 loader threads' generic-proxy stores become visible
// to the tensor core's async proxy, then each arrives on the `full` barrier (count 128)
__device__ __forceinline__ void fa_publish(uint64_t* full) {
  fa_proxy_fence();
  mbar_arrive(full);
}

// Every kernel is warp-specialised: the LAST warpgroup (128 threads) converts the next tiles
// (fp32 global -> bf16 swizzled shared memory) into a second buffer while the compute
// warpgroups run softmax-type math on the current block and one thread issues the MMAs, so
// global-load latency hides behind the block in flight.

// ============================================================== forward
// 256 threads: warps 0-3 = the 128 query rows (TMEM lanes), warps 4-7 = loader.
__global__ void __launch_bounds__(256, 1) k_fa_fwd(const __grid_constant__ FaParams p) {
  COEX_PDL_ENTER();
  stamp(p.ds, SK_ATTN);
  extern __shared__ __align__(1024) unsigned char fa_raw[];
  unsigned char* sm = (unsigned char*)(((uintptr_t)fa_raw + 1023) & ~(uintptr_t)1023);
  unsigned char* sQ = sm;
  unsigned char* sK = sm + FA_TILE;              // [2] K buffers, then [2] V buffers
  unsigned char* sV = sm + 3 * FA_TILE;
  unsigned char* sP = sm + 5 * FA_TILE;          // two sub-tiles
  uint64_t* bar = (uint64_t*)(sm + 7 * FA_TILE);
  uint64_t *kv_full = bar, *kv_empty = bar + 2, *q_full = bar + 4, *s_done = bar + 5, *o_done = bar + 6;
  uint32_t* tslot = (uint32_t*)(bar + 8);
  const int tid = threadIdx.x, warp = tid >> 5;
  const int nqb = p.T / FA_BLK;
  const int qb = nqb - 1 - (int)(blockIdx.x / p.BH);   // heaviest query blocks first
  const int bh = (int)(blockIdx.x % p.BH);
  const long long hoff = (long long)bh * p.T * FA_D;
  float* O = pick_out<float>(p.out, res<float>(p.pa), res<float>(p.pb));
  publish_early(p.out, O);
  count_op(p.ds);
  if (tid == 0) {
    for (int i = 0; i < 2; ++i) {
      mbar_init(&kv_full[i], 128);
      mbar_init(&kv_empty[i], 1);
    }
    mbar_init(q_full, 128);
    mbar_init(s_done, 1);
    mbar_init(o_done, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 0) fa_tmem_alloc(tslot, 256);
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = *tslot;
  if (tid >= 128) {                                  // ===== loader warpgroup
    const float* K = res<float>(p.k) + hoff;
    const float* V = res<float>(p.v) + hoff;
    fa_load<128>(sQ, res<float>(p.q) + hoff, qb * FA_BLK);
    fa_publish(q_full);
    for (int j = 0; j <= qb; ++j) {
      const int b = j & 1;
      if (j >= 2) mbar_wait(&kv_empty[b], (uint32_t)(((j - 2) >> 1) & 1));
      fa_load<128>(sK + b * FA_TILE, K, j * FA_BLK);
      fa_load<128>(sV + b * FA_TILE, V, j * FA_BLK);
      fa_publish(&kv_full[b]);
    }
  } else {                                           // ===== softmax rows + MMA issuer
    const uint32_t lane = (uint32_t)(warp * 32) << 16;
    const uint32_t tS = tmem, tO = tmem + 128;
    constexpr uint32_t idS = idesc_bf16_f32(128, 128, false, false);
    constexpr uint32_t idO = idesc_bf16_f32(128, 64, false, true);
    const float sc2 = p.scale * FA_LOG2E;
    float o[FA_D];
#pragma unroll
    for (int e = 0; e < FA_D; ++e) o[e] = 0.f;
    float m = -INFINITY, l = 0.f;
    mbar_wait(q_full, 0);
    for (int j = 0; j <= qb; ++j) {
      const int b = j & 1;
      if (tid == 0) {
        mbar_wait(&kv_full[b], (uint32_t)((j >> 1) & 1));
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        fa_mma_k64(tS, sQ, sK + b * FA_TILE, idS, false);
        fa_commit(s_done);
      }
      mbar_wait(s_done, (uint32_t)(j & 1));
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      const bool diag = j == qb;
      float mx = m;
      float v[32];
#pragma unroll 1
      for (int c = 0; c < 128; c += 32) {
        fa_ld32(tS + lane + c, v);
#pragma unroll
        for (int i = 0; i < 32; ++i)
          if (!diag || c + i <= tid) mx = fmaxf(mx, v[i] * sc2);
      }
      const float alpha = exp2f(m - mx);           // m == -inf on the first block: alpha = 0
      float rs = 0.f;
#pragma unroll 1
      for (int c = 0; c < 128; c += 32) {
        fa_ld32(tS + lane + c, v);
#pragma unroll
        for (int i = 0; i < 32; ++i) {
          const float e = (!diag || c + i <= tid) ? exp2f(v[i] * sc2 - mx) : 0.f;
          v[i] = e;
          rs += e;
        }
        fa_store_row32(sP, tid, c, v);
      }
      l = l * alpha + rs;
      m = mx;
      fa_proxy_fence();
      asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
      fa_bar(1, 128);
      if (tid == 0) {
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        // O_blk = P . V: K = 128 keys in two 64-key sub-tiles of P; V is an MN-major B operand
        // ([keys][64] rows: K steps of 16 keys = 2048 B)
        const unsigned char* vb = sV + b * FA_TILE;
#pragma unroll
        for (int k = 0; k < FA_BLK / 16; ++k)
          fa_mma(tO, fa_desc(sP + (k >> 2) * FA_TILE, 16) + 2 * (k & 3), fa_desc(vb, 8192) + 128 * k, idO,
                 k > 0 ? 1u : 0u);
        fa_commit(o_done);
        fa_commit(&kv_empty[b]);                   // K / V buffer b free once these MMAs retire
      }
      mbar_wait(o_done, (uint32_t)(j & 1));
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
#pragma unroll
      for (int c = 0; c < FA_D; c += 32) {
        fa_ld32(tO + lane + c, v);
#pragma unroll
        for (int i = 0; i < 32; ++i) o[c + i] = o[c + i] * alpha + v[i];
      }
    }
    // epilogue: O / l through shared memory (coalesced row stores), lse = m + log2(l)
    const float inv = 1.f / l;
    p.lse[(long long)bh * p.T + qb * FA_BLK + tid] = m + log2f(l);
    float* stage = (float*)sK;                     // [128][68] fp32 over the K / V buffers (64 KB)
#pragma unroll
    for (int e = 0; e < FA_D; e += 4)
      *(float4*)(stage + tid * 68 + e) = make_float4(o[e] * inv, o[e + 1] * inv, o[e + 2] * inv, o[e + 3] * inv);
    fa_bar(1, 128);
    float* Ob = O + hoff + (long long)qb * FA_BLK * FA_D;
    for (int u = tid; u < FA_BLK * 16; u += 128) {
      const int r = u >> 4, c4 = u & 15;
      *(float4*)(Ob + r * FA_D + c4 * 4) = *(const float4*)(stage + r * 68 + c4 * 4);
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 0) fa_tmem_free(tmem, 256);
  publish_late(p.out, O);
}

// ============================================================== delta = rowsum(dO * O)
__global__ void __launch_bounds__(256) k_fa_delta(const __grid_constant__ FaParams p) {
  COEX_PDL_ENTER();
  stamp(p.ds, SK_ATTN_DELTA);
  const float* dO = res<float>(p.dout);
  const float* O = res<float>(p.o);
  const long long rows = (long long)p.BH * p.T;
  const int lane = threadIdx.x & 15;             // 16 threads per 64-wide row (one float4 each)
  for (long long r = ((long long)blockIdx.x * blockDim.x + threadIdx.x) >> 4; r < rows;
       r += ((long long)gridDim.x * blockDim.x) >> 4) {
    const float4 a = *(const float4*)(dO + r * FA_D + lane * 4), b = *(const float4*)(O + r * FA_D + lane * 4);
    float s = a.x * b.x + a.y * b.y + a.z * b.z + a.w * b.w;
#pragma unroll
    for (int off = 8; off > 0; off >>= 1) s += __shfl_xor_sync(0xffffffffu, s, off);
    if (lane == 0) p.delta[r] = s;
  }
}

// P and dS of one (query block, key block) pair from the S / dP accumulators: thread (row r,
// column half h) handles 64 keys; writes bf16 P and dS rows into the two [128][128] tiles
template <bool WANT_P>
__device__ __forceinline__ void fa_pds(uint32_t tS, uint32_t tdP, uint32_t lane, int r, int h, bool diag, float lse2,
                                       float dl, float sc2, float scale, unsigned char* sP, unsigned char* sdS) {
  float s[32], d[32];
#pragma unroll 1
  for (int c = h * 64; c < h * 64 + 64; c += 32) {
    fa_ld32(tS + lane + c, s);
    fa_ld32(tdP + lane + c, d);
#pragma unroll
    for (int i = 0; i < 32; ++i) {
      const float pr = (!diag || c + i <= r) ? exp2f(s[i] * sc2 - lse2) : 0.f;
      s[i] = pr;
      d[i] = scale * pr * (d[i] - dl);
    }
    if (WANT_P) fa_store_row32(sP, r, c, s);
    fa_store_row32(sdS, r, c, d);
  }
}

// ============================================================== backward: dK, dV per key block
// 384 threads: warps 0-7 = (query row r, key half h) of the S / dP tiles, warps 8-11 = loader
// of the next query block's Q and dO tiles (double-buffered).
__global__ void __launch_bounds__(384, 1) k_fa_bwd_kv(const __grid_constant__ FaParams p) {
  COEX_PDL_ENTER();
  stamp(p.ds, SK_ATTN_KV);
  extern __shared__ __align__(1024) unsigned char fa_raw[];
  unsigned char* sm = (unsigned char*)(((uintptr_t)fa_raw + 1023) & ~(uintptr_t)1023);
  unsigned char* sK = sm;
  unsigned char* sV = sm + FA_TILE;
  unsigned char* sQ = sm + 2 * FA_TILE;          // [2]
  unsigned char* sdO = sm + 4 * FA_TILE;         // [2]
  unsigned char* sP = sm + 6 * FA_TILE;          // [128 q][128 keys] (two sub-tiles)
  unsigned char* sdS = sm + 8 * FA_TILE;         // same
  uint64_t* bar = (uint64_t*)(sm + 10 * FA_TILE);
  uint64_t *qd_full = bar, *qd_empty = bar + 2, *kv_full = bar + 4, *s_done = bar + 5, *o_done = bar + 6;
  uint32_t* tslot = (uint32_t*)(bar + 8);
  const int tid = threadIdx.x, warp = tid >> 5;
  const int nb = p.T / FA_BLK;
  const int kb = (int)(blockIdx.x / p.BH);       // key block (low = most query blocks: first)
  const int bh = (int)(blockIdx.x % p.BH);
  const long long hoff = (long long)bh * p.T * FA_D;
  float* dK = pick_out<float>(p.out2, res<float>(p.pa), res<float>(p.pb));
  float* dV = pick_out<float>(p.out3, res<float>(p.pa), res<float>(p.pb));
  publish_early(p.out2, dK);
  publish_early(p.out3, dV);
  count_op(p.ds);
  if (tid == 0) {
    for (int i = 0; i < 2; ++i) {
      mbar_init(&qd_full[i], 128);
      mbar_init(&qd_empty[i], 1);
    }
    mbar_init(kv_full, 128);
    mbar_init(s_done, 1);
    mbar_init(o_done, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 0) fa_tmem_alloc(tslot, 512);
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = *tslot;
  const uint32_t tS = tmem, tdP = tmem + 128, tdV = tmem + 256, tdK = tmem + 320;
  if (tid >= 256) {                                  // ===== loader warpgroup
    const float* Q = res<float>(p.q) + hoff;
    const float* dO = res<float>(p.dout) + hoff;
    fa_load<128>(sK, res<float>(p.k) + hoff, kb * FA_BLK);
    fa_load<128>(sV, res<float>(p.v) + hoff, kb * FA_BLK);
    fa_publish(kv_full);
    int it = 0;
    for (int qb = kb; qb < nb; ++qb, ++it) {
      const int b = it & 1;
      if (it >= 2) mbar_wait(&qd_empty[b], (uint32_t)(((it - 2) >> 1) & 1));
      fa_load<128>(sQ + b * FA_TILE, Q, qb * FA_BLK);
      fa_load<128>(sdO + b * FA_TILE, dO, qb * FA_BLK);
      fa_publish(&qd_full[b]);
    }
  } else {                                           // ===== compute warpgroups + MMA issuer
    const int r = tid & 127, h = tid >> 7;
    const uint32_t lane = (uint32_t)((warp & 3) * 32) << 16;
    constexpr uint32_t idS = idesc_bf16_f32(128, 128, false, false);
    constexpr uint32_t idKV = idesc_bf16_f32(128, 64, true, true);
    const float sc2 = p.scale * FA_LOG2E;
    if (tid == 0) mbar_wait(kv_full, 0);
    int it = 0;
    for (int qb = kb; qb < nb; ++qb, ++it) {
      const int b = it & 1;
      const long long row = (long long)bh * p.T + qb * FA_BLK + r;
      const float lse2 = p.lse[row], dl = p.delta[row];
      if (tid == 0) {
        mbar_wait(&qd_full[b], (uint32_t)((it >> 1) & 1));
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        fa_mma_k64(tS, sQ + b * FA_TILE, sK, idS, false);      // S = Q . K^T
        fa_mma_k64(tdP, sdO + b * FA_TILE, sV, idS, false);    // dP = dO . V^T
        fa_commit(s_done);
      }
      // s_done also retires the previous block's dV / dK MMAs (issued earlier by the same
      // thread): sP / sdS are free to overwrite
      mbar_wait(s_done, (uint32_t)(it & 1));
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      fa_pds<true>(tS, tdP, lane, r, h, qb == kb, lse2, dl, sc2, p.scale, sP, sdS);
      fa_proxy_fence();
      asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
      fa_bar(1, 256);
      if (tid == 0) {
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        // dV += P^T . dO, dK += dS^T . Q: A = the [q][keys] tile read MN-major (M = keys in two
        // 64-key blocks 16 KB apart, K = query rows: steps of 16 rows = 2048 B); B = the
        // [q][64] tile read MN-major (N = head dim)
        const unsigned char* qbuf = sQ + b * FA_TILE;
        const unsigned char* obuf = sdO + b * FA_TILE;
#pragma unroll
        for (int k = 0; k < FA_BLK / 16; ++k) {
          const uint32_t acc = (it > 0 || k > 0) ? 1u : 0u;
          fa_mma(tdV, fa_desc(sP, FA_TILE) + 128 * k, fa_desc(obuf, 8192) + 128 * k, idKV, acc);
          fa_mma(tdK, fa_desc(sdS, FA_TILE) + 128 * k, fa_desc(qbuf, 8192) + 128 * k, idKV, acc);
        }
        fa_commit(&qd_empty[b]);
      }
    }
    if (tid == 0) fa_commit(o_done);
    mbar_wait(o_done, 0);
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    // epilogue: warps 0-3 dV, warps 4-7 dK (row = key), staged through shared memory
    float* stage = (float*)sQ + h * (FA_BLK * 68);  // two [128][68] fp32 stages (68 KB of sQ..sdS)
    {
      float v[32];
      const uint32_t tacc = h ? tdK : tdV;
#pragma unroll 1
      for (int c = 0; c < FA_D; c += 32) {
        fa_ld32(tacc + lane + c, v);
#pragma unroll
        for (int i = 0; i < 32; i += 4)
          *(float4*)(stage + r * 68 + c + i) = make_float4(v[i], v[i + 1], v[i + 2], v[i + 3]);
      }
    }
    fa_bar(1, 256);
    for (int u = tid; u < 2 * FA_BLK * 16; u += 256) {
      const int w = u / (FA_BLK * 16), rr = (u >> 4) & 127, c4 = u & 15;
      float* dst = (w ? dK : dV) + hoff + (long long)(kb * FA_BLK + rr) * FA_D + c4 * 4;
      *(float4*)dst = *(const float4*)((float*)sQ + w * (FA_BLK * 68) + rr * 68 + c4 * 4);
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 0) fa_tmem_free(tmem, 512);
  publish_late(p.out2, dK);
  publish_late(p.out3, dV);
}

// ============================================================== backward: dQ per query block
// 384 threads: warps 0-7 compute, warps 8-11 load the next key block's K and V tiles.
__global__ void __launch_bounds__(384, 1) k_fa_bwd_q(const __grid_constant__ FaParams p) {
  COEX_PDL_ENTER();
  stamp(p.ds, SK_ATTN_Q);
  extern __shared__ __align__(1024) unsigned char fa_raw[];
  unsigned char* sm = (unsigned char*)(((uintptr_t)fa_raw + 1023) & ~(uintptr_t)1023);
  unsigned char* sQ = sm;
  unsigned char* sdO = sm + FA_TILE;
  unsigned char* sK = sm + 2 * FA_TILE;          // [2]
  unsigned char* sV = sm + 4 * FA_TILE;          // [2]
  unsigned char* sdS = sm + 6 * FA_TILE;         // [128 q][128 keys]
  uint64_t* bar = (uint64_t*)(sm + 8 * FA_TILE);
  uint64_t *kv_full = bar, *kv_empty = bar + 2, *q_full = bar + 4, *s_done = bar + 5, *o_done = bar + 6;
  uint32_t* tslot = (uint32_t*)(bar + 8);
  const int tid = threadIdx.x, warp = tid >> 5;
  const int nb = p.T / FA_BLK;
  const int qb = nb - 1 - (int)(blockIdx.x / p.BH);
  const int bh = (int)(blockIdx.x % p.BH);
  const long long hoff = (long long)bh * p.T * FA_D;
  float* dQ = pick_out<float>(p.out, res<float>(p.pa), res<float>(p.pb));
  publish_early(p.out, dQ);
  count_op(p.ds);
  if (tid == 0) {
    for (int i = 0; i < 2; ++i) {
      mbar_init(&kv_full[i], 128);
      mbar_init(&kv_empty[i], 1);
    }
    mbar_init(q_full, 128);
    mbar_init(s_done, 1);
    mbar_init(o_done, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 0) fa_tmem_alloc(tslot, 512);
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = *tslot;
  const uint32_t tS = tmem, tdP = tmem + 128, tdQ = tmem + 256;
  if (tid >= 256) {                                  // ===== loader warpgroup
    const float* K = res<float>(p.k) + hoff;
    const float* V = res<float>(p.v) + hoff;
    fa_load<128>(sQ, res<float>(p.q) + hoff, qb * FA_BLK);
    fa_load<128>(sdO, res<float>(p.dout) + hoff, qb * FA_BLK);
    fa_publish(q_full);
    for (int kb = 0; kb <= qb; ++kb) {
      const int b = kb & 1;
      if (kb >= 2) mbar_wait(&kv_empty[b], (uint32_t)(((kb - 2) >> 1) & 1));
      fa_load<128>(sK + b * FA_TILE, K, kb * FA_BLK);
      fa_load<128>(sV + b * FA_TILE, V, kb * FA_BLK);
      fa_publish(&kv_full[b]);
    }
  } else {                                           // ===== compute warpgroups + MMA issuer
    const int r = tid & 127, h = tid >> 7;
    const uint32_t lane = (uint32_t)((warp & 3) * 32) << 16;
    constexpr uint32_t idS = idesc_bf16_f32(128, 128, false, false);
    constexpr uint32_t idQ = idesc_bf16_f32(128, 64, false, true);
    const float sc2 = p.scale * FA_LOG2E;
    const long long row = (long long)bh * p.T + qb * FA_BLK + r;
    const float lse2 = p.lse[row], dl = p.delta[row];
    if (tid == 0) mbar_wait(q_full, 0);
    for (int kb = 0; kb <= qb; ++kb) {
      const int b = kb & 1;
      if (tid == 0) {
        mbar_wait(&kv_full[b], (uint32_t)((kb >> 1) & 1));
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        fa_mma_k64(tS, sQ, sK + b * FA_TILE, idS, false);
        fa_mma_k64(tdP, sdO, sV + b * FA_TILE, idS, false);
        fa_commit(s_done);
      }
      mbar_wait(s_done, (uint32_t)(kb & 1));        // (also retires the previous dQ MMAs: sdS free)
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      fa_pds<false>(tS, tdP, lane, r, h, kb == qb, lse2, dl, sc2, p.scale, nullptr, sdS);
      fa_proxy_fence();
      asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
      fa_bar(1, 256);
      if (tid == 0) {
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        // dQ += dS . K: A = dS K-major (K = keys, two sub-tiles), B = K tile MN-major (N = 64)
        const unsigned char* kbuf = sK + b * FA_TILE;
#pragma unroll
        for (int k = 0; k < FA_BLK / 16; ++k)
          fa_mma(tdQ, fa_desc(sdS + (k >> 2) * FA_TILE, 16) + 2 * (k & 3), fa_desc(kbuf, 8192) + 128 * k, idQ,
                 (kb > 0 || k > 0) ? 1u : 0u);
        fa_commit(&kv_empty[b]);
      }
    }
    if (tid == 0) fa_commit(o_done);
    mbar_wait(o_done, 0);
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    float* stage = (float*)sK;                     // [128][68] fp32 over the K / V buffers
    if (h == 0) {
      float v[32];
#pragma unroll 1
      for (int c = 0; c < FA_D; c += 32) {
        fa_ld32(tdQ + lane + c, v);
#pragma unroll
        for (int i = 0; i < 32; i += 4)
          *(float4*)(stage + r * 68 + c + i) = make_float4(v[i], v[i + 1], v[i + 2], v[i + 3]);
      }
    }
    fa_bar(1, 256);
    for (int u = tid; u < FA_BLK * 16; u += 256) {
      const int rr = u >> 4, c4 = u & 15;
      *(float4*)(dQ + hoff + (long long)(qb * FA_BLK + rr) * FA_D + c4 * 4) = *(const float4*)(stage + rr * 68 + c4 * 4);
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 0) fa_tmem_free(tmem, 512);
  publish_late(p.out, dQ);
}

constexpr size_t kFaFwdSmem = 7 * FA_TILE + 1024 + 128;
constexpr size_t kFaKvSmem = 10 * FA_TILE + 1024 + 128;
constexpr size_t kFaQSmem = 8 * FA_TILE + 1024 + 128;

}  // namespace coex
