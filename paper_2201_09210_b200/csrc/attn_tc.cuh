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
  int H;                     // heads per row of the operand layout (1: [BH][T][64])
  long long rs;              // row pitch in floats (64, or H * 64 for the merged layout)
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

// issue-only TMEM load of 32 columns (completion: fa_ld_wait, then fa_ld_dep on the registers)
__device__ __forceinline__ void fa_ld32_issue(uint32_t taddr, uint32_t (&r)[32]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
      "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]), "=r"(r[8]),
        "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]), "=r"(r[16]),
        "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]),
        "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
      : "r"(taddr));
}
__device__ __forceinline__ void fa_ld_wait() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }
// empty volatile asm "redefining" the registers after the wait: their uses cannot move above it
__device__ __forceinline__ void fa_ld_dep(uint32_t (&r)[32]) {
  asm volatile(""
               : "+r"(r[0]), "+r"(r[1]), "+r"(r[2]), "+r"(r[3]), "+r"(r[4]), "+r"(r[5]), "+r"(r[6]), "+r"(r[7]),
                 "+r"(r[8]), "+r"(r[9]), "+r"(r[10]), "+r"(r[11]), "+r"(r[12]), "+r"(r[13]), "+r"(r[14]), "+r"(r[15]),
                 "+r"(r[16]), "+r"(r[17]), "+r"(r[18]), "+r"(r[19]), "+r"(r[20]), "+r"(r[21]), "+r"(r[22]),
                 "+r"(r[23]), "+r"(r[24]), "+r"(r[25]), "+r"(r[26]), "+r"(r[27]), "+r"(r[28]), "+r"(r[29]),
                 "+r"(r[30]), "+r"(r[31]));
}

// row t of head bh: [BH][T][64] (H == 1, rs == 64) or the merged [B][T][H*64] layout of the
// projections the heads are split from (H heads, row pitch rs = H * 64)
template <typename F>
__device__ __forceinline__ F* fa_row(F* base, const FaParams& p, int bh, long long t) {
  return base + ((long long)(bh / p.H) * p.T + t) * p.rs + (long long)(bh % p.H) * FA_D;
}

// ---- fp32 tile staging through the bulk-copy (TMA) engine.  The operands are fp32 rows
// reached through runtime cells (no static tensor map), so the loader warpgroup issues 1-D
// cp.async.bulk copies -- one 32 KB copy per tile when the head's rows are contiguous, else
// one 256-byte copy per row -- into a fp32 staging tile that completes on an mbarrier; the
// copies for block j+1 fly while block j is converted (smem -> bf16 swizzled smem) and used.
constexpr int FA_STG = FA_BLK * FA_D * 4;       // one fp32 [128][64] staging tile: 32 KB

__device__ __forceinline__ void fa_bulk(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   smem_u32(dst)),
               "l"(src), "r"(bytes), "r"(smem_u32(bar))
               : "memory");
}
// loader thread lt (0..127): rows [t0, t0 + 128) of head bh -> fp32 staging tile
__device__ __forceinline__ void fa_stage_issue(unsigned char* stg, const FaParams& p, const float* base, int bh,
                                               int t0, uint64_t* full, int lt) {
  if (p.rs == FA_D) {
    if (lt == 0) fa_bulk(stg, fa_row(base, p, bh, t0), FA_STG, full);
  } else {
    fa_bulk(stg + lt * (FA_D * 4), fa_row(base, p, bh, t0 + lt), FA_D * 4, full);
  }
}
// fp32 staging tile -> bf16 128-B-swizzled tile (128 loader threads; conflict-free both sides)
__device__ __forceinline__ void fa_convert(unsigned char* dst, const unsigned char* stg, int lt) {
#pragma unroll 4
  for (int u = lt; u < FA_BLK * 8; u += 128) {
    const int r = u >> 3, c = u & 7;
    const float4 a = *(const float4*)(stg + r * 256 + c * 32), b = *(const float4*)(stg + r * 256 + c * 32 + 16);
    __nv_bfloat162 v0 = __floats2bfloat162_rn(a.x, a.y), v1 = __floats2bfloat162_rn(a.z, a.w);
    __nv_bfloat162 v2 = __floats2bfloat162_rn(b.x, b.y), v3 = __floats2bfloat162_rn(b.z, b.w);
    uint4 o;
    o.x = *(uint32_t*)&v0; o.y = *(uint32_t*)&v1; o.z = *(uint32_t*)&v2; o.w = *(uint32_t*)&v3;
    *(uint4*)(dst + fa_sw(r, c)) = o;
  }
}
// one staged pair of tiles (a, b) for the next phase of `full`: expect, then issue
__device__ __forceinline__ void fa_stage_pair(unsigned char* stg, const FaParams& p, const float* a, const float* b,
                                              int bh, int ta, int tb, uint64_t* full, int lt) {
  if (lt == 0) mbar_expect_tx(full, (b ? 2 : 1) * FA_STG);
  fa_stage_issue(stg, p, a, bh, ta, full, lt);
  if (b) fa_stage_issue(stg + FA_STG, p, b, bh, tb, full, lt);
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
// One CTA per (head, PAIR of 128-query tiles 2i / 2i+1): the two tiles share every K / V block
// and run as a ping-pong on the tensor core -- while one softmax warpgroup works on its S
// block, the single MMA thread computes the other tile's S and P.V.  416 threads:
//   warps 0-3  softmax of tile A (query tile 2i, rows = TMEM lanes), warps 4-7 tile B (2i+1);
//   warps 8-11 loader (fp32 rows -> bf16 128-B-swizzled tiles, K / V double-buffered);
//   warp 12    MMA issuer (one elected thread).
// O accumulates in TMEM (P.V with accumulate); the running row max is kept lazily (log2
// domain, rescale of O / l only when a block raises it by more than FA_RESCALE, warp-uniform),
// so un-normalised probabilities stay below 2^FA_RESCALE.
// TMEM (512 columns): S_A 0-127 | S_B 128-255 | O_A 256-319 | O_B 320-383.
constexpr float FA_RESCALE = 8.f;

__device__ __forceinline__ float fa_ex2(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
__device__ __forceinline__ void fa_st32(uint32_t taddr, const float (&v)[32]) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,"
      "%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};" ::"r"(taddr),
      "f"(v[0]), "f"(v[1]), "f"(v[2]), "f"(v[3]), "f"(v[4]), "f"(v[5]), "f"(v[6]), "f"(v[7]), "f"(v[8]), "f"(v[9]),
      "f"(v[10]), "f"(v[11]), "f"(v[12]), "f"(v[13]), "f"(v[14]), "f"(v[15]), "f"(v[16]), "f"(v[17]), "f"(v[18]),
      "f"(v[19]), "f"(v[20]), "f"(v[21]), "f"(v[22]), "f"(v[23]), "f"(v[24]), "f"(v[25]), "f"(v[26]), "f"(v[27]),
      "f"(v[28]), "f"(v[29]), "f"(v[30]), "f"(v[31])
      : "memory");
}

// pass 1 over one S row (128 keys in TMEM, two 32-column loads per wait): raw maximum over
// the unmasked keys
template <bool DIAG>
__device__ __forceinline__ float fa_rowmax(uint32_t tS, int r) {
  float mx = -INFINITY;
#pragma unroll 1
  for (int c = 0; c < FA_BLK; c += 64) {
    uint32_t a[32], b[32];
    fa_ld32_issue(tS + c, a);
    fa_ld32_issue(tS + c + 32, b);
    fa_ld_wait();
    fa_ld_dep(a);
    fa_ld_dep(b);
#pragma unroll
    for (int i = 0; i < 32; ++i) {
      if (!DIAG || c + i <= r) mx = fmaxf(mx, __uint_as_float(a[i]));
      if (!DIAG || c + 32 + i <= r) mx = fmaxf(mx, __uint_as_float(b[i]));
    }
  }
  return mx;
}
// pass 2: P = 2^(s * sc2 - m) (bf16 into the swizzled P tile), returns the row sum
template <bool DIAG>
__device__ __forceinline__ float fa_rowexp(uint32_t tS, int r, float sc2, float m, unsigned char* sP) {
  float rs0 = 0.f, rs1 = 0.f;
#pragma unroll 1
  for (int c = 0; c < FA_BLK; c += 64) {
    uint32_t a[32], b[32];
    fa_ld32_issue(tS + c, a);
    fa_ld32_issue(tS + c + 32, b);
    fa_ld_wait();
    fa_ld_dep(a);
    fa_ld_dep(b);
    float v[32];
#pragma unroll
    for (int i = 0; i < 32; ++i) {
      v[i] = (!DIAG || c + i <= r) ? fa_ex2(fmaf(__uint_as_float(a[i]), sc2, -m)) : 0.f;
      rs0 += v[i];
    }
    fa_store_row32(sP, r, c, v);
#pragma unroll
    for (int i = 0; i < 32; ++i) {
      v[i] = (!DIAG || c + 32 + i <= r) ? fa_ex2(fmaf(__uint_as_float(b[i]), sc2, -m)) : 0.f;
      rs1 += v[i];
    }
    fa_store_row32(sP, r, c + 32, v);
  }
  return rs0 + rs1;
}

__global__ void __launch_bounds__(416, 1) k_fa_fwd(const __grid_constant__ FaParams p) {
  COEX_PDL_ENTER();
  stamp(p.ds, SK_ATTN);
  extern __shared__ __align__(1024) unsigned char fa_raw[];
  unsigned char* sm = (unsigned char*)(((uintptr_t)fa_raw + 1023) & ~(uintptr_t)1023);
  unsigned char* sQ = sm;                        // [2 tiles]
  unsigned char* sK = sm + 2 * FA_TILE;          // [2 buffers]
  unsigned char* sV = sm + 4 * FA_TILE;          // [2 buffers]
  unsigned char* sP = sm + 6 * FA_TILE;          // [2 tiles] x two 64-key sub-tiles
  unsigned char* stg = sm + 10 * FA_TILE;        // fp32 staging: K | V (first Q_A | Q_B)
  uint64_t* bar = (uint64_t*)(sm + 14 * FA_TILE);
  uint64_t *kv_full = bar, *kv_empty = bar + 2, *q_full = bar + 4, *s_full = bar + 5, *p_full = bar + 7,
           *o_done = bar + 9, *stg_full = bar + 11;
  uint32_t* tslot = (uint32_t*)(bar + 12);
  const int tid = threadIdx.x, warp = tid >> 5;
  const int nqb = p.T / FA_BLK, npair = (nqb + 1) / 2;
  const int pi = npair - 1 - (int)(blockIdx.x / p.BH);   // heaviest pairs first
  const int bh = (int)(blockIdx.x % p.BH);
  const int qA = 2 * pi;
  const bool hasB = qA + 1 < nqb;
  const int nk = hasB ? qA + 2 : qA + 1;                 // key blocks of the pair (tile t: qA + t + 1)
  float* O = pick_out<float>(p.out, res<float>(p.pa), res<float>(p.pb));
  publish_early(p.out, O);
  count_op(p.ds);
  if (tid == 0) {
    for (int i = 0; i < 2; ++i) {
      mbar_init(&kv_full[i], 128);
      mbar_init(&kv_empty[i], 1);
      mbar_init(&s_full[i], 1);
      mbar_init(&p_full[i], 128);
      mbar_init(&o_done[i], 1);
    }
    mbar_init(q_full, 128);
    mbar_init(stg_full, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 0) fa_tmem_alloc(tslot, 512);
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = *tslot;
  if (warp >= 8 && warp < 12) {                      // ===== loader warpgroup
    const float* Q = res<float>(p.q);
    const float* K = res<float>(p.k);
    const float* V = res<float>(p.v);
    const int lt = tid & 127;
    fa_stage_pair(stg, p, Q, hasB ? Q : nullptr, bh, qA * FA_BLK, (qA + 1) * FA_BLK, stg_full, lt);
    mbar_wait(stg_full, 0);
    fa_convert(sQ, stg, lt);
    if (hasB) fa_convert(sQ + FA_TILE, stg + FA_STG, lt);
    fa_bar(4, 128);                                  // staging drained
    fa_stage_pair(stg, p, K, V, bh, 0, 0, stg_full, lt);
    fa_publish(q_full);
    for (int j = 0; j < nk; ++j) {
      const int b = j & 1;
      mbar_wait(stg_full, (uint32_t)((j + 1) & 1));
      if (j >= 2) mbar_wait(&kv_empty[b], (uint32_t)(((j - 2) >> 1) & 1));
      fa_convert(sK + b * FA_TILE, stg, lt);
      fa_convert(sV + b * FA_TILE, stg + FA_STG, lt);
      fa_publish(&kv_full[b]);
      fa_bar(4, 128);
      if (j + 1 < nk) fa_stage_pair(stg, p, K, V, bh, (j + 1) * FA_BLK, (j + 1) * FA_BLK, stg_full, lt);
    }
  } else if (warp == 12) {                           // ===== MMA issuer
    if ((tid & 31) == 0) {
      constexpr uint32_t idS = idesc_bf16_f32(128, 128, false, false);
      constexpr uint32_t idO = idesc_bf16_f32(128, 64, false, true);
      const int ntile[2] = {qA + 1, qA + 2};
      auto pv = [&](int t, int j) {                  // O_t += P_t . V(j)
        mbar_wait(&p_full[t], (uint32_t)(j & 1));
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        const unsigned char* pt = sP + t * 2 * FA_TILE;
        const unsigned char* vb = sV + (j & 1) * FA_TILE;
#pragma unroll
        for (int k = 0; k < FA_BLK / 16; ++k)
          fa_mma(tmem + 256 + 64 * t, fa_desc(pt + (k >> 2) * FA_TILE, 16) + 2 * (k & 3), fa_desc(vb, 8192) + 128 * k,
                 idO, (j > 0 || k > 0) ? 1u : 0u);
        fa_commit(&o_done[t]);
      };
      mbar_wait(q_full, 0);
      for (int j = 0; j < nk; ++j) {
        const int b = j & 1;
        mbar_wait(&kv_full[b], (uint32_t)((j >> 1) & 1));
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        for (int t = 0; t < (hasB ? 2 : 1); ++t) {
          if (j > 0 && j - 1 < ntile[t]) pv(t, j - 1);
          if (j < ntile[t]) {
            fa_mma_k64(tmem + 128 * t, sQ + t * FA_TILE, sK + b * FA_TILE, idS, false);
            fa_commit(&s_full[t]);
          }
        }
        if (j > 0) fa_commit(&kv_empty[(j - 1) & 1]);
      }
      for (int t = 0; t < (hasB ? 2 : 1); ++t)
        if (ntile[t] == nk) pv(t, nk - 1);
    }
  } else if (warp < 4 || hasB) {                     // ===== softmax warpgroup t
    const int t = warp >> 2, r = tid & 127, qb = qA + t;
    const uint32_t lane = (uint32_t)((warp & 3) * 32) << 16;
    const uint32_t tS = tmem + lane + 128 * t, tO = tmem + lane + 256 + 64 * t;
    unsigned char* sPt = sP + t * 2 * FA_TILE;
    const float sc2 = p.scale * FA_LOG2E;
    float m = -INFINITY, l = 0.f;
    for (int j = 0; j <= qb; ++j) {
      mbar_wait(&s_full[t], (uint32_t)(j & 1));
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      const bool diag = j == qb;
      const float mx = (diag ? fa_rowmax<true>(tS, r) : fa_rowmax<false>(tS, r)) * sc2;
      bool waited = false;
      if (j == 0) {
        m = mx;
      } else {
        const bool need = mx > m + FA_RESCALE;
        if (__any_sync(0xffffffffu, need)) {         // warp-uniform: tcgen05.ld / st are collective
          mbar_wait(&o_done[t], (uint32_t)((j - 1) & 1));
          asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
          waited = true;
          const float alpha = need ? fa_ex2(m - mx) : 1.f;
          float v[32];
#pragma unroll
          for (int c = 0; c < FA_D; c += 32) {
            fa_ld32(tO + c, v);
#pragma unroll
            for (int i = 0; i < 32; ++i) v[i] *= alpha;
            fa_st32(tO + c, v);
          }
          asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
          l *= alpha;
          if (need) m = mx;
        }
      }
      if (j > 0 && !waited) mbar_wait(&o_done[t], (uint32_t)((j - 1) & 1));   // P_t free again
      l += diag ? fa_rowexp<true>(tS, r, sc2, m, sPt) : fa_rowexp<false>(tS, r, sc2, m, sPt);
      fa_proxy_fence();
      asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
      mbar_arrive(&p_full[t]);
    }
    mbar_wait(&o_done[t], (uint32_t)(qb & 1));         // the last P.V
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    // epilogue: O / l through this tile's P buffer (free now; 128 x 64 fp32 = 32 KB, float4
    // slots XOR-swizzled by row), coalesced row stores; lse = m + log2(l)
    const float inv = 1.f / l;
    p.lse[(long long)bh * p.T + qb * FA_BLK + r] = m + log2f(l);
    float4* stage = (float4*)sPt;
    {
      float v[32];
#pragma unroll
      for (int c = 0; c < FA_D; c += 32) {
        fa_ld32(tO + c, v);
#pragma unroll
        for (int i = 0; i < 32; i += 4)
          stage[r * 16 + (((c + i) >> 2) ^ (r & 15))] = make_float4(v[i] * inv, v[i + 1] * inv, v[i + 2] * inv,
                                                                     v[i + 3] * inv);
      }
    }
    fa_bar(1 + t, 128);
    for (int u = r; u < FA_BLK * 16; u += 128) {
      const int rr = u >> 4, c4 = u & 15;
      *(float4*)(fa_row(O, p, bh, qb * FA_BLK + rr) + c4 * 4) = stage[rr * 16 + (c4 ^ (rr & 15))];
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 0) fa_tmem_free(tmem, 512);
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
    const int bh = (int)(r / p.T);
    const long long t = r - (long long)bh * p.T;
    const float4 a = *(const float4*)(fa_row(dO, p, bh, t) + lane * 4), b = *(const float4*)(fa_row(O, p, bh, t) + lane * 4);
    float s = a.x * b.x + a.y * b.y + a.z * b.z + a.w * b.w;
#pragma unroll
    for (int off = 8; off > 0; off >>= 1) s += __shfl_xor_sync(0xffffffffu, s, off);
    if (lane == 0) p.delta[r] = s;
  }
}

// P and dS of one (query block, key block) pair from the S / dP accumulators: thread (row r,
// column half h) handles 64 keys -- the four 32-column TMEM loads (S, dP) issued together, one
// wait -- and writes bf16 P and dS rows into the two [128][128] tiles
template <bool WANT_P, bool DIAG>
__device__ __forceinline__ void fa_pds(uint32_t tS, uint32_t tdP, int r, int h, float lse2, float dl, float sc2,
                                       float scale, unsigned char* sP, unsigned char* sdS) {
  uint32_t s0[32], s1[32], d0[32], d1[32];
  const int c0 = h * 64;
  fa_ld32_issue(tS + c0, s0);
  fa_ld32_issue(tdP + c0, d0);
  fa_ld32_issue(tS + c0 + 32, s1);
  fa_ld32_issue(tdP + c0 + 32, d1);
  fa_ld_wait();
  fa_ld_dep(s0);
  fa_ld_dep(d0);
  fa_ld_dep(s1);
  fa_ld_dep(d1);
  auto half = [&](uint32_t (&sr)[32], uint32_t (&dr)[32], int c) {
    float pv[32], dv[32];
#pragma unroll
    for (int i = 0; i < 32; ++i) {
      const float pr = (!DIAG || c + i <= r) ? fa_ex2(fmaf(__uint_as_float(sr[i]), sc2, -lse2)) : 0.f;
      pv[i] = pr;
      dv[i] = (scale * pr) * (__uint_as_float(dr[i]) - dl);
    }
    if (WANT_P) fa_store_row32(sP, r, c, pv);
    fa_store_row32(sdS, r, c, dv);
  };
  half(s0, d0, c0);
  half(s1, d1, c0 + 32);
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
  unsigned char* stg = sm + 10 * FA_TILE;        // fp32 staging: Q | dO (first K | V)
  uint64_t* bar = (uint64_t*)(sm + 14 * FA_TILE);
  uint64_t *qd_full = bar, *qd_empty = bar + 2, *kv_full = bar + 4, *s_done = bar + 5, *o_done = bar + 6,
           *stg_full = bar + 7;
  uint32_t* tslot = (uint32_t*)(bar + 8);
  const int tid = threadIdx.x, warp = tid >> 5;
  const int nb = p.T / FA_BLK;
  const int kb = (int)(blockIdx.x / p.BH);       // key block (low = most query blocks: first)
  const int bh = (int)(blockIdx.x % p.BH);
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
    mbar_init(stg_full, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 0) fa_tmem_alloc(tslot, 512);
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = *tslot;
  const uint32_t tS = tmem, tdP = tmem + 128, tdV = tmem + 256, tdK = tmem + 320;
  if (tid >= 256) {                                  // ===== loader warpgroup
    const float* Q = res<float>(p.q);
    const float* dO = res<float>(p.dout);
    const int lt = tid & 127;
    fa_stage_pair(stg, p, res<float>(p.k), res<float>(p.v), bh, kb * FA_BLK, kb * FA_BLK, stg_full, lt);
    mbar_wait(stg_full, 0);
    fa_convert(sK, stg, lt);
    fa_convert(sV, stg + FA_STG, lt);
    fa_bar(4, 128);
    fa_stage_pair(stg, p, Q, dO, bh, kb * FA_BLK, kb * FA_BLK, stg_full, lt);
    fa_publish(kv_full);
    int it = 0;
    for (int qb = kb; qb < nb; ++qb, ++it) {
      const int b = it & 1;
      mbar_wait(stg_full, (uint32_t)((it + 1) & 1));
      if (it >= 2) mbar_wait(&qd_empty[b], (uint32_t)(((it - 2) >> 1) & 1));
      fa_convert(sQ + b * FA_TILE, stg, lt);
      fa_convert(sdO + b * FA_TILE, stg + FA_STG, lt);
      fa_publish(&qd_full[b]);
      fa_bar(4, 128);
      if (qb + 1 < nb) fa_stage_pair(stg, p, Q, dO, bh, (qb + 1) * FA_BLK, (qb + 1) * FA_BLK, stg_full, lt);
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
      if (qb == kb) fa_pds<true, true>(tS + lane, tdP + lane, r, h, lse2, dl, sc2, p.scale, sP, sdS);
      else fa_pds<true, false>(tS + lane, tdP + lane, r, h, lse2, dl, sc2, p.scale, sP, sdS);
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
      float* dst = fa_row(w ? dK : dV, p, bh, kb * FA_BLK + rr) + c4 * 4;
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
  unsigned char* stg = sm + 8 * FA_TILE;         // fp32 staging: K | V (first Q | dO)
  uint64_t* bar = (uint64_t*)(sm + 12 * FA_TILE);
  uint64_t *kv_full = bar, *kv_empty = bar + 2, *q_full = bar + 4, *s_done = bar + 5, *o_done = bar + 6,
           *stg_full = bar + 7;
  uint32_t* tslot = (uint32_t*)(bar + 8);
  const int tid = threadIdx.x, warp = tid >> 5;
  const int nb = p.T / FA_BLK;
  const int qb = nb - 1 - (int)(blockIdx.x / p.BH);
  const int bh = (int)(blockIdx.x % p.BH);
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
    mbar_init(stg_full, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 0) fa_tmem_alloc(tslot, 512);
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = *tslot;
  const uint32_t tS = tmem, tdP = tmem + 128, tdQ = tmem + 256;
  if (tid >= 256) {                                  // ===== loader warpgroup
    const float* K = res<float>(p.k);
    const float* V = res<float>(p.v);
    const int lt = tid & 127;
    fa_stage_pair(stg, p, res<float>(p.q), res<float>(p.dout), bh, qb * FA_BLK, qb * FA_BLK, stg_full, lt);
    mbar_wait(stg_full, 0);
    fa_convert(sQ, stg, lt);
    fa_convert(sdO, stg + FA_STG, lt);
    fa_bar(4, 128);
    fa_stage_pair(stg, p, K, V, bh, 0, 0, stg_full, lt);
    fa_publish(q_full);
    for (int kb = 0; kb <= qb; ++kb) {
      const int b = kb & 1;
      mbar_wait(stg_full, (uint32_t)((kb + 1) & 1));
      if (kb >= 2) mbar_wait(&kv_empty[b], (uint32_t)(((kb - 2) >> 1) & 1));
      fa_convert(sK + b * FA_TILE, stg, lt);
      fa_convert(sV + b * FA_TILE, stg + FA_STG, lt);
      fa_publish(&kv_full[b]);
      fa_bar(4, 128);
      if (kb + 1 <= qb) fa_stage_pair(stg, p, K, V, bh, (kb + 1) * FA_BLK, (kb + 1) * FA_BLK, stg_full, lt);
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
      if (kb == qb) fa_pds<false, true>(tS + lane, tdP + lane, r, h, lse2, dl, sc2, p.scale, nullptr, sdS);
      else fa_pds<false, false>(tS + lane, tdP + lane, r, h, lse2, dl, sc2, p.scale, nullptr, sdS);
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
      *(float4*)(fa_row(dQ, p, bh, qb * FA_BLK + rr) + c4 * 4) = *(const float4*)(stage + rr * 68 + c4 * 4);
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 0) fa_tmem_free(tmem, 512);
  publish_late(p.out, dQ);
}

// forward grid: one CTA per (head, pair of query tiles)
inline unsigned fa_fwd_blocks(const FaParams& p) { return (unsigned)(p.BH * ((p.T / FA_BLK + 1) / 2)); }

constexpr size_t kFaFwdSmem = 14 * FA_TILE + 1024 + 128;
constexpr size_t kFaKvSmem = 14 * FA_TILE + 1024 + 128;
constexpr size_t kFaQSmem = 12 * FA_TILE + 1024 + 128;

}  // namespace coex
