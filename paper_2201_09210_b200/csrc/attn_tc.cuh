// attn_tc.cuh -- fused causal attention on the tcgen05 tensor cores (bf16 precision mode).
//
// The planner (planner.py _attn_groups) recognises one layer's hand-written attention in the
// step program -- forward  S = bmm_nt(q, k), P = causal_softmax(S, scale), O = bmm(P, v);
// backward dP = bmm_nt(dO, v), dS = softmax_grad(P, dP, scale), dQ = bmm(dS, k),
// dK = bmm_tn(dS, q), dV = bmm_tn(P, dO) (oracle/kernels.py transformer_kernel; extension op
// set) -- and runs it as flash attention: the [B*H, T, T] scores and
// probabilities never reach HBM.
//
//   k_fa_prep_qkv  q, k, v (fp32 rows, [BH][T][64] or the merged [B][T][H*64] projection
//                  layout) -> bf16 128 x 64 tiles stored in global memory in their exact
//                  128-B-swizzled shared-memory byte order, once per tensor.  Every attention
//                  CTA then moves a tile with ONE 16 KB cp.async.bulk copy (no conversion in
//                  the loaders; a tile is re-read by up to T/128 CTAs from L2).
//   k_fa_fwd       one CTA per (head, PAIR of 128-query tiles): two softmax warpgroups, one MMA
//                  thread, one loader thread.  S = Q.K^T in 64-key halves into double-buffered
//                  TMEM, online softmax (lazy rescale), P (bf16) to shared memory, O += P.V
//                  accumulated in TMEM.  Writes O and the per-row log2-sum-exp.
//   k_fa_prep_do   dO -> bf16 tiles, and delta = rowsum(dO * O) (= sum_j dP * P per row).
//   k_fa_bwd_kv    one CTA per (head, 128-key block): per query block at or after it, S and
//                  dP on the tensor cores, P = exp2(S*scale*log2e - lse) and
//                  dS = scale * P * (dP - delta) in registers, both to shared memory;
//                  dV += P^T.dO and dK += dS^T.Q accumulate in TMEM (the same shared tile
//                  serves K-major and MN-major operands -- only the descriptor differs).
//   k_fa_bwd_q     one CTA per (head, 128-query block): S, dP, dS again and dQ += dS.K.
//
// All three attention kernels are warp-specialised: compute warps (rows = TMEM lanes), one
// MMA-issuing thread, one bulk-copy loader thread; K / V (or Q / dO) tiles are triple-buffered,
// and the compute warps release the S / dP accumulators as soon as they hold them in
// registers, so the next block's MMAs overlap the softmax-type math.
//
// Head dim 64 and T a multiple of 128.  Operands rounded to bf16 exactly where the unfused
// bf16 path rounds them (every GEMM operand), accumulation fp32 (tolerance 2e-2, north_star).
#pragma once
#include "gemm_tc.cuh"

namespace coex {

constexpr int FA_BLK = 128;                   // query rows / keys per block
constexpr int FA_D = 64;                      // head dim
constexpr int FA_TILE = FA_BLK * FA_D * 2;    // one bf16 [128][64] 128-B-swizzled tile: 16 KB
constexpr int FA_NBUF = 3;                    // streamed-tile buffers
constexpr float FA_LOG2E = 1.4426950408889634f;
constexpr float FA_RESCALE = 8.f;             // lazy-rescale threshold (log2 units)

struct FaParams {
  DevState* ds;
  In q, k, v, o, dout;       // fp32 rows: element (bh, t, e) at fa_row(base, bh, t) + e
  int BH, T;
  int H;                     // heads per row of the operand layout (1: [BH][T][64])
  long long rs;              // row pitch in floats (64, or H * 64 for the merged layout)
  float scale;               // logits = scale * q.k
  float* lse;                // [BH][T] log2-domain row log-sum-exp of scale*q.k (fwd -> bwd)
  float* delta;              // [BH][T] rowsum(dO * O)
  unsigned char* tiles;      // bf16 swizzled tiles: q | k | v | dO, each BH * (T/128) * 16 KB
  Out out, out2, out3;       // fwd: O | bwd_kv: dK (out2), dV (out3) | bwd_q: dQ (out)
  In pa, pb;                 // ping-pong output choice of the node being written
  long long* dbg;            // non-null (COEX_FA_DBG, eager only): CTA 0 event clocks
  __nv_bfloat16* sh[3];      // bf16 copies for GEMM-only readers (fwd: O | bwd: dQ, dK, dV), same rows
};

// global tile (tensor w in q, k, v, dO = 0..3; head bh; block j)
__device__ __forceinline__ unsigned char* fa_tile(const FaParams& p, int w, int bh, int j) {
  const long long nb = p.T / FA_BLK;
  return p.tiles + (((long long)w * p.BH + bh) * nb + j) * FA_TILE;
}

// row t of head bh: [BH][T][64] (H == 1, rs == 64) or the merged [B][T][H*64] layout of the
// projections the heads are split from (H heads, row pitch rs = H * 64)
template <typename F>
__device__ __forceinline__ F* fa_row(F* base, const FaParams& p, int bh, long long t) {
  return base + ((long long)(bh / p.H) * p.T + t) * p.rs + (long long)(bh % p.H) * FA_D;
}

// fp32 float4 of row t, columns 4*c4.. -> the output and, when present, its bf16 copy
__device__ __forceinline__ void fa_store4(float* out, __nv_bfloat16* sh, const FaParams& p, int bh, long long t, int c4,
                                          float4 v) {
  *(float4*)(fa_row(out, p, bh, t) + c4 * 4) = v;
  if (sh != nullptr) {
    __nv_bfloat162 a = __floats2bfloat162_rn(v.x, v.y), b = __floats2bfloat162_rn(v.z, v.w);
    *(uint2*)(fa_row(sh, p, bh, t) + c4 * 4) = make_uint2(*(uint32_t*)&a, *(uint32_t*)&b);
  }
}

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

// MMA issue and commit are executed by a WHOLE warp (operands warp-uniform) with one lane
// elected inside the instruction sequence: the compiler keeps the descriptors on the uniform
// datapath, and an issue costs ~the tensor pipe's own time (probes/mma_probe.cu: a single-lane
// issuer pays ~82 cycles per MMA, warp-wide + elect ~55 at N=64 and 65 at N=128).
__device__ __forceinline__ void fa_mma(uint32_t d_tmem, uint64_t da, uint64_t db, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p, e;\n\t"
      "elect.sync _|e, 0xffffffff;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(d_tmem),
      "l"(da), "l"(db), "r"(idesc), "r"(acc)
      : "memory");
}
__device__ __forceinline__ void fa_commit(uint64_t* bar) {
  asm volatile(
      "{\n\t.reg .pred e;\n\telect.sync _|e, 0xffffffff;\n\t"
      "@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n\t}" ::"r"(smem_u32(bar))
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
__device__ __forceinline__ float fa_ex2(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

// one bf16 tile (16 KB, already in shared-memory byte order) global -> shared, completing on `bar`
__device__ __forceinline__ void fa_bulk(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   smem_u32(dst)),
               "l"(src), "r"(bytes), "r"(smem_u32(bar))
               : "memory");
}

// 32 consecutive keys [k0, k0 + 32) of one row r of a [128][128] bf16 probability-type tile
// stored as two K-major [128][64] swizzled sub-tiles (keys 0-63 | 64-127)
__device__ __forceinline__ void fa_store_row32(unsigned char* tile, int r, int k0, const float (&v)[32]) {
  unsigned char* sub = tile + (k0 >> 6) * FA_TILE;
  const int cbase = (k0 & 63) >> 3;
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    __nv_bfloat162 w0 = __floats2bfloat162_rn(v[8 * q + 0], v[8 * q + 1]);
    __nv_bfloat162 w1 = __floats2bfloat162_rn(v[8 * q + 2], v[8 * q + 3]);
    __nv_bfloat162 w2 = __floats2bfloat162_rn(v[8 * q + 4], v[8 * q + 5]);
    __nv_bfloat162 w3 = __floats2bfloat162_rn(v[8 * q + 6], v[8 * q + 7]);
    asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(smem_u32(sub + fa_sw(r, cbase + q))),
                 "r"(*(uint32_t*)&w0), "r"(*(uint32_t*)&w1), "r"(*(uint32_t*)&w2), "r"(*(uint32_t*)&w3)
                 : "memory");
  }
}
__device__ __forceinline__ void fa_store_row32u(unsigned char* tile, int r, int k0, const uint32_t (&v)[32]) {
  float f[32];
#pragma unroll
  for (int i = 0; i < 32; ++i) f[i] = __uint_as_float(v[i]);
  fa_store_row32(tile, r, k0, f);
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
// compute side of an MMA hand-off: the generic-proxy smem stores become visible to the tensor
// core's async proxy and the TMEM reads are ordered before the barrier, then arrive
__device__ __forceinline__ void fa_handoff(uint64_t* bar) {
  fa_proxy_fence();
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  mbar_arrive(bar);
}
__device__ __forceinline__ void fa_after_wait(uint64_t* bar, uint32_t parity) {
  mbar_wait(bar, parity);
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
}

// ============================================================== tile preparation
// fp32 rows [t0, t0 + 128) of head bh -> one bf16 tile in swizzled byte order; 8 threads per
// 256-byte row (coalesced reads), each writing one 16-byte chunk (coalesced 128-byte rows)
__device__ __forceinline__ void fa_tile_convert(unsigned char* dst, const FaParams& p, const float* base, int bh,
                                                int t0, int u) {
  const int r = u >> 3, c = u & 7;
  const float* s = fa_row(base, p, bh, t0 + r) + c * 8;
  const float4 a = *(const float4*)s, b = *(const float4*)(s + 4);
  __nv_bfloat162 v0 = __floats2bfloat162_rn(a.x, a.y), v1 = __floats2bfloat162_rn(a.z, a.w);
  __nv_bfloat162 v2 = __floats2bfloat162_rn(b.x, b.y), v3 = __floats2bfloat162_rn(b.z, b.w);
  uint4 o;
  o.x = *(uint32_t*)&v0; o.y = *(uint32_t*)&v1; o.z = *(uint32_t*)&v2; o.w = *(uint32_t*)&v3;
  *(uint4*)(dst + fa_sw(r, c)) = o;
}

// q, k, v -> tiles (grid.y = tensor); one 8-element unit per thread, grid-stride
__global__ void __launch_bounds__(256) k_fa_prep_qkv(const __grid_constant__ FaParams p) {
  COEX_PDL_ENTER();
  stamp(p.ds, SK_ATTN_DELTA);
  const int w = blockIdx.y;
  const float* base = res<float>(w == 0 ? p.q : w == 1 ? p.k : p.v);
  const int nb = p.T / FA_BLK;
  const long long units = (long long)p.BH * nb * FA_BLK * 8;
  for (long long g = (long long)blockIdx.x * blockDim.x + threadIdx.x; g < units;
       g += (long long)gridDim.x * blockDim.x) {
    const long long tile = g >> 10;
    const int bh = (int)(tile / nb), j = (int)(tile % nb);
    fa_tile_convert(fa_tile(p, w, bh, j), p, base, bh, j * FA_BLK, (int)(g & 1023));
  }
}

// dO -> tiles and delta[row] = rowsum(dO * O) (8 threads per row, shuffle-reduced)
__global__ void __launch_bounds__(256) k_fa_prep_do(const __grid_constant__ FaParams p) {
  COEX_PDL_ENTER();
  stamp(p.ds, SK_ATTN_DELTA);
  const float* dO = res<float>(p.dout);
  const float* O = res<float>(p.o);
  const int nb = p.T / FA_BLK;
  const long long units = (long long)p.BH * nb * FA_BLK * 8;     // multiple of 8: rows never split
  for (long long g = (long long)blockIdx.x * blockDim.x + threadIdx.x; g < units;
       g += (long long)gridDim.x * blockDim.x) {
    const long long tile = g >> 10;
    const int bh = (int)(tile / nb), j = (int)(tile % nb), u = (int)(g & 1023);
    const int r = u >> 3, c = u & 7;
    fa_tile_convert(fa_tile(p, 3, bh, j), p, dO, bh, j * FA_BLK, u);
    const float* a = fa_row(dO, p, bh, (long long)j * FA_BLK + r) + c * 8;
    const float* b = fa_row(O, p, bh, (long long)j * FA_BLK + r) + c * 8;
    const float4 a0 = *(const float4*)a, a1 = *(const float4*)(a + 4);
    const float4 b0 = *(const float4*)b, b1 = *(const float4*)(b + 4);
    float s = a0.x * b0.x + a0.y * b0.y + a0.z * b0.z + a0.w * b0.w + a1.x * b1.x + a1.y * b1.y + a1.z * b1.z +
              a1.w * b1.w;
    s += __shfl_xor_sync(0xffffffffu, s, 1);
    s += __shfl_xor_sync(0xffffffffu, s, 2);
    s += __shfl_xor_sync(0xffffffffu, s, 4);
    if (c == 0) p.delta[(long long)bh * p.T + (long long)j * FA_BLK + r] = s;
  }
}

// ============================================================== forward
// One 64-key half of an S row is read from TMEM once: the raw row maximum over the unmasked
// keys (key k0 + i of the 128-key block is masked when k0 + i > r), then in place
// P = 2^(s * sc2 - m) -> bf16 into the half's P sub-tile; returns the row sum.
template <bool DIAG>
__device__ __forceinline__ float fa_max64(const uint32_t (&a)[32], const uint32_t (&b)[32], int r, int k0) {
  float m0 = -INFINITY, m1 = -INFINITY;
#pragma unroll
  for (int i = 0; i < 32; ++i) {
    if (!DIAG || k0 + i <= r) m0 = fmaxf(m0, __uint_as_float(a[i]));
    if (!DIAG || k0 + 32 + i <= r) m1 = fmaxf(m1, __uint_as_float(b[i]));
  }
  return fmaxf(m0, m1);
}
template <bool DIAG>
__device__ __forceinline__ float fa_exp64(const uint32_t (&a)[32], const uint32_t (&b)[32], int r, int k0, float sc2,
                                          float m, unsigned char* sP) {
  float v[32], rs0 = 0.f, rs1 = 0.f;
#pragma unroll
  for (int i = 0; i < 32; ++i) {
    v[i] = (!DIAG || k0 + i <= r) ? fa_ex2(fmaf(__uint_as_float(a[i]), sc2, -m)) : 0.f;
    rs0 += v[i];
  }
  fa_store_row32(sP, r, 0, v);
#pragma unroll
  for (int i = 0; i < 32; ++i) {
    v[i] = (!DIAG || k0 + 32 + i <= r) ? fa_ex2(fmaf(__uint_as_float(b[i]), sc2, -m)) : 0.f;
    rs1 += v[i];
  }
  fa_store_row32(sP, r, 32, v);
  return rs0 + rs1;
}

// One CTA per (head, PAIR of 128-query tiles 2i / 2i+1): the two tiles share every K / V block
// and alternate on the tensor core.  320 threads:
//   warps 0-3  softmax of tile A (query tile 2i, rows = TMEM lanes), warps 4-7 tile B (2i+1);
//   warp 8     MMA issuer (one thread); warp 9 loader (one thread, bulk copies).
// The tensor core works in 64-key HALF blocks u = 2j + h: each tile has two S buffers in TMEM
// (S(u + 1) is computed while the softmax works on S(u)) and two P sub-tiles (P(u) is written
// while P.V(u - 1) may still read the other).  O accumulates in TMEM; the running row max is
// kept lazily (rescale of O / l only when a half raises it by more than FA_RESCALE, warp-
// uniform), so un-normalised probabilities stay below 2^FA_RESCALE.
// TMEM (512 columns): S_A 0-127 | S_B 128-255 | O_A 256-319 | O_B 320-383.
__global__ void __launch_bounds__(320, 1) k_fa_fwd(const __grid_constant__ FaParams p) {
  COEX_PDL_ENTER();
  stamp(p.ds, SK_ATTN);
  extern __shared__ __align__(1024) unsigned char fa_raw[];
  unsigned char* sm = (unsigned char*)(((uintptr_t)fa_raw + 1023) & ~(uintptr_t)1023);
  unsigned char* sQ = sm;                                // [2 tiles]
  unsigned char* sK = sm + 2 * FA_TILE;                  // [FA_NBUF]
  unsigned char* sV = sm + (2 + FA_NBUF) * FA_TILE;      // [FA_NBUF]
  unsigned char* sP = sm + (2 + 2 * FA_NBUF) * FA_TILE;  // [2 tiles] x two 64-key sub-tiles
  uint64_t* bar = (uint64_t*)(sm + (6 + 2 * FA_NBUF) * FA_TILE);
  // per tile t and half h: s_full[2t + h], p_full[2t + h], o_done[2t + h]
  uint64_t *kv_full = bar, *kv_empty = bar + FA_NBUF, *q_full = bar + 2 * FA_NBUF, *s_full = q_full + 1,
           *p_full = s_full + 4, *o_done = p_full + 4;
  uint32_t* tslot = (uint32_t*)(o_done + 4);
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
    for (int i = 0; i < FA_NBUF; ++i) {
      mbar_init(&kv_full[i], 1);
      mbar_init(&kv_empty[i], 1);
    }
    for (int i = 0; i < 4; ++i) {
      mbar_init(&s_full[i], 1);
      mbar_init(&p_full[i], 128);
      mbar_init(&o_done[i], 1);
    }
    mbar_init(q_full, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 0) fa_tmem_alloc(tslot, 512);
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = *tslot;
  if (warp == 9) {                                   // ===== loader (bulk copies of ready tiles)
    if ((tid & 31) == 0) {
      mbar_expect_tx(q_full, (hasB ? 2 : 1) * FA_TILE);
      fa_bulk(sQ, fa_tile(p, 0, bh, qA), FA_TILE, q_full);
      if (hasB) fa_bulk(sQ + FA_TILE, fa_tile(p, 0, bh, qA + 1), FA_TILE, q_full);
      for (int j = 0; j < nk; ++j) {
        const int b = j % FA_NBUF;
        if (j >= FA_NBUF) mbar_wait(&kv_empty[b], (uint32_t)((j / FA_NBUF - 1) & 1));
        mbar_expect_tx(&kv_full[b], 2 * FA_TILE);
        fa_bulk(sK + b * FA_TILE, fa_tile(p, 1, bh, j), FA_TILE, &kv_full[b]);
        fa_bulk(sV + b * FA_TILE, fa_tile(p, 2, bh, j), FA_TILE, &kv_full[b]);
      }
    }
  } else if (warp == 8) {                            // ===== MMA issuer
    {                                              // whole warp: uniform descriptors
      constexpr uint32_t idS = idesc_bf16_f32(128, 64, false, false);
      constexpr uint32_t idO = idesc_bf16_f32(128, 64, false, true);
      const int nt = hasB ? 2 : 1;
      const int U[2] = {2 * (qA + 1), 2 * (qA + 2)};   // half blocks of tile t
      const int Umax = 2 * nk;
      auto smma = [&](int t, int u) {                  // S_t(u) = Q_t . K(u/2)[half]^T -> buffer u & 1
        const unsigned char* kt = sK + ((u >> 1) % FA_NBUF) * FA_TILE + (u & 1) * (FA_TILE / 2);
        fa_mma_k64(tmem + 128 * t + 64 * (u & 1), sQ + t * FA_TILE, kt, idS, false);
        fa_commit(&s_full[2 * t + (u & 1)]);
      };
      auto pv = [&](int t, int u) {                    // O_t += P_t[half] . V(u/2)[half]
        fa_after_wait(&p_full[2 * t + (u & 1)], (uint32_t)((u >> 1) & 1));
        const unsigned char* pt = sP + (2 * t + (u & 1)) * FA_TILE;
        const unsigned char* vb = sV + ((u >> 1) % FA_NBUF) * FA_TILE;
#pragma unroll
        for (int k = 0; k < 4; ++k)
          fa_mma(tmem + 256 + 64 * t, fa_desc(pt, 16) + 2 * k, fa_desc(vb, 8192) + 128 * (4 * (u & 1) + k), idO,
                 (u > 0 || k > 0) ? 1u : 0u);
        fa_commit(&o_done[2 * t + (u & 1)]);
      };
      mbar_wait(q_full, 0);
      fa_after_wait(&kv_full[0], 0);
      for (int t = 0; t < nt; ++t) {
        smma(t, 0);
        smma(t, 1);
      }
      long long* dbg = (p.dbg && blockIdx.x == 0) ? p.dbg + 2048 : nullptr;
      for (int u = 1; u <= Umax; ++u) {
        const int un = u + 1;                          // S half issued this round
        if (dbg) dbg[4 * u] = clock64();
        if (un < Umax && (un & 1) == 0)
          fa_after_wait(&kv_full[(un >> 1) % FA_NBUF], (uint32_t)(((un >> 1) / FA_NBUF) & 1));
        if (dbg) dbg[4 * u + 1] = clock64();
        for (int t = 0; t < nt; ++t) {
          if (u - 1 < U[t]) pv(t, u - 1);
          if (dbg) dbg[4 * u + 2 + t] = clock64();
          if (un < U[t]) smma(t, un);
        }
        if ((u - 1) & 1) fa_commit(&kv_empty[((u - 1) >> 1) % FA_NBUF]);   // block (u-1)/2 consumed
      }
    }
  } else if (warp < 4 || hasB) {                     // ===== softmax warpgroup t
    const int t = warp >> 2, r = tid & 127, qb = qA + t;
    const uint32_t lane = (uint32_t)((warp & 3) * 32) << 16;
    const uint32_t tS = tmem + lane + 128 * t, tO = tmem + lane + 256 + 64 * t;
    unsigned char* sPt = sP + 2 * t * FA_TILE;
    const float sc2 = p.scale * FA_LOG2E;
    const int Ut = 2 * (qb + 1);
    long long* dbg = (p.dbg && blockIdx.x == 0 && r == 0) ? p.dbg + t * 1024 : nullptr;
    float m = -INFINITY, l = 0.f;
    for (int u = 0; u < Ut; ++u) {
      const int h = u & 1;
      if (dbg) dbg[4 * u] = clock64();
      fa_after_wait(&s_full[2 * t + h], (uint32_t)((u >> 1) & 1));
      if (dbg) dbg[4 * u + 1] = clock64();
      const bool diag = (u >> 1) == qb;
      uint32_t sa[32], sb[32];
      fa_ld32_issue(tS + 64 * h, sa);
      fa_ld32_issue(tS + 64 * h + 32, sb);
      fa_ld_wait();
      fa_ld_dep(sa);
      fa_ld_dep(sb);
      const float mx = (diag ? fa_max64<true>(sa, sb, r, 64 * h) : fa_max64<false>(sa, sb, r, 64 * h)) * sc2;
      bool waited = false;
      if (u == 0) {
        m = mx;
      } else {
        const bool need = mx > m + FA_RESCALE;
        if (__any_sync(0xffffffffu, need)) {         // warp-uniform: tcgen05.ld / st are collective
          fa_after_wait(&o_done[2 * t + (h ^ 1)], (uint32_t)(((u - 1) >> 1) & 1));   // every P.V so far
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
      if (dbg) dbg[4 * u + 2] = clock64();
      if (u >= 2 && !waited) mbar_wait(&o_done[2 * t + h], (uint32_t)(((u - 2) >> 1) & 1));   // sub-tile h free
      unsigned char* ph = sPt + h * FA_TILE;
      l += diag ? fa_exp64<true>(sa, sb, r, 64 * h, sc2, m, ph) : fa_exp64<false>(sa, sb, r, 64 * h, sc2, m, ph);
      fa_handoff(&p_full[2 * t + h]);
      if (dbg) dbg[4 * u + 3] = clock64();
    }
    fa_after_wait(&o_done[2 * t + 1], (uint32_t)(((Ut - 1) >> 1) & 1));   // the last P.V
    // epilogue: O / l through this tile's P buffer (free now: 2 sub-tiles = 128 x 64 fp32,
    // float4 slots XOR-swizzled by row), coalesced row stores; lse = m + log2(l)
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
      fa_store4(O, p.sh[0], p, bh, qb * FA_BLK + rr, c4, stage[rr * 16 + (c4 ^ (rr & 15))]);
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 0) fa_tmem_free(tmem, 512);
  publish_late(p.out, O);
}

// ============================================================== backward
// Compute thread (row r, key half h) of one (query block, key block) pair: S and dP (64 keys
// each) into registers -- four 32-column TMEM loads, one wait -- after which the accumulators
// may be overwritten; then P = 2^(s*sc2 - lse) and dS = scale * P * (dP - delta) in place.
__device__ __forceinline__ void fa_ld_sdp(uint32_t tS, uint32_t tdP, int h, uint32_t (&s0)[32], uint32_t (&s1)[32],
                                          uint32_t (&d0)[32], uint32_t (&d1)[32]) {
  fa_ld32_issue(tS + 64 * h, s0);
  fa_ld32_issue(tdP + 64 * h, d0);
  fa_ld32_issue(tS + 64 * h + 32, s1);
  fa_ld32_issue(tdP + 64 * h + 32, d1);
  fa_ld_wait();
  fa_ld_dep(s0);
  fa_ld_dep(d0);
  fa_ld_dep(s1);
  fa_ld_dep(d1);
}
template <bool DIAG>
__device__ __forceinline__ void fa_pds32(uint32_t (&s)[32], uint32_t (&d)[32], int r, int c, float lse2, float dl,
                                         float sc2, float scale) {
#pragma unroll
  for (int i = 0; i < 32; ++i) {
    const float pr = (!DIAG || c + i <= r) ? fa_ex2(fmaf(__uint_as_float(s[i]), sc2, -lse2)) : 0.f;
    s[i] = __float_as_uint(pr);
    d[i] = __float_as_uint((scale * pr) * (__uint_as_float(d[i]) - dl));
  }
}
template <bool DIAG>
__device__ __forceinline__ void fa_pds(uint32_t (&s0)[32], uint32_t (&s1)[32], uint32_t (&d0)[32], uint32_t (&d1)[32],
                                       int r, int h, float lse2, float dl, float sc2, float scale) {
  fa_pds32<DIAG>(s0, d0, r, 64 * h, lse2, dl, sc2, scale);
  fa_pds32<DIAG>(s1, d1, r, 64 * h + 32, lse2, dl, sc2, scale);
}

// dK, dV per key block.  320 threads: warps 0-7 = (query row r, key half h) of the S / dP
// tiles, warp 8 = MMA issuer, warp 9 = loader of the query blocks' Q and dO tiles.
// MMA order per query block i: [S(i), dP(i)] once the compute warps hold block i-1 in
// registers, then [dV += P(i-1)^T.dO(i-1), dK += dS(i-1)^T.Q(i-1)] once P / dS(i-1) are stored.
// TMEM: S 0-127 | dP 128-255 | dV 256-319 | dK 320-383.
__global__ void __launch_bounds__(320, 1) k_fa_bwd_kv(const __grid_constant__ FaParams p) {
  COEX_PDL_ENTER();
  stamp(p.ds, SK_ATTN_KV);
  extern __shared__ __align__(1024) unsigned char fa_raw[];
  unsigned char* sm = (unsigned char*)(((uintptr_t)fa_raw + 1023) & ~(uintptr_t)1023);
  unsigned char* sK = sm;
  unsigned char* sV = sm + FA_TILE;
  unsigned char* sQ = sm + 2 * FA_TILE;                  // [FA_NBUF]
  unsigned char* sdO = sm + (2 + FA_NBUF) * FA_TILE;     // [FA_NBUF]
  unsigned char* sP = sm + (2 + 2 * FA_NBUF) * FA_TILE;  // [128 q][128 keys] (two sub-tiles)
  unsigned char* sdS = sP + 2 * FA_TILE;                 // same
  uint64_t* bar = (uint64_t*)(sm + (6 + 2 * FA_NBUF) * FA_TILE);
  uint64_t *qd_full = bar, *qd_empty = bar + FA_NBUF, *kv_full = bar + 2 * FA_NBUF, *s_done = kv_full + 1,
           *s_free = kv_full + 2, *p_ready = kv_full + 3, *pd_free = kv_full + 4, *o_done = kv_full + 5;
  uint32_t* tslot = (uint32_t*)(o_done + 1);
  const int tid = threadIdx.x, warp = tid >> 5;
  const int nb = p.T / FA_BLK;
  const int kb = (int)(blockIdx.x / p.BH);       // key block (low = most query blocks: first)
  const int bh = (int)(blockIdx.x % p.BH);
  const int nit = nb - kb;
  float* dK = pick_out<float>(p.out2, res<float>(p.pa), res<float>(p.pb));
  float* dV = pick_out<float>(p.out3, res<float>(p.pa), res<float>(p.pb));
  publish_early(p.out2, dK);
  publish_early(p.out3, dV);
  count_op(p.ds);
  if (tid == 0) {
    for (int i = 0; i < FA_NBUF; ++i) {
      mbar_init(&qd_full[i], 1);
      mbar_init(&qd_empty[i], 1);
    }
    mbar_init(kv_full, 1);
    mbar_init(s_done, 1);
    mbar_init(s_free, 256);
    mbar_init(p_ready, 256);
    mbar_init(pd_free, 1);
    mbar_init(o_done, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 0) fa_tmem_alloc(tslot, 512);
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = *tslot;
  const uint32_t tS = tmem, tdP = tmem + 128, tdV = tmem + 256, tdK = tmem + 320;
  if (warp == 9) {                                   // ===== loader
    if ((tid & 31) == 0) {
      mbar_expect_tx(kv_full, 2 * FA_TILE);
      fa_bulk(sK, fa_tile(p, 1, bh, kb), FA_TILE, kv_full);
      fa_bulk(sV, fa_tile(p, 2, bh, kb), FA_TILE, kv_full);
      for (int i = 0; i < nit; ++i) {
        const int b = i % FA_NBUF;
        if (i >= FA_NBUF) mbar_wait(&qd_empty[b], (uint32_t)((i / FA_NBUF - 1) & 1));
        mbar_expect_tx(&qd_full[b], 2 * FA_TILE);
        fa_bulk(sQ + b * FA_TILE, fa_tile(p, 0, bh, kb + i), FA_TILE, &qd_full[b]);
        fa_bulk(sdO + b * FA_TILE, fa_tile(p, 3, bh, kb + i), FA_TILE, &qd_full[b]);
      }
    }
  } else if (warp == 8) {                            // ===== MMA issuer
    {                                              // whole warp: uniform descriptors
      constexpr uint32_t idS = idesc_bf16_f32(128, 128, false, false);
      constexpr uint32_t idKV = idesc_bf16_f32(128, 64, true, true);
      auto kvmma = [&](int i) {                      // dV += P^T . dO(i), dK += dS^T . Q(i)
        fa_after_wait(p_ready, (uint32_t)(i & 1));
        // A = the [q][keys] tile read MN-major (M = keys in two 64-key blocks 16 KB apart, K =
        // query rows: steps of 16 rows = 2048 B); B = the [q][64] tile read MN-major (N = 64)
        const unsigned char* qbuf = sQ + (i % FA_NBUF) * FA_TILE;
        const unsigned char* obuf = sdO + (i % FA_NBUF) * FA_TILE;
#pragma unroll
        for (int k = 0; k < FA_BLK / 16; ++k) {
          const uint32_t acc = (i > 0 || k > 0) ? 1u : 0u;
          fa_mma(tdV, fa_desc(sP, FA_TILE) + 128 * k, fa_desc(obuf, 8192) + 128 * k, idKV, acc);
          fa_mma(tdK, fa_desc(sdS, FA_TILE) + 128 * k, fa_desc(qbuf, 8192) + 128 * k, idKV, acc);
        }
        fa_commit(pd_free);
        fa_commit(&qd_empty[i % FA_NBUF]);
      };
      fa_after_wait(kv_full, 0);
      for (int i = 0; i < nit; ++i) {
        const int b = i % FA_NBUF;
        fa_after_wait(&qd_full[b], (uint32_t)((i / FA_NBUF) & 1));
        if (i > 0) fa_after_wait(s_free, (uint32_t)((i - 1) & 1));
        fa_mma_k64(tS, sQ + b * FA_TILE, sK, idS, false);       // S = Q . K^T
        fa_mma_k64(tdP, sdO + b * FA_TILE, sV, idS, false);     // dP = dO . V^T
        fa_commit(s_done);
        if (i > 0) kvmma(i - 1);
      }
      kvmma(nit - 1);
      fa_commit(o_done);
    }
  } else {                                           // ===== compute warps
    const int r = tid & 127, h = tid >> 7;
    const uint32_t lane = (uint32_t)((warp & 3) * 32) << 16;
    const float sc2 = p.scale * FA_LOG2E;
    for (int i = 0; i < nit; ++i) {
      const int qb = kb + i;
      const long long row = (long long)bh * p.T + qb * FA_BLK + r;
      const float lse2 = p.lse[row], dl = p.delta[row];
      uint32_t s0[32], s1[32], d0[32], d1[32];
      fa_after_wait(s_done, (uint32_t)(i & 1));
      fa_ld_sdp(tS + lane, tdP + lane, h, s0, s1, d0, d1);
      asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
      mbar_arrive(s_free);                           // S / dP accumulators may be overwritten
      if (qb == kb) fa_pds<true>(s0, s1, d0, d1, r, h, lse2, dl, sc2, p.scale);
      else fa_pds<false>(s0, s1, d0, d1, r, h, lse2, dl, sc2, p.scale);
      if (i > 0) mbar_wait(pd_free, (uint32_t)((i - 1) & 1));   // previous dV / dK MMAs retired
      fa_store_row32u(sP, r, 64 * h, s0);
      fa_store_row32u(sP, r, 64 * h + 32, s1);
      fa_store_row32u(sdS, r, 64 * h, d0);
      fa_store_row32u(sdS, r, 64 * h + 32, d1);
      fa_handoff(p_ready);
    }
    fa_after_wait(o_done, 0);
    // epilogue: warps 0-3 dV, warps 4-7 dK (row = key), staged through shared memory
    float* stage = (float*)sQ + h * (FA_BLK * 68);  // two [128][68] fp32 stages (68 KB over sQ..sdO)
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
      fa_store4(w ? dK : dV, w ? p.sh[1] : p.sh[2], p, bh, kb * FA_BLK + rr, c4,
                *(const float4*)((float*)sQ + w * (FA_BLK * 68) + rr * 68 + c4 * 4));
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 0) fa_tmem_free(tmem, 512);
  publish_late(p.out2, dK);
  publish_late(p.out3, dV);
}

// dQ per query block.  320 threads: warps 0-7 compute, warp 8 MMA issuer, warp 9 loader of
// the key blocks' K and V tiles.  TMEM: S 0-127 | dP 128-255 | dQ 256-319.
__global__ void __launch_bounds__(320, 1) k_fa_bwd_q(const __grid_constant__ FaParams p) {
  COEX_PDL_ENTER();
  stamp(p.ds, SK_ATTN_Q);
  extern __shared__ __align__(1024) unsigned char fa_raw[];
  unsigned char* sm = (unsigned char*)(((uintptr_t)fa_raw + 1023) & ~(uintptr_t)1023);
  unsigned char* sQ = sm;
  unsigned char* sdO = sm + FA_TILE;
  unsigned char* sK = sm + 2 * FA_TILE;                  // [FA_NBUF]
  unsigned char* sV = sm + (2 + FA_NBUF) * FA_TILE;      // [FA_NBUF]
  unsigned char* sdS = sm + (2 + 2 * FA_NBUF) * FA_TILE; // [128 q][128 keys]
  uint64_t* bar = (uint64_t*)(sm + (4 + 2 * FA_NBUF) * FA_TILE);
  uint64_t *kv_full = bar, *kv_empty = bar + FA_NBUF, *q_full = bar + 2 * FA_NBUF, *s_done = q_full + 1,
           *s_free = q_full + 2, *p_ready = q_full + 3, *pd_free = q_full + 4, *o_done = q_full + 5;
  uint32_t* tslot = (uint32_t*)(o_done + 1);
  const int tid = threadIdx.x, warp = tid >> 5;
  const int nb = p.T / FA_BLK;
  const int qb = nb - 1 - (int)(blockIdx.x / p.BH);
  const int bh = (int)(blockIdx.x % p.BH);
  float* dQ = pick_out<float>(p.out, res<float>(p.pa), res<float>(p.pb));
  publish_early(p.out, dQ);
  count_op(p.ds);
  if (tid == 0) {
    for (int i = 0; i < FA_NBUF; ++i) {
      mbar_init(&kv_full[i], 1);
      mbar_init(&kv_empty[i], 1);
    }
    mbar_init(q_full, 1);
    mbar_init(s_done, 1);
    mbar_init(s_free, 256);
    mbar_init(p_ready, 256);
    mbar_init(pd_free, 1);
    mbar_init(o_done, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 0) fa_tmem_alloc(tslot, 512);
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = *tslot;
  const uint32_t tS = tmem, tdP = tmem + 128, tdQ = tmem + 256;
  if (warp == 9) {                                   // ===== loader
    if ((tid & 31) == 0) {
      mbar_expect_tx(q_full, 2 * FA_TILE);
      fa_bulk(sQ, fa_tile(p, 0, bh, qb), FA_TILE, q_full);
      fa_bulk(sdO, fa_tile(p, 3, bh, qb), FA_TILE, q_full);
      for (int kb = 0; kb <= qb; ++kb) {
        const int b = kb % FA_NBUF;
        if (kb >= FA_NBUF) mbar_wait(&kv_empty[b], (uint32_t)((kb / FA_NBUF - 1) & 1));
        mbar_expect_tx(&kv_full[b], 2 * FA_TILE);
        fa_bulk(sK + b * FA_TILE, fa_tile(p, 1, bh, kb), FA_TILE, &kv_full[b]);
        fa_bulk(sV + b * FA_TILE, fa_tile(p, 2, bh, kb), FA_TILE, &kv_full[b]);
      }
    }
  } else if (warp == 8) {                            // ===== MMA issuer
    {                                              // whole warp: uniform descriptors
      constexpr uint32_t idS = idesc_bf16_f32(128, 128, false, false);
      constexpr uint32_t idQ = idesc_bf16_f32(128, 64, false, true);
      auto qmma = [&](int kb) {                      // dQ += dS . K(kb)
        fa_after_wait(p_ready, (uint32_t)(kb & 1));
        // A = dS K-major (K = keys, two sub-tiles), B = K tile MN-major (N = 64)
        const unsigned char* kbuf = sK + (kb % FA_NBUF) * FA_TILE;
#pragma unroll
        for (int k = 0; k < FA_BLK / 16; ++k)
          fa_mma(tdQ, fa_desc(sdS + (k >> 2) * FA_TILE, 16) + 2 * (k & 3), fa_desc(kbuf, 8192) + 128 * k, idQ,
                 (kb > 0 || k > 0) ? 1u : 0u);
        fa_commit(pd_free);
        fa_commit(&kv_empty[kb % FA_NBUF]);
      };
      fa_after_wait(q_full, 0);
      for (int kb = 0; kb <= qb; ++kb) {
        const int b = kb % FA_NBUF;
        fa_after_wait(&kv_full[b], (uint32_t)((kb / FA_NBUF) & 1));
        if (kb > 0) fa_after_wait(s_free, (uint32_t)((kb - 1) & 1));
        fa_mma_k64(tS, sQ, sK + b * FA_TILE, idS, false);
        fa_mma_k64(tdP, sdO, sV + b * FA_TILE, idS, false);
        fa_commit(s_done);
        if (kb > 0) qmma(kb - 1);
      }
      qmma(qb);
      fa_commit(o_done);
    }
  } else {                                           // ===== compute warps
    const int r = tid & 127, h = tid >> 7;
    const uint32_t lane = (uint32_t)((warp & 3) * 32) << 16;
    const float sc2 = p.scale * FA_LOG2E;
    const long long row = (long long)bh * p.T + qb * FA_BLK + r;
    const float lse2 = p.lse[row], dl = p.delta[row];
    for (int kb = 0; kb <= qb; ++kb) {
      uint32_t s0[32], s1[32], d0[32], d1[32];
      fa_after_wait(s_done, (uint32_t)(kb & 1));
      fa_ld_sdp(tS + lane, tdP + lane, h, s0, s1, d0, d1);
      asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
      mbar_arrive(s_free);
      if (kb == qb) fa_pds<true>(s0, s1, d0, d1, r, h, lse2, dl, sc2, p.scale);
      else fa_pds<false>(s0, s1, d0, d1, r, h, lse2, dl, sc2, p.scale);
      if (kb > 0) mbar_wait(pd_free, (uint32_t)((kb - 1) & 1));   // previous dQ MMAs retired: dS free
      fa_store_row32u(sdS, r, 64 * h, d0);
      fa_store_row32u(sdS, r, 64 * h + 32, d1);
      fa_handoff(p_ready);
    }
    fa_after_wait(o_done, 0);
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
      fa_store4(dQ, p.sh[0], p, bh, qb * FA_BLK + rr, c4, *(const float4*)(stage + rr * 68 + c4 * 4));
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 0) fa_tmem_free(tmem, 512);
  publish_late(p.out, dQ);
}

// launch geometry
constexpr int FA_THREADS = 320;
inline unsigned fa_fwd_blocks(const FaParams& p) { return (unsigned)(p.BH * ((p.T / FA_BLK + 1) / 2)); }
inline unsigned fa_prep_blocks(const FaParams& p) {
  const long long units = (long long)p.BH * p.T * 8, b = (units + 255) / 256;
  return (unsigned)(b < 148 * 8 ? b : 148 * 8);   // 8 blocks per SM, grid-stride
}
inline size_t fa_tiles_bytes(int BH, int T) { return (size_t)4 * BH * T * FA_D * 2; }
constexpr size_t kFaFwdSmem = (6 + 2 * FA_NBUF) * FA_TILE + 1024 + 256;
constexpr size_t kFaKvSmem = (6 + 2 * FA_NBUF) * FA_TILE + 1024 + 256;
constexpr size_t kFaQSmem = (4 + 2 * FA_NBUF) * FA_TILE + 1024 + 256;

}  // namespace coex
