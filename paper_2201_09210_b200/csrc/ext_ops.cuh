// ext_ops.cuh -- sm_100a kernels of the extension op set for configs C2-C5
// (SURVEY §2.4, §8(a) row a*).  The reference has no such ops; the semantics
// these kernels implement are the builder's f64 restatement in
// oracle/kernels.py (ext_kernel), NHWC layout throughout.
//
// Convolutions are lowered to GEMMs:
//   conv2d     = im2col(x) [N*Ho*Wo, k*k*C] . w [k*k*C, F]
//   conv2d_t   = col2im(x [N*H*W, C] . w^T [C, k*k*F])       (conv2d's input gradient)
//   conv2d_dw  = im2col(x)^T [k*k*C, N*Ho*Wo] . dy [N*Ho*Wo, F]
// The GEMM is the tcgen05 kernel (bf16 mode; operands written straight into
// the bf16 K-major TMA layout by k_im2col / k_cvt_bf16) or the SIMT parity
// kernel (f64 / fp32 modes; bitwise equal to the oracle in f64).
//
// Batch-norm family: one column-statistics kernel (k_colstats, all rows x all
// channels in one pass, double accumulators, last-block finalisation) plus an
// elementwise apply kernel.
#pragma once
#include <cuda_bf16.h>

#include "kernels.cuh"

namespace coex {

constexpr double kBnEps = 1e-5;

// ------------------------------------------------------------------ im2col
struct Im2colParams {
  DevState* ds;
  In x;                      // [N, H, W, C]
  long long N, H, W, C, Ho, Wo;
  int k, s, p;
  void* dst;
  long long ld;              // row pitch of dst (elements)
  int trans;                 // 0: dst[m][kk] (m = output pixel, kk = (ky, kx, c)); 1: dst[kk][m]
};

template <typename Tin>
__device__ __forceinline__ Tin im2col_at(const Tin* x, const Im2colParams& p, long long m, long long kk) {
  const long long Kc = (long long)p.k * p.k * p.C;
  if (kk >= Kc) return Tin(0);
  const long long c = kk % p.C;
  const long long kx = (kk / p.C) % p.k;
  const long long ky = kk / ((long long)p.C * p.k);
  const long long ox = m % p.Wo;
  const long long oy = (m / p.Wo) % p.Ho;
  const long long n = m / (p.Wo * p.Ho);
  const long long iy = oy * p.s - p.p + ky, ix = ox * p.s - p.p + kx;
  if (iy < 0 || iy >= p.H || ix < 0 || ix >= p.W) return Tin(0);
  return x[((n * p.H + iy) * p.W + ix) * p.C + c];
}

template <typename Tout> __device__ __forceinline__ Tout cvt_to(double v) { return (Tout)v; }
template <> __device__ __forceinline__ __nv_bfloat16 cvt_to<__nv_bfloat16>(double v) {
  return __float2bfloat16_rn((float)v);
}

// Row-major destination: grid-stride over (m, kk), kk fastest (coalesced stores; the reads
// of one (ky, kx) run are contiguous channels).  bf16 destinations store 8 per thread.
template <typename Tin, typename Tout>
__global__ void __launch_bounds__(256) k_im2col(Im2colParams p) {
  COEX_PDL_ENTER();
  stamp(p.ds, SK_IM2COL);
  const Tin* x = res<Tin>(p.x);
  const long long M = p.N * p.Ho * p.Wo;
  const long long stride = (long long)gridDim.x * blockDim.x;
  if (!p.trans) {
    constexpr int V = sizeof(Tout) == 2 ? 8 : 1;
    const long long per_row = p.ld / V;
    const long long total = M * per_row;
    for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < total; i += stride) {
      const long long m = i / per_row, kk0 = (i % per_row) * V;
      Tout* d = (Tout*)p.dst + m * p.ld + kk0;
      if constexpr (V == 8) {
        __align__(16) Tout v[8];
#pragma unroll
        for (int j = 0; j < 8; ++j) v[j] = cvt_to<Tout>((double)im2col_at(x, p, m, kk0 + j));
        *(uint4*)d = *(const uint4*)v;
      } else {
        d[0] = cvt_to<Tout>((double)im2col_at(x, p, m, kk0));
      }
    }
    return;
  }
  // transposed destination dst[kk][m]: 32 x 32 tiles through shared memory
  __shared__ float tile[32][33];
  const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;
  const long long Kc = (long long)p.k * p.k * p.C;
  const long long tm = (p.ld + 31) / 32, tk = (Kc + 31) / 32;
  for (long long t = blockIdx.x; t < tm * tk; t += gridDim.x) {
    const long long m0 = (t % tm) * 32, k0 = (t / tm) * 32;
    for (int j = ty; j < 32; j += 8) {
      const long long m = m0 + j, kk = k0 + tx;
      tile[j][tx] = (m < M && kk < Kc) ? (float)im2col_at(x, p, m, kk) : 0.f;
    }
    __syncthreads();
    for (int j = ty; j < 32; j += 8) {
      const long long kk = k0 + j, m = m0 + tx;
      if (kk < Kc && m < p.ld) ((Tout*)p.dst)[kk * p.ld + m] = cvt_to<Tout>((double)tile[tx][j]);
    }
    __syncthreads();
  }
}

// Vectorised bf16 im2col (C % 8 == 0): one thread = 8 consecutive channels of one
// (pixel, ky, kx) = two float4 loads, one 16-byte store.  Each block owns a contiguous range
// of output pixels; a thread keeps its (ky, kx, channel-group) fixed and walks pixels with
// incremental (n, oy, ox) arithmetic -- no divisions in the loop.
__global__ void __launch_bounds__(256) k_im2col_bf16v(Im2colParams p) {
  COEX_PDL_ENTER();
  stamp(p.ds, SK_IM2COL);
  const float* x = res<float>(p.x);
  const int C8 = (int)(p.C / 8), k = p.k, H = (int)p.H, W = (int)p.W, Ho = (int)p.Ho, Wo = (int)p.Wo;
  const int Q = k * k * C8;                         // 16-byte units per row (ld == Kc)
  const long long M = p.N * p.Ho * p.Wo;
  const int t = threadIdx.x;
  const int rpi = Q >= 256 ? 1 : 256 / Q;           // rows per block iteration
  const int qpt = (Q + 255) / 256;                  // units per thread and row
  const int lane_q = Q >= 256 ? t : t % Q, lane_r = Q >= 256 ? 0 : t / Q;
  if (lane_r >= rpi) return;
  const long long r_begin = M * blockIdx.x / gridDim.x, r_end = M * (blockIdx.x + 1) / gridDim.x;
  for (int qi = 0; qi < qpt; ++qi) {
    const int q = lane_q + qi * 256;
    if (q >= Q) break;
    const int ky = q / (k * C8), r2 = q - ky * k * C8, kx = r2 / C8, cg = r2 - kx * C8;
    long long m = r_begin + lane_r;
    if (m >= r_end) continue;
    int ox = (int)(m % Wo);
    long long tq = m / Wo;
    int oy = (int)(tq % Ho);
    long long n = tq / Ho;
    for (; m < r_end; m += rpi) {
      const int iy = oy * p.s - p.p + ky, ix = ox * p.s - p.p + kx;
      uint4 out = make_uint4(0u, 0u, 0u, 0u);
      if (iy >= 0 && iy < H && ix >= 0 && ix < W) {
        const float4* src = (const float4*)(x + ((n * H + iy) * W + ix) * p.C + cg * 8);
        const float4 a = __ldg(src), b = __ldg(src + 1);
        __nv_bfloat162 v0 = __floats2bfloat162_rn(a.x, a.y), v1 = __floats2bfloat162_rn(a.z, a.w);
        __nv_bfloat162 v2 = __floats2bfloat162_rn(b.x, b.y), v3 = __floats2bfloat162_rn(b.z, b.w);
        out.x = *(uint32_t*)&v0; out.y = *(uint32_t*)&v1; out.z = *(uint32_t*)&v2; out.w = *(uint32_t*)&v3;
      }
      *(uint4*)((__nv_bfloat16*)p.dst + m * p.ld + (long long)q * 8) = out;
      ox += rpi;
      while (ox >= Wo) {
        ox -= Wo;
        if (++oy == Ho) { oy = 0; ++n; }
      }
    }
  }
}

// Transposed bf16 im2col dst[kk][m] (weight-gradient operand, K = output pixels), C % 4 == 0:
// 64 m x 32 kk tiles; each thread loads float4 runs of channels (8 threads per pixel row)
// and the tile is written back along pixels as bf16 pairs.
__global__ void __launch_bounds__(256) k_im2col_bf16t(Im2colParams p) {
  COEX_PDL_ENTER();
  stamp(p.ds, SK_IM2COL);
  const float* x = res<float>(p.x);
  __shared__ float tile[64][33];
  const int t = threadIdx.x;
  const int C = (int)p.C, k = p.k, H = (int)p.H, W = (int)p.W, Ho = (int)p.Ho, Wo = (int)p.Wo;
  const long long Kc = (long long)k * k * C;
  const unsigned M = (unsigned)(p.N * p.Ho * p.Wo);
  const long long tm = (p.ld + 63) / 64, tk = (Kc + 31) / 32;
  const int kq = t & 7, rl = t >> 3;                 // 8 float4 groups x 32 rows per pass
  const int tx = t & 31, ty = t >> 5;
  for (long long tt = blockIdx.x; tt < tm * tk; tt += gridDim.x) {
    const long long m0 = (tt % tm) * 64, k0 = (tt / tm) * 32;
    const long long kk = k0 + 4 * kq;
    const int c = (int)(kk % C), kx = (int)((kk / C) % k), ky = (int)(kk / ((long long)C * k));
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int j = rl + 32 * h;
      const unsigned m = (unsigned)(m0 + j);
      float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
      if (m < M && kk < Kc) {
        const int ox = (int)(m % (unsigned)Wo);
        const unsigned r = m / (unsigned)Wo;
        const int oy = (int)(r % (unsigned)Ho);
        const long long n = r / (unsigned)Ho;
        const int iy = oy * p.s - p.p + ky, ix = ox * p.s - p.p + kx;
        if (iy >= 0 && iy < H && ix >= 0 && ix < W) v = *(const float4*)(x + ((n * H + iy) * W + ix) * C + c);
      }
      tile[j][4 * kq] = v.x; tile[j][4 * kq + 1] = v.y; tile[j][4 * kq + 2] = v.z; tile[j][4 * kq + 3] = v.w;
    }
    __syncthreads();
    for (int j = ty; j < 32; j += 8) {
      const long long kr = k0 + j, m = m0 + 2 * tx;
      if (kr < Kc && m < p.ld) {
        __nv_bfloat162 v = __floats2bfloat162_rn(tile[2 * tx][j], tile[2 * tx + 1][j]);
        *(__nv_bfloat162*)((__nv_bfloat16*)p.dst + kr * p.ld + m) = v;
      }
    }
    __syncthreads();
  }
}

// Scalar bf16 im2col for C % 8 != 0 (e.g. the 3-channel image layer): one thread = one
// 8-element unit of a row, 32-bit index arithmetic.
__global__ void __launch_bounds__(256) k_im2col_bf16s(Im2colParams p) {
  COEX_PDL_ENTER();
  stamp(p.ds, SK_IM2COL);
  const float* x = res<float>(p.x);
  const int C = (int)p.C, k = p.k, H = (int)p.H, W = (int)p.W, Ho = (int)p.Ho, Wo = (int)p.Wo;
  const int Kc = k * k * C;
  const int Q = (int)(p.ld / 8);
  const long long total = p.N * p.Ho * p.Wo * Q;
  const long long stride = (long long)gridDim.x * blockDim.x;
  for (long long u = (long long)blockIdx.x * blockDim.x + threadIdx.x; u < total; u += stride) {
    const unsigned m = (unsigned)(u / Q);
    const int q = (int)(u - (long long)m * Q);
    const int ox = (int)(m % (unsigned)Wo);
    const unsigned r = m / (unsigned)Wo;
    const int oy = (int)(r % (unsigned)Ho);
    const long long n = r / (unsigned)Ho;
    __align__(16) __nv_bfloat16 v[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      const int kk = q * 8 + j;
      float val = 0.f;
      if (kk < Kc) {
        const int c = kk % C, kx = (kk / C) % k, ky = kk / (C * k);
        const int iy = oy * p.s - p.p + ky, ix = ox * p.s - p.p + kx;
        if (iy >= 0 && iy < H && ix >= 0 && ix < W) val = x[((n * H + iy) * W + ix) * C + c];
      }
      v[j] = __float2bfloat16_rn(val);
    }
    *(uint4*)((__nv_bfloat16*)p.dst + (long long)m * p.ld + (long long)q * 8) = *(const uint4*)v;
  }
}

// Few-channel bf16 im2col (C and k compile-time: the image layers, C = 3): one thread per
// output row builds the whole k*k*C row in registers (no per-element index division) and
// stores it as 16-byte units; the row pitch's tail is zeroed.
template <int C, int K>
__global__ void __launch_bounds__(256) k_im2col_small(Im2colParams p) {
  COEX_PDL_ENTER();
  stamp(p.ds, SK_IM2COL);
  const float* x = res<float>(p.x);
  constexpr int KC = K * K * C, KP = (KC + 7) / 8 * 8;
  const int H = (int)p.H, W = (int)p.W, Ho = (int)p.Ho, Wo = (int)p.Wo;
  const long long M = p.N * p.Ho * p.Wo;
  for (long long m = (long long)blockIdx.x * blockDim.x + threadIdx.x; m < M; m += (long long)gridDim.x * blockDim.x) {
    const int ox = (int)(m % Wo);
    const long long r = m / Wo;
    const int oy = (int)(r % Ho);
    const long long n = r / Ho;
    __align__(16) __nv_bfloat16 v[KP];
#pragma unroll
    for (int ky = 0; ky < K; ++ky) {
      const int iy = oy * p.s - p.p + ky;
#pragma unroll
      for (int kx = 0; kx < K; ++kx) {
        const int ix = ox * p.s - p.p + kx;
        const bool ok = iy >= 0 && iy < H && ix >= 0 && ix < W;
        const float* src = x + ((n * H + (ok ? iy : 0)) * W + (ok ? ix : 0)) * C;
#pragma unroll
        for (int c = 0; c < C; ++c) v[(ky * K + kx) * C + c] = __float2bfloat16_rn(ok ? __ldg(src + c) : 0.f);
      }
    }
#pragma unroll
    for (int j = KC; j < KP; ++j) v[j] = __float2bfloat16_rn(0.f);
    __nv_bfloat16* d = (__nv_bfloat16*)p.dst + m * p.ld;
#pragma unroll
    for (int q = 0; q < KP / 8; ++q) *(uint4*)(d + q * 8) = *(const uint4*)(v + q * 8);
    for (long long j = KP; j < p.ld; j += 8) *(uint4*)(d + j) = make_uint4(0, 0, 0, 0);
  }
}

// f64 parity path for the transposed operand is not needed: the SIMT GEMM reads the
// row-major im2col buffer with trans_a (element-exact), so only float tiles go through smem.

// ------------------------------------------------------------------ col2im
// out[n, oy, ox, f] = sum over (ky, kx) ascending of cols[(n, iy, ix), (ky, kx, f)] with
// oy = iy*s - p + ky, from +0.0 (oracle/kernels.py col2im).
struct Col2imParams {
  DevState* ds;
  const void* cols;          // [N*H*W][k*k*F] in the accumulation type
  long long N, H, W, F, Ho, Wo;
  int k, s, p;
  In a, b;                   // node operands (ping-pong output choice only)
  Out out;
};

template <typename Tc, typename T>
__global__ void __launch_bounds__(256) k_col2im(Col2imParams p) {
  COEX_PDL_ENTER();
  stamp(p.ds, SK_COL2IM);
  T* o = pick_out<T>(p.out, res<T>(p.a), res<T>(p.b));
  publish_early(p.out, o);
  count_op(p.ds);
  const Tc* cols = (const Tc*)p.cols;
  const long long total = p.N * p.Ho * p.Wo * p.F;
  const long long kkF = (long long)p.k * p.k * p.F;
  const long long stride = (long long)gridDim.x * blockDim.x;
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < total; i += stride) {
    const long long f = i % p.F;
    const long long ox = (i / p.F) % p.Wo;
    const long long oy = (i / (p.F * p.Wo)) % p.Ho;
    const long long n = i / (p.F * p.Wo * p.Ho);
    double acc = 0.0;
    for (int ky = 0; ky < p.k; ++ky) {
      const long long ty = oy + p.p - ky;
      if (ty < 0 || ty % p.s) continue;
      const long long iy = ty / p.s;
      if (iy >= p.H) continue;
      for (int kx = 0; kx < p.k; ++kx) {
        const long long tx = ox + p.p - kx;
        if (tx < 0 || tx % p.s) continue;
        const long long ix = tx / p.s;
        if (ix >= p.W) continue;
        const double v = (double)cols[((n * p.H + iy) * p.W + ix) * kkF + ((long long)ky * p.k + kx) * p.F + f];
        if constexpr (sizeof(T) == 8) acc = __dadd_rn(acc, v);
        else acc = (double)__fadd_rn((float)acc, (float)v);
      }
    }
    o[i] = (T)acc;
  }
  publish_late(p.out, o);
}

// Vectorised col2im (F % V == 0, V = 4 or 1): one thread = V channels of one output pixel;
// only the (ky, kx) taps congruent with the output position are visited, ascending.  Blocks
// own contiguous pixel ranges; threads keep their channel group and walk pixels
// incrementally (no divisions in the loop).
// Few-channel col2im (F compile-time, the image-producing conv2d_t): one thread per output
// pixel accumulates its F channels over the taps in ascending (ky, kx) order from +0 -- the
// same per-element order as k_col2im_v -- reading each tap's F floats contiguously.
template <int F>
__global__ void __launch_bounds__(256) k_col2im_px(Col2imParams p) {
  COEX_PDL_ENTER();
  stamp(p.ds, SK_COL2IM);
  float* o = pick_out<float>(p.out, res<float>(p.a), res<float>(p.b));
  publish_early(p.out, o);
  count_op(p.ds);
  const float* cols = (const float*)p.cols;
  const int k = p.k, s = p.s, pd = p.p, H = (int)p.H, W = (int)p.W, Ho = (int)p.Ho, Wo = (int)p.Wo;
  const long long kkF = (long long)k * k * F;
  const long long P = p.N * p.Ho * p.Wo;
  for (long long pix = (long long)blockIdx.x * blockDim.x + threadIdx.x; pix < P;
       pix += (long long)gridDim.x * blockDim.x) {
    const int ox = (int)(pix % Wo);
    const long long tq = pix / Wo;
    const int oy = (int)(tq % Ho);
    const long long n = tq / Ho;
    float acc[F];
#pragma unroll
    for (int f = 0; f < F; ++f) acc[f] = 0.f;
    const int ty0 = oy + pd, tx0 = ox + pd;
    for (int ky = ty0 % s; ky < k; ky += s) {
      const int iy = (ty0 - ky) / s;
      if (ty0 - ky < 0 || iy >= H) continue;
      for (int kx = tx0 % s; kx < k; kx += s) {
        const int ix = (tx0 - kx) / s;
        if (tx0 - kx < 0 || ix >= W) continue;
        const float* src = cols + ((n * H + iy) * W + ix) * kkF + ((long long)ky * k + kx) * F;
#pragma unroll
        for (int f = 0; f < F; ++f) acc[f] = __fadd_rn(acc[f], __ldg(src + f));
      }
    }
#pragma unroll
    for (int f = 0; f < F; ++f) o[pix * F + f] = acc[f];
  }
  publish_late(p.out, o);
}

template <int V>
__global__ void __launch_bounds__(256) k_col2im_v(Col2imParams p) {
  COEX_PDL_ENTER();
  stamp(p.ds, SK_COL2IM);
  float* o = pick_out<float>(p.out, res<float>(p.a), res<float>(p.b));
  publish_early(p.out, o);
  count_op(p.ds);
  const float* cols = (const float*)p.cols;
  const int F4 = (int)(p.F / V), k = p.k, s = p.s, pd = p.p, H = (int)p.H, W = (int)p.W;
  const int Ho = (int)p.Ho, Wo = (int)p.Wo;
  const long long kkF = (long long)k * k * p.F;
  const long long P = p.N * p.Ho * p.Wo;
  const int t = threadIdx.x;
  const int rpi = F4 >= 256 ? 1 : 256 / F4;
  const int fpt = (F4 + 255) / 256;
  const int lane_f = F4 >= 256 ? t : t % F4, lane_r = F4 >= 256 ? 0 : t / F4;
  if (lane_r < rpi) {
    const long long r_begin = P * blockIdx.x / gridDim.x, r_end = P * (blockIdx.x + 1) / gridDim.x;
    for (int fi = 0; fi < fpt; ++fi) {
      const int f4 = lane_f + fi * 256;
      if (f4 >= F4) break;
      long long pix = r_begin + lane_r;
      if (pix >= r_end) continue;
      int ox = (int)(pix % Wo);
      long long tq = pix / Wo;
      int oy = (int)(tq % Ho);
      long long n = tq / Ho;
      for (; pix < r_end; pix += rpi) {
        float acc[V];
#pragma unroll
        for (int v = 0; v < V; ++v) acc[v] = 0.f;
        const int ty0 = oy + pd, tx0 = ox + pd;
        for (int ky = ty0 % s; ky < k; ky += s) {
          const int iy = (ty0 - ky) / s;
          if (ty0 - ky < 0 || iy >= H) continue;
          for (int kx = tx0 % s; kx < k; kx += s) {
            const int ix = (tx0 - kx) / s;
            if (tx0 - kx < 0 || ix >= W) continue;
            const float* src = cols + ((n * H + iy) * W + ix) * kkF + ((long long)ky * k + kx) * p.F + f4 * V;
            if constexpr (V == 4) {
              const float4 v = __ldg((const float4*)src);
              acc[0] = __fadd_rn(acc[0], v.x); acc[1] = __fadd_rn(acc[1], v.y);
              acc[2] = __fadd_rn(acc[2], v.z); acc[3] = __fadd_rn(acc[3], v.w);
            } else {
              acc[0] = __fadd_rn(acc[0], __ldg(src));
            }
          }
        }
        if constexpr (V == 4) *(float4*)(o + pix * p.F + f4 * 4) = make_float4(acc[0], acc[1], acc[2], acc[3]);
        else o[pix * p.F + f4] = acc[0];
        ox += rpi;
        while (ox >= Wo) {
          ox -= Wo;
          if (++oy == Ho) { oy = 0; ++n; }
        }
      }
    }
  }
  publish_late(p.out, o);
}

// fp32 NHWC -> bf16 NHWC with a zero border of P pixels ([N][H+2P][W+2P][C]; the border is
// never written -- the workspace is zeroed once), the source of the implicit-GEMM gathers:
// TMA boxes then start at non-negative coordinates.  C % 8 == 0; 8 channels per thread.
struct PadCvtParams {
  DevState* ds;
  In x;
  __nv_bfloat16* dst;
  long long N;
  int H, W, C, P;
};
__global__ void __launch_bounds__(256) k_cvt_pad_bf16(PadCvtParams p) {
  COEX_PDL_ENTER();
  stamp(p.ds, SK_CVT);
  const float* x = res<float>(p.x);
  const int C8 = p.C / 8, Wp = p.W + 2 * p.P, Hp = p.H + 2 * p.P;
  // the zero border is rewritten every pass: the destination is shared scratch
  if (p.P > 0) {
    const int P2 = 2 * p.P;
    const long long tb = p.N * P2 * Wp * C8;             // top / bottom border rows
    const long long sd = p.N * p.H * P2 * C8;            // left / right border columns
    for (long long u = (long long)blockIdx.x * blockDim.x + threadIdx.x; u < tb + sd;
         u += (long long)gridDim.x * blockDim.x) {
      long long pix;
      if (u < tb) {
        const long long q = u / C8, r = q / Wp;
        const int i = (int)(r % P2);
        pix = ((r / P2) * Hp + (i < p.P ? i : p.H + i)) * Wp + q % Wp;
      } else {
        const long long q = (u - tb) / C8, r = q / P2;
        const int j = (int)(q % P2);
        pix = ((r / p.H) * Hp + r % p.H + p.P) * Wp + (j < p.P ? j : p.W + j);
      }
      *(uint4*)(p.dst + pix * p.C + (u % C8) * 8) = make_uint4(0, 0, 0, 0);
    }
  }
  const long long total = p.N * p.H * p.W * C8;
  for (long long u = (long long)blockIdx.x * blockDim.x + threadIdx.x; u < total;
       u += (long long)gridDim.x * blockDim.x) {
    const long long pix = u / C8;
    const int cg = (int)(u - pix * C8);
    const int w = (int)(pix % p.W);
    const long long t = pix / p.W;
    const int h = (int)(t % p.H);
    const long long n = t / p.H;
    const float4* src = (const float4*)(x + pix * p.C + cg * 8);
    const float4 a = __ldg(src), b = __ldg(src + 1);
    __nv_bfloat162 v0 = __floats2bfloat162_rn(a.x, a.y), v1 = __floats2bfloat162_rn(a.z, a.w);
    __nv_bfloat162 v2 = __floats2bfloat162_rn(b.x, b.y), v3 = __floats2bfloat162_rn(b.z, b.w);
    uint4 o;
    o.x = *(uint32_t*)&v0; o.y = *(uint32_t*)&v1; o.z = *(uint32_t*)&v2; o.w = *(uint32_t*)&v3;
    *(uint4*)(p.dst + ((n * Hp + h + p.P) * Wp + w + p.P) * p.C + cg * 8) = o;
  }
}

// Sub-pixel conv2d_t weights: for output phase (py, px) the taps ky = ky0 + (T-1-jy)*so,
// ky0 = (py + pad) mod so (likewise x), stacked as bf16 [phase][(jy, jx, c)][pitch(F)] -- the
// MN-major B operand of the phase GEMMs.  w is conv2d_t's weight [k*k*F][C].
struct WPhaseParams {
  DevState* ds;
  In w;
  __nv_bfloat16* dst;
  long long ld;              // row pitch of dst (>= F, multiple of 8)
  int k, so, pad, T, C, F;
};
__global__ void __launch_bounds__(256) k_convt_wphase(WPhaseParams p) {
  COEX_PDL_ENTER();
  stamp(p.ds, SK_CVT);
  const float* w = res<float>(p.w);
  const long long krows = (long long)p.T * p.T * p.C;
  const long long rows = (long long)p.so * p.so * krows;
  const long long total = rows * p.ld;
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < total;
       i += (long long)gridDim.x * blockDim.x) {
    const long long r = i / p.ld;
    const int f = (int)(i - r * p.ld);
    float v = 0.f;
    if (f < p.F) {
      const int ph = (int)(r / krows);
      const int rem = (int)(r - (long long)ph * krows);
      const int tap = rem / p.C, c = rem - tap * p.C;
      const int jy = tap / p.T, jx = tap - jy * p.T;
      const int py = ph / p.so, px = ph - py * p.so;
      const int ky = (py + p.pad) % p.so + (p.T - 1 - jy) * p.so;
      const int kx = (px + p.pad) % p.so + (p.T - 1 - jx) * p.so;
      v = w[(((long long)ky * p.k + kx) * p.F + f) * p.C + c];
    }
    p.dst[i] = __float2bfloat16_rn(v);
  }
}

// ------------------------------------------------------------------ column statistics
// Per-channel (last axis) sums over all leading rows, in double, with a per-channel shift
// K_c = x[0, c] (numerically a centred one-pass): S1 = sum(x-K), S2 = sum((x-K)^2),
// D1 = sum(dy), D2 = sum(dy*(x-K)).  Blocks write partials; the last block to finish
// combines them in block order (deterministic) and finalises.
enum ColMode { COL_SUM_ROWS = 0, COL_BN = 1, COL_BN_DX = 2, COL_BN_DGAMMA = 3 };
constexpr int kColMaxSlots = 8;    // channels per thread (C <= 8 * 256)
constexpr int kColReplicas = 8;    // atomic accumulators (spreads same-address contention)

struct ColStatsParams {
  DevState* ds;
  In x, dy;
  long long R, C;
  int mode;
  double* part;              // [gridDim.x][C][4] partials, or [C][4] accumulator when atomic
  int atomic;
  double* stats;             // [C][4]: mean, rstd, mean(dy), mean(dy*xhat)   (COL_BN, COL_BN_DX)
  unsigned int* counter;     // zero-initialised; reset by the last block
  In a, b;                   // node operands (ping-pong output choice only)
  Out out;                   // [C] result (COL_SUM_ROWS, COL_BN_DGAMMA)
  int extra;                 // COL_BN_DX fused backward: also write dgamma / dbeta [C]
  Out out_g, out_b;
  long long chunk_rows;      // BULK: rows per streamed chunk (a multiple of the rows per pass)
  int raw;                   // synchronised batch norm (data parallel): no shift; the last block
                             // writes the raw [C][4] sums sum(x), sum(x^2), sum(dy), sum(dy*x) to
                             // `stats` for the cross-rank all-reduce and k_bn_finalize
};

// 1-D bulk copy global -> shared, completion counted on an mbarrier (BULK column statistics)
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   smem_u32(dst)),
               "l"((uint64_t)src), "r"(bytes), "r"(smem_u32(bar))
               : "memory");
}
constexpr int kColStages = 4;      // BULK: chunks in flight per block

// V = channels per thread (4: float4 loads when C % 4 == 0 and T = float; else 1); rows
// unrolled by 4 so each thread keeps several independent loads in flight.
//
// BULK (float, V = 4, S = 1): the block's rows are one contiguous range, streamed through a
// kColStages-deep shared-memory ring by 1-D bulk copies (thread 0 issues, mbarriers count the
// bytes) -- the bytes in flight no longer depend on registers per thread, so large tensors
// run at HBM rate with two blocks per SM.
template <typename T, int V, int S, bool DY, bool BULK = false>
__global__ void __launch_bounds__(256) k_colstats(ColStatsParams p) {
  COEX_PDL_ENTER();
  stamp(p.ds, SK_COLSTATS);
  const T* x = res<T>(p.x);
  constexpr bool with_dy = DY;
  const T* dy = with_dy ? res<T>(p.dy) : nullptr;
  const bool final_out = p.mode == COL_SUM_ROWS || p.mode == COL_BN_DGAMMA;
  T* o = nullptr;
  if (final_out) {
    o = pick_out<T>(p.out, res<T>(p.a), p.b.cell || p.b.direct ? res<T>(p.b) : nullptr);
    publish_early(p.out, o);
  }
  count_op(p.ds);
  const long long C = p.C, R = p.R;
  const long long CV = C / V;                      // vector lanes per row
  const int L = (int)(CV < 256 ? CV : 256);
  const int rpi = 256 / L;
  const int t = threadIdx.x, cc = t % L, rr = t / L;
  const int slots = (int)((CV + L - 1) / L);
  const long long r_begin = R * blockIdx.x / gridDim.x, r_end = R * (blockIdx.x + 1) / gridDim.x;
  double a1[S][V], a2[S][V], a3[S][V], a4[S][V], sh[S][V];
#pragma unroll
  for (int j = 0; j < S; ++j)
#pragma unroll
    for (int v = 0; v < V; ++v) {
      a1[j][v] = a2[j][v] = a3[j][v] = a4[j][v] = 0.0;
      const long long c = (cc + (long long)j * L) * V + v;
      sh[j][v] = (p.mode != COL_SUM_ROWS && !p.raw && j < slots && c < C) ? (double)x[c] : 0.0;
    }
  if constexpr (BULK) {
    extern __shared__ __align__(128) unsigned char col_dsm[];
    __shared__ uint64_t full[kColStages];
    const long long cr = p.chunk_rows, cf = cr * C;
    float* xs = (float*)col_dsm;
    float* gs = xs + kColStages * cf;
    const long long nch = (r_end - r_begin + cr - 1) / cr;
    if (t == 0) {
      for (int q = 0; q < kColStages; ++q) mbar_init(&full[q], 1);
      asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    auto issue = [&](long long i) {
      const int q = (int)(i % kColStages);
      const long long r0 = r_begin + i * cr;
      const long long nr = r_end - r0 < cr ? r_end - r0 : cr;
      const uint32_t bytes = (uint32_t)(nr * C * 4);
      mbar_expect_tx(&full[q], with_dy ? 2 * bytes : bytes);
      bulk_g2s(xs + q * cf, x + r0 * C, bytes, &full[q]);
      if (with_dy) bulk_g2s(gs + q * cf, dy + r0 * C, bytes, &full[q]);
    };
    if (t == 0)
      for (long long i = 0; i < nch && i < kColStages; ++i) issue(i);
    const long long c0 = (long long)cc * V;
    for (long long i = 0; i < nch; ++i) {
      const int q = (int)(i % kColStages);
      mbar_wait(&full[q], (uint32_t)((i / kColStages) & 1));
      const long long nr = r_end - (r_begin + i * cr) < cr ? r_end - (r_begin + i * cr) : cr;
      if (rr < rpi && c0 < C) {
        for (long long r = rr; r < nr; r += rpi) {
          const float4 f = *(const float4*)(xs + q * cf + r * C + c0);
          const float xv[4] = {f.x, f.y, f.z, f.w};
          float gv[4] = {0.f, 0.f, 0.f, 0.f};
          if (with_dy) {
            const float4 g = *(const float4*)(gs + q * cf + r * C + c0);
            gv[0] = g.x; gv[1] = g.y; gv[2] = g.z; gv[3] = g.w;
          }
#pragma unroll
          for (int v = 0; v < V; ++v) {
            const double d = (double)xv[v] - sh[0][v];
            a1[0][v] += d;
            a2[0][v] += d * d;
            if (with_dy) {
              a3[0][v] += (double)gv[v];
              a4[0][v] += (double)gv[v] * d;
            }
          }
        }
      }
      __syncthreads();                      // stage q consumed by every thread
      if (t == 0 && i + kColStages < nch) issue(i + kColStages);
    }
  } else if (rr < rpi) {
#pragma unroll
    for (int j = 0; j < S; ++j) {
      if (j >= slots) break;
      const long long c0 = (cc + (long long)j * L) * V;
      if (c0 >= C) break;
      long long r = r_begin + rr;
      for (; r + 3 * rpi < r_end; r += 4 * rpi) {
        T xv[4][V], gv[4][V];
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          const long long off = (r + (long long)q * rpi) * C + c0;
          if constexpr (V == 4) {
            const float4 f = *(const float4*)(x + off);
            xv[q][0] = f.x; xv[q][1] = f.y; xv[q][2] = f.z; xv[q][3] = f.w;
            if (with_dy) {
              const float4 g = *(const float4*)(dy + off);
              gv[q][0] = g.x; gv[q][1] = g.y; gv[q][2] = g.z; gv[q][3] = g.w;
            }
          } else {
            xv[q][0] = x[off];
            if (with_dy) gv[q][0] = dy[off];
          }
        }
#pragma unroll
        for (int q = 0; q < 4; ++q)
#pragma unroll
          for (int v = 0; v < V; ++v) {
            const double d = (double)xv[q][v] - sh[j][v];
            a1[j][v] += d;
            a2[j][v] += d * d;
            if (with_dy) {
              const double g = (double)gv[q][v];
              a3[j][v] += g;
              a4[j][v] += g * d;
            }
          }
      }
      for (; r < r_end; r += rpi) {
#pragma unroll
        for (int v = 0; v < V; ++v) {
          const long long off = r * C + c0 + v;
          const double d = (double)x[off] - sh[j][v];
          a1[j][v] += d;
          a2[j][v] += d * d;
          if (with_dy) {
            const double g = (double)dy[off];
            a3[j][v] += g;
            a4[j][v] += g * d;
          }
        }
      }
    }
  }
  __shared__ double sm[256][4];
  for (int j = 0; j < slots && j < S; ++j) {
    for (int v = 0; v < V; ++v) {
      sm[t][0] = a1[j][v]; sm[t][1] = a2[j][v]; sm[t][2] = a3[j][v]; sm[t][3] = a4[j][v];
      __syncthreads();
      const long long c = (t + (long long)j * L) * V + v;
      if (t < L && c < C) {
        double acc[4] = {0.0, 0.0, 0.0, 0.0};
        for (int q = 0; q < rpi; ++q)
          for (int u = 0; u < 4; ++u) acc[u] += sm[q * L + t][u];
        if (p.atomic) {        // tolerance modes: fp64 atomics into one of kColReplicas [C][4] accumulators
          double* dst = p.part + ((long long)(blockIdx.x % kColReplicas) * C + c) * 4;
          for (int u = 0; u < 4; ++u) atomicAdd(dst + u, acc[u]);
        } else {               // parity mode: per-block partials merged in block order
          double* dst = p.part + ((long long)blockIdx.x * C + c) * 4;
          for (int u = 0; u < 4; ++u) dst[u] = acc[u];
        }
      }
      __syncthreads();
    }
  }
  // last block: combine partials (block order) and finalise.  The CTA barrier orders every
  // thread's partial writes before thread 0's cumulative gpu-scope fence and arrival.
  __shared__ unsigned int last;
  __syncthreads();
  if (t == 0) {
    __threadfence();
    last = (atomicAdd(p.counter, 1u) == gridDim.x - 1) ? 1u : 0u;
    if (last) __threadfence();
  }
  __syncthreads();
  if (!last) return;
  for (long long c = t; c < C; c += blockDim.x) {
    // four interleaved accumulators (fixed combination order: deterministic), L2 loads
    // (the partials were written by other blocks; this SM never cached them)
    double acc[4][4] = {{0.0}};
    const double2* q = (const double2*)(p.part + c * 4);
    const long long stride2 = 2 * C;                // two double2 per channel per block
    const unsigned int nb = p.atomic ? (gridDim.x < (unsigned)kColReplicas ? gridDim.x : (unsigned)kColReplicas)
                                     : gridDim.x;
    unsigned int b = 0;
    for (; b + 4 <= nb; b += 4) {
#pragma unroll
      for (int w = 0; w < 4; ++w) {
        const double2 u = __ldcg(q + (long long)(b + w) * stride2), v = __ldcg(q + (long long)(b + w) * stride2 + 1);
        acc[w][0] += u.x; acc[w][1] += u.y; acc[w][2] += v.x; acc[w][3] += v.y;
      }
    }
    for (; b < nb; ++b) {
      const double2 u = __ldcg(q + (long long)b * stride2), v = __ldcg(q + (long long)b * stride2 + 1);
      acc[0][0] += u.x; acc[0][1] += u.y; acc[0][2] += v.x; acc[0][3] += v.y;
    }
    if (p.atomic) {                                 // leave the accumulators zeroed for the next launch
      for (unsigned int r = 0; r < nb; ++r) {
        double2* z = (double2*)(p.part + ((long long)r * C + c) * 4);
        z[0] = make_double2(0.0, 0.0);
        z[1] = make_double2(0.0, 0.0);
      }
    }
    const double s1 = (acc[0][0] + acc[1][0]) + (acc[2][0] + acc[3][0]);
    const double s2 = (acc[0][1] + acc[1][1]) + (acc[2][1] + acc[3][1]);
    const double d1 = (acc[0][2] + acc[1][2]) + (acc[2][2] + acc[3][2]);
    const double d2 = (acc[0][3] + acc[1][3]) + (acc[2][3] + acc[3][3]);
    if (p.mode == COL_SUM_ROWS) {
      o[c] = (T)s1;
      continue;
    }
    if (p.raw) {                                    // rank-local sums: all-reduced, then finalised
      double* st = p.stats + c * 4;
      st[0] = s1;
      st[1] = s2;
      st[2] = d1;
      st[3] = d2;
      continue;
    }
    const double m1 = s1 / (double)R;
    const double mean = (double)x[c] + m1;
    double var = s2 / (double)R - m1 * m1;
    if (var < 0.0) var = 0.0;
    const double rstd = 1.0 / sqrt(var + kBnEps);
    const double sdx = rstd * (d2 - m1 * d1);          // sum(dy * xhat)
    if (p.mode == COL_BN_DGAMMA) {
      o[c] = (T)sdx;
      continue;
    }
    if (p.extra) {                                  // fused backward: dgamma = sum(dy*xhat), dbeta = sum(dy)
      T* og = pick_out<T>(p.out_g, x, dy);
      T* ob = pick_out<T>(p.out_b, x, dy);
      og[c] = (T)sdx;
      ob[c] = (T)d1;
    }
    double* st = p.stats + c * 4;
    st[0] = mean;
    st[1] = rstd;
    st[2] = d1 / (double)R;
    st[3] = sdx / (double)R;
  }
  if (t == 0) *p.counter = 0u;
  if (p.extra) {
    __syncthreads();
    if (t == 0) {                                   // the finishing block publishes both
      T* og = pick_out<T>(p.out_g, x, dy);
      T* ob = pick_out<T>(p.out_b, x, dy);
      for (int i = 0; i < p.out_g.npub; ++i) *p.out_g.pub[i] = og;
      for (int i = 0; i < p.out_b.npub; ++i) *p.out_b.pub[i] = ob;
    }
  }
  if (final_out) {
    __syncthreads();
    if (t == 0 && p.out.late != nullptr)   // single finishing block publishes
      for (int i = 0; i < p.out.npub; ++i) *p.out.pub[i] = o;
  }
}

// Synchronised batch norm (data parallel): the all-reduced raw sums of every
// rank's rows -> mean, rstd, mean(dy), mean(dy*xhat) over the GLOBAL batch (R = global rows),
// the same finalisation as k_colstats with shift 0.  BN_DGAMMA writes sum(dy*xhat) (global,
// replicated).  One block.
struct BnFinalizeParams {
  DevState* ds;
  double* stats;             // [C][4] in: raw global sums; out: mean, rstd, mean(dy), mean(dy*xhat)
  long long C;
  double R;
  int mode;                  // COL_BN, COL_BN_DX, COL_BN_DGAMMA
  In a, b;                   // node operands (ping-pong output choice only)
  Out out;                   // COL_BN_DGAMMA: [C]
};

template <typename T>
__global__ void __launch_bounds__(256) k_bn_finalize(BnFinalizeParams p) {
  COEX_PDL_ENTER();
  stamp(p.ds, SK_COLSTATS);
  T* o = nullptr;
  if (p.mode == COL_BN_DGAMMA) {
    o = pick_out<T>(p.out, res<T>(p.a), p.b.cell || p.b.direct ? res<T>(p.b) : nullptr);
    publish_early(p.out, o);
  }
  for (long long c = threadIdx.x; c < p.C; c += blockDim.x) {
    double* st = p.stats + c * 4;
    const double s1 = st[0], s2 = st[1], d1 = st[2], d2 = st[3];
    const double mean = s1 / p.R;
    double var = s2 / p.R - mean * mean;
    if (var < 0.0) var = 0.0;
    const double rstd = 1.0 / sqrt(var + kBnEps);
    const double sdx = rstd * (d2 - mean * d1);      // sum(dy * xhat)
    if (p.mode == COL_BN_DGAMMA) {
      o[c] = (T)sdx;
      continue;
    }
    st[0] = mean;
    st[1] = rstd;
    st[2] = d1 / p.R;
    st[3] = sdx / p.R;
  }
  if (o) publish_late(p.out, o);
}

// ------------------------------------------------------------------ batch-norm apply
struct BnApplyParams {
  DevState* ds;
  In x, g, third;            // BATCHNORM: third = beta [C]; BATCHNORM_DX: third = dy (x's shape)
  const double* stats;       // [C][4]
  long long n, C;
  int dx;                    // 0: y = ((x-mean)*rstd)*g + b; 1: dx = (dy - m(dy) - xhat*m(dy*xhat)) * (g*rstd)
  Out out;
  int act;                   // >= 0: also write act(y) (EW_RELU / EW_LRELU) to out2
  Out out2;
};

template <typename T>
__global__ void __launch_bounds__(256) k_bn_apply(BnApplyParams p) {
  COEX_PDL_ENTER();
  stamp(p.ds, SK_BNAPPLY);
  const T* x = res<T>(p.x);
  const T* g = res<T>(p.g);
  const T* z = res<T>(p.third);
  T* o = pick_out<T>(p.out, x, g);
  T* o2 = p.act >= 0 ? pick_out<T>(p.out2, x, g) : nullptr;
  publish_early(p.out, o);
  if (o2) publish_early(p.out2, o2);
  count_op(p.ds);
  const long long stride = (long long)gridDim.x * blockDim.x;
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < p.n; i += stride) {
    const long long c = i % p.C;
    const double* st = p.stats + c * 4;
    const double xhat = ((double)x[i] - st[0]) * st[1];
    double r;
    if (!p.dx) r = xhat * (double)g[c] + (double)z[c];
    else r = (((double)z[i] - st[2]) - xhat * st[3]) * ((double)g[c] * st[1]);
    o[i] = (T)r;
    if (o2) o2[i] = ew_apply(p.act, (T)r, (T)0);
  }
  publish_late(p.out, o);
  if (o2) publish_late(p.out2, o2);
}

// Vectorised apply (float, C % 4 == 0): per-channel affine coefficients in shared memory,
// one float4 per thread.  BATCHNORM: y = x*A + B;  BATCHNORM_DX: dx = dy*A + x*B + D with
// A = g*rstd, B = -g*rstd^2*mean(dy*xhat), D = g*rstd*(rstd*mean*mean(dy*xhat) - mean(dy)).
__global__ void __launch_bounds__(256) k_bn_apply_v4(BnApplyParams p) {
  COEX_PDL_ENTER();
  stamp(p.ds, SK_BNAPPLY);
  extern __shared__ float coef[];                    // [3][C]
  const float* x = res<float>(p.x);
  const float* g = res<float>(p.g);
  const float* z = res<float>(p.third);
  float* o = pick_out<float>(p.out, x, g);
  float* o2 = p.act >= 0 ? pick_out<float>(p.out2, x, g) : nullptr;
  publish_early(p.out, o);
  if (o2) publish_early(p.out2, o2);
  count_op(p.ds);
  const int C = (int)p.C;
  for (int c = threadIdx.x; c < C; c += blockDim.x) {
    const double* st = p.stats + (long long)c * 4;
    const double gr = (double)g[c] * st[1];
    if (!p.dx) {
      coef[c] = (float)gr;
      coef[C + c] = (float)((double)z[c] - st[0] * gr);
    } else {
      coef[c] = (float)gr;
      coef[C + c] = (float)(-gr * st[1] * st[3]);
      coef[2 * C + c] = (float)(gr * (st[1] * st[0] * st[3] - st[2]));
    }
  }
  __syncthreads();
  const long long n4 = p.n / 4;
  const long long stride = (long long)gridDim.x * blockDim.x;
  const int C4 = C / 4;
  for (long long u = (long long)blockIdx.x * blockDim.x + threadIdx.x; u < n4; u += stride) {
    const int c = (int)(u % C4) * 4;
    const float4 xv = ((const float4*)x)[u];
    float4 r;
    if (!p.dx) {
      r.x = fmaf(xv.x, coef[c], coef[C + c]);
      r.y = fmaf(xv.y, coef[c + 1], coef[C + c + 1]);
      r.z = fmaf(xv.z, coef[c + 2], coef[C + c + 2]);
      r.w = fmaf(xv.w, coef[c + 3], coef[C + c + 3]);
    } else {
      const float4 gv = ((const float4*)z)[u];
      r.x = fmaf(gv.x, coef[c], fmaf(xv.x, coef[C + c], coef[2 * C + c]));
      r.y = fmaf(gv.y, coef[c + 1], fmaf(xv.y, coef[C + c + 1], coef[2 * C + c + 1]));
      r.z = fmaf(gv.z, coef[c + 2], fmaf(xv.z, coef[C + c + 2], coef[2 * C + c + 2]));
      r.w = fmaf(gv.w, coef[c + 3], fmaf(xv.w, coef[C + c + 3], coef[2 * C + c + 3]));
    }
    ((float4*)o)[u] = r;
    if (o2) {
      const int a = p.act;
      ((float4*)o2)[u] = make_float4(ew_apply(a, r.x, 0.f), ew_apply(a, r.y, 0.f), ew_apply(a, r.z, 0.f),
                                     ew_apply(a, r.w, 0.f));
    }
  }
  publish_late(p.out, o);
  if (o2) publish_late(p.out2, o2);
}

// ------------------------------------------------------------------ pooling (config C3)
// NHWC, channels innermost (coalesced).  MODE 0 maxpool, 2 avgpool: one thread per output
// element, taps in (ky, kx) order (max: strict '>' so the first maximum wins, -inf padding;
// avg: zero padding, sum / k^2).  MODE 1 maxpool_grad, 3 avgpool_grad: one thread per INPUT
// element gathering the covering windows in ascending (oy, ox) order (max: the window's
// argmax recomputed, or read from the per-window tap indices MODE 6 wrote; no atomics,
// deterministic).  MODE 4 global average pool (thread per
// (n, c), row-major sequential sum / (H*W)), MODE 5 its gradient -- oracle/kernels.py
// pool_kernel.
struct PoolParams {
  DevState* ds;
  In x, dy;
  Out out;
  long long N, H, W, C, Ho, Wo;
  int k, s, p;
  unsigned char* idx;        // maxpool_grad: per-window argmax tap (ky*k + kx), written by MODE 6
};

template <typename T, int MODE>
__global__ void __launch_bounds__(256) k_pool(PoolParams p) {
  COEX_PDL_ENTER();
  stamp(p.ds, SK_POOL);
  const T* x = res<T>(p.x);
  const T* dy = (MODE & 1) ? res<T>(p.dy) : nullptr;       // modes 1, 3, 5 take (x, dy)
  if (MODE == 6) {                       // maxpool_grad pass 1: argmax tap of every window
    const long long total = p.N * p.Ho * p.Wo * p.C;
    for (long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x; e < total;
         e += (long long)gridDim.x * blockDim.x) {
      const long long c = e % p.C, pix = e / p.C;
      const long long ox = pix % p.Wo, oy = (pix / p.Wo) % p.Ho, n = pix / (p.Wo * p.Ho);
      T m = (T)-INFINITY;
      int arg = -1, first = -1;
      for (int ky = 0; ky < p.k; ++ky) {
        const long long iy = oy * p.s - p.p + ky;
        if (iy < 0 || iy >= p.H) continue;
        for (int kx = 0; kx < p.k; ++kx) {
          const long long ix = ox * p.s - p.p + kx;
          if (ix < 0 || ix >= p.W) continue;
          const T v = x[((n * p.H + iy) * p.W + ix) * p.C + c];
          if (first < 0) first = ky * p.k + kx;
          if (v > m) { m = v; arg = ky * p.k + kx; }
        }
      }
      p.idx[e] = (unsigned char)(arg < 0 ? first : arg);
    }
    return;
  }
  T* o = pick_out<T>(p.out, x, dy);
  publish_early(p.out, o);
  count_op(p.ds);
  const long long C = p.C;
  const int k = p.k, s = p.s, pd = p.p;
  const long long stride = (long long)gridDim.x * blockDim.x;
  if (MODE == 4) {                       // global average pool: thread per (n, c)
    const long long hw = p.H * p.W;
    for (long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x; e < p.N * C; e += stride) {
      const T* xp = x + (e / C) * hw * C + e % C;
      T acc = (T)0;
      for (long long i = 0; i < hw; ++i) acc = acc + xp[i * C];
      o[e] = acc / (T)hw;
    }
  } else if (MODE == 5) {                // its gradient: dy[n, c] / (H*W) broadcast
    const long long hw = p.H * p.W, total = p.N * hw * C;
    for (long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x; e < total; e += stride)
      o[e] = dy[(e / (hw * C)) * C + e % C] / (T)hw;
  } else if (MODE == 0 || MODE == 2) {
    const long long total = p.N * p.Ho * p.Wo * C;
    for (long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x; e < total; e += stride) {
      const long long c = e % C, pix = e / C;
      const long long ox = pix % p.Wo, oy = (pix / p.Wo) % p.Ho, n = pix / (p.Wo * p.Ho);
      T acc = MODE == 0 ? (T)-INFINITY : (T)0;
      for (int ky = 0; ky < k; ++ky) {
        const long long iy = oy * s - pd + ky;
        if (iy < 0 || iy >= p.H) continue;
        for (int kx = 0; kx < k; ++kx) {
          const long long ix = ox * s - pd + kx;
          if (ix < 0 || ix >= p.W) continue;
          const T v = x[((n * p.H + iy) * p.W + ix) * C + c];
          if (MODE == 0) { if (v > acc) acc = v; }
          else acc = acc + v;
        }
      }
      o[e] = MODE == 0 ? acc : acc / (T)(k * k);
    }
  } else {
    const long long total = p.N * p.H * p.W * C;
    for (long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x; e < total; e += stride) {
      const long long c = e % C, pix = e / C;
      const long long ix = pix % p.W, iy = (pix / p.W) % p.H, n = pix / (p.W * p.H);
      // windows oy with oy*s - p <= iy <= oy*s - p + k - 1
      long long oy0 = iy + pd - k + 1;
      oy0 = oy0 <= 0 ? 0 : (oy0 + s - 1) / s;
      long long oy1 = (iy + pd) / s;
      if (oy1 > p.Ho - 1) oy1 = p.Ho - 1;
      long long ox0 = ix + pd - k + 1;
      ox0 = ox0 <= 0 ? 0 : (ox0 + s - 1) / s;
      long long ox1 = (ix + pd) / s;
      if (ox1 > p.Wo - 1) ox1 = p.Wo - 1;
      T acc = (T)0;
      for (long long oy = oy0; oy <= oy1; ++oy) {
        for (long long ox = ox0; ox <= ox1; ++ox) {
          const long long w = ((n * p.Ho + oy) * p.Wo + ox) * C + c;
          if (MODE == 3) { acc = acc + dy[w]; continue; }
          if (p.idx != nullptr) {          // argmax from pass 1
            if (p.idx[w] == (unsigned char)((iy - (oy * s - pd)) * k + (ix - (ox * s - pd)))) acc = acc + dy[w];
            continue;
          }
          const T g = dy[w];
          // argmax: strict '>' from -inf; no tap above -inf -> the first in-bounds tap
          T m = (T)-INFINITY;
          long long ay = -1, ax = -1, fy = -1, fx = -1;
          for (int ky = 0; ky < k; ++ky) {
            const long long yy = oy * s - pd + ky;
            if (yy < 0 || yy >= p.H) continue;
            for (int kx = 0; kx < k; ++kx) {
              const long long xx = ox * s - pd + kx;
              if (xx < 0 || xx >= p.W) continue;
              const T v = x[((n * p.H + yy) * p.W + xx) * C + c];
              if (fy < 0) { fy = yy; fx = xx; }
              if (v > m) { m = v; ay = yy; ax = xx; }
            }
          }
          if (ay < 0) { ay = fy; ax = fx; }
          if (ay == iy && ax == ix) acc = acc + g;
        }
      }
      o[e] = MODE == 3 ? acc / (T)(k * k) : acc;
    }
  }
  publish_late(p.out, o);
}

}  // namespace coex
