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
  stamp(p.ds, SK_FUSED);
  if (skip(p.ds)) return;
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
  stamp(p.ds, SK_FUSED);
  if (skip(p.ds)) return;
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

// ------------------------------------------------------------------ column statistics
// Per-channel (last axis) sums over all leading rows, in double, with a per-channel shift
// K_c = x[0, c] (numerically a centred one-pass): S1 = sum(x-K), S2 = sum((x-K)^2),
// D1 = sum(dy), D2 = sum(dy*(x-K)).  Blocks write partials; the last block to finish
// combines them in block order (deterministic) and finalises.
enum ColMode { COL_SUM_ROWS = 0, COL_BN = 1, COL_BN_DX = 2, COL_BN_DGAMMA = 3 };
constexpr int kColMaxSlots = 8;    // channels per thread (C <= 8 * 256)

struct ColStatsParams {
  DevState* ds;
  In x, dy;
  long long R, C;
  int mode;
  double* part;              // [gridDim.x][C][4]
  double* stats;             // [C][4]: mean, rstd, mean(dy), mean(dy*xhat)   (COL_BN, COL_BN_DX)
  unsigned int* counter;     // zero-initialised; reset by the last block
  In a, b;                   // node operands (ping-pong output choice only)
  Out out;                   // [C] result (COL_SUM_ROWS, COL_BN_DGAMMA)
};

template <typename T>
__global__ void __launch_bounds__(256) k_colstats(ColStatsParams p) {
  stamp(p.ds, SK_REDUCE);
  if (skip(p.ds)) return;
  const T* x = res<T>(p.x);
  const bool with_dy = p.mode == COL_BN_DX || p.mode == COL_BN_DGAMMA;
  const T* dy = with_dy ? res<T>(p.dy) : nullptr;
  const bool final_out = p.mode == COL_SUM_ROWS || p.mode == COL_BN_DGAMMA;
  T* o = nullptr;
  if (final_out) {
    o = pick_out<T>(p.out, res<T>(p.a), p.b.cell || p.b.direct ? res<T>(p.b) : nullptr);
    publish_early(p.out, o);
  }
  count_op(p.ds);
  const long long C = p.C, R = p.R;
  const int L = (int)(C < 256 ? C : 256);          // lanes per row
  const int rpi = 256 / L;                         // rows per iteration
  const int t = threadIdx.x, cc = t % L, rr = t / L;
  const int slots = (int)((C + L - 1) / L);
  // row range of this block
  const long long r_begin = R * blockIdx.x / gridDim.x, r_end = R * (blockIdx.x + 1) / gridDim.x;
  double a1[kColMaxSlots], a2[kColMaxSlots], a3[kColMaxSlots], a4[kColMaxSlots], sh[kColMaxSlots];
#pragma unroll
  for (int j = 0; j < kColMaxSlots; ++j) {
    a1[j] = a2[j] = a3[j] = a4[j] = 0.0;
    const long long c = cc + (long long)j * L;
    sh[j] = (p.mode != COL_SUM_ROWS && j < slots && c < C) ? (double)x[c] : 0.0;
  }
  if (rr < rpi) {
    for (long long r = r_begin + rr; r < r_end; r += rpi) {
#pragma unroll
      for (int j = 0; j < kColMaxSlots; ++j) {
        const long long c = cc + (long long)j * L;
        if (j < slots && c < C) {
          const double v = (double)x[r * C + c] - sh[j];
          a1[j] += v;
          a2[j] += v * v;
          if (with_dy) {
            const double g = (double)dy[r * C + c];
            a3[j] += g;
            a4[j] += g * v;
          }
        }
      }
    }
  }
  __shared__ double sm[256][4];
  for (int j = 0; j < slots; ++j) {
    sm[t][0] = a1[j]; sm[t][1] = a2[j]; sm[t][2] = a3[j]; sm[t][3] = a4[j];
    __syncthreads();
    const long long c = t + (long long)j * L;
    if (t < L && c < C) {
      double s[4] = {0.0, 0.0, 0.0, 0.0};
      for (int q = 0; q < rpi; ++q)
        for (int u = 0; u < 4; ++u) s[u] += sm[q * L + t][u];
      double* dst = p.part + ((long long)blockIdx.x * C + c) * 4;
      for (int u = 0; u < 4; ++u) dst[u] = s[u];
    }
    __syncthreads();
  }
  // last block: combine partials (block order) and finalise
  __shared__ unsigned int last;
  __threadfence();
  if (t == 0) last = (atomicAdd(p.counter, 1u) == gridDim.x - 1) ? 1u : 0u;
  __syncthreads();
  if (!last) return;
  __threadfence();
  for (long long c = t; c < C; c += blockDim.x) {
    double s1 = 0.0, s2 = 0.0, d1 = 0.0, d2 = 0.0;
    for (unsigned int b = 0; b < gridDim.x; ++b) {
      const double* q = p.part + ((long long)b * C + c) * 4;
      s1 += q[0]; s2 += q[1]; d1 += q[2]; d2 += q[3];
    }
    if (p.mode == COL_SUM_ROWS) {
      o[c] = (T)s1;
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
    double* st = p.stats + c * 4;
    st[0] = mean;
    st[1] = rstd;
    st[2] = d1 / (double)R;
    st[3] = sdx / (double)R;
  }
  if (t == 0) *p.counter = 0u;
  if (final_out) {
    __syncthreads();
    if (t == 0 && p.out.late != nullptr)   // single finishing block publishes
      for (int i = 0; i < p.out.npub; ++i) *p.out.pub[i] = o;
  }
}

// ------------------------------------------------------------------ batch-norm apply
struct BnApplyParams {
  DevState* ds;
  In x, g, third;            // BATCHNORM: third = beta [C]; BATCHNORM_DX: third = dy (x's shape)
  const double* stats;       // [C][4]
  long long n, C;
  int dx;                    // 0: y = ((x-mean)*rstd)*g + b; 1: dx = (dy - m(dy) - xhat*m(dy*xhat)) * (g*rstd)
  Out out;
};

template <typename T>
__global__ void __launch_bounds__(256) k_bn_apply(BnApplyParams p) {
  stamp(p.ds, SK_EW);
  if (skip(p.ds)) return;
  const T* x = res<T>(p.x);
  const T* g = res<T>(p.g);
  const T* z = res<T>(p.third);
  T* o = pick_out<T>(p.out, x, g);
  publish_early(p.out, o);
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
  }
  publish_late(p.out, o);
}

}  // namespace coex
