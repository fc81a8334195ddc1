// xformer_ops.cuh -- sm_100a kernels of the transformer extension op set (config C4,
// GPT-2 small; SURVEY §2.4, §8(a) row a*).  Semantics: oracle/kernels.py
// transformer_kernel (builder-defined, parity unpinned by the reference).
//
// Row kernels (layernorm, causal softmax, cross-entropy) give one warp (or one block
// for vocabulary-wide rows) to a row, keep the row in registers / L1, and reduce with
// warp shuffles in double.  Column sums (ln_dgamma) reuse the fp64-atomic replicated
// accumulator scheme of k_colstats.  The batched GEMMs (bmm*) are lowered by the runtime
// to the tcgen05 kernel (bf16 mode, 3-D tensor maps) or the batched SIMT kernel.
#pragma once
#include <cooperative_groups.h>
#include "ext_ops.cuh"

namespace coex {

constexpr double kLnEps = 1e-5;
constexpr double kGeluC = 0.7978845608028654;

struct RowParams {
  DevState* ds;
  In x, y, z;                // operands (meaning per kernel)
  long long rows, d;         // row count, row length
  int T;                     // causal softmax: rows per [T, T] block
  double scale;
  long long vocab;           // embedding / cross-entropy
  double* acc;               // column accumulators (ln_dgamma) / per-row losses (cross-entropy)
  unsigned int* counter;
  Out out;
  __nv_bfloat16* shadow;     // optional bf16 copy of the output (consumed by batched GEMMs)
  Out out2;                  // fused cross-entropy: the loss (out = the gradient)
  long long spitch;          // shadow row pitch (elements; >= d, multiple of 8)
  int skip_f32;              // fused cross-entropy: the fp32 gradient has no reader (GEMMs read the shadow)
};

template <typename A>
__device__ __forceinline__ A warp_sum(A v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}
template <typename A>
__device__ __forceinline__ A warp_max(A v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}
// softmax-type rows accumulate in the storage precision's natural type (f64 parity mode:
// double; fp32 / bf16 modes: float -- exp in double would make them ALU-bound)
template <typename T> struct AccT { typedef float type; };
template <> struct AccT<double> { typedef double type; };
__device__ __forceinline__ float ex(float v) { return __expf(v); }
__device__ __forceinline__ double ex(double v) { return exp(v); }

// last-block election after every block wrote its part (threadfence + counter)
__device__ __forceinline__ bool last_block(unsigned int* counter) {
  __shared__ unsigned int last;
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    last = (atomicAdd(counter, 1u) == gridDim.x - 1) ? 1u : 0u;
    if (last) __threadfence();
  }
  __syncthreads();
  return last != 0;
}

// ------------------------------------------------------------------ embedding
// out[r, :] = table[clip(ids[r]), :]   (x = table [V, d], y = ids [rows])
template <typename T>
__global__ void __launch_bounds__(256) k_embed(RowParams p) {
  COEX_PDL_ENTER();
  stamp(p.ds, SK_EMBED);
  const T* tab = res<T>(p.x);
  const T* ids = res<T>(p.y);
  T* o = pick_out<T>(p.out, tab, ids);
  publish_early(p.out, o);
  count_op(p.ds);
  const long long total = p.rows * p.d;
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < total; i += (long long)gridDim.x * blockDim.x) {
    const long long r = i / p.d, c = i - r * p.d;
    double f = floor((double)ids[r]);
    long long v = f < 0 ? 0 : (f > (double)(p.vocab - 1) ? p.vocab - 1 : (long long)f);
    o[i] = tab[v * p.d + c];
  }
  publish_late(p.out, o);
}

// out[v, :] = sum over rows r with ids[r] == v of dy[r, :] (atomics; the output is zeroed
// by the preceding k_zero launch)   (x = ids [rows], y = dy [rows, d])
template <typename T>
__global__ void __launch_bounds__(256) k_embed_dw(RowParams p) {
  COEX_PDL_ENTER();
  stamp(p.ds, SK_EMBED);
  const T* ids = res<T>(p.x);
  const T* dy = res<T>(p.y);
  T* o = pick_out<T>(p.out, ids, dy);
  publish_early(p.out, o);
  count_op(p.ds);
  const long long total = p.rows * p.d;
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < total; i += (long long)gridDim.x * blockDim.x) {
    const long long r = i / p.d, c = i - r * p.d;
    double f = floor((double)ids[r]);
    long long v = f < 0 ? 0 : (f > (double)(p.vocab - 1) ? p.vocab - 1 : (long long)f);
    atomicAdd(o + v * p.d + c, dy[i]);
  }
  publish_late(p.out, o);
}

struct ZeroParams {
  DevState* ds;
  Out out;
  long long bytes;
  In a, b;
};
__global__ void __launch_bounds__(256) k_zero(ZeroParams p) {
  COEX_PDL_ENTER();
  char* o = pick_out<char>(p.out, p.a.cell || p.a.direct ? res<char>(p.a) : nullptr,
                           p.b.cell || p.b.direct ? res<char>(p.b) : nullptr);
  const long long n16 = p.bytes / 16;
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n16; i += (long long)gridDim.x * blockDim.x)
    ((uint4*)o)[i] = make_uint4(0u, 0u, 0u, 0u);
  for (long long i = n16 * 16 + (long long)blockIdx.x * blockDim.x + threadIdx.x; i < p.bytes;
       i += (long long)gridDim.x * blockDim.x)
    o[i] = 0;
}

// ------------------------------------------------------------------ bias add
// out = x + b[i % d]
template <typename T>
__global__ void __launch_bounds__(256) k_bias_add(RowParams p) {
  COEX_PDL_ENTER();
  stamp(p.ds, SK_BIAS);
  const T* x = res<T>(p.x);
  const T* b = res<T>(p.y);
  T* o = pick_out<T>(p.out, x, b);
  publish_early(p.out, o);
  count_op(p.ds);
  const long long total = p.rows * p.d;
  const long long stride = (long long)gridDim.x * blockDim.x;
  if (sizeof(T) == 4 && (p.d & 3) == 0) {
    const long long d4 = p.d / 4;
    for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < total / 4; i += stride) {
      const float4 v = ((const float4*)x)[i];
      const float4 w = ((const float4*)b)[i % d4];
      ((float4*)o)[i] = make_float4(__fadd_rn(v.x, w.x), __fadd_rn(v.y, w.y), __fadd_rn(v.z, w.z), __fadd_rn(v.w, w.w));
    }
  } else {
    for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < total; i += stride)
      o[i] = ew_apply(EW_ADD, x[i], b[i % p.d]);
  }
  publish_late(p.out, o);
}

// ------------------------------------------------------------------ relative-attention skew (C5)
// Rows of [.., T, T] blocks, one warp per row, i = row index inside its block, s = T-1-i:
//   UN = 0 (rel_skew):   out[c] = c <= i ? x[c + s] : 0
//   UN = 1 (rel_unskew): out[m] = m >= s ? x[m - s] : 0      (the adjoint)
// Both are shifted contiguous copies: coalesced reads and writes, HBM-bound.
template <typename T, int UN>
__global__ void __launch_bounds__(256) k_rel_skew(RowParams p) {
  COEX_PDL_ENTER();
  stamp(p.ds, SK_SKEW);
  const T* x = res<T>(p.x);
  T* o = pick_out<T>(p.out, x, nullptr);
  publish_early(p.out, o);
  count_op(p.ds);
  const int lane = threadIdx.x & 31;
  const long long warps = (long long)gridDim.x * (blockDim.x / 32);
  const long long d = p.d;
  for (long long r = (long long)blockIdx.x * (blockDim.x / 32) + threadIdx.x / 32; r < p.rows; r += warps) {
    const long long i = r % d, sh = d - 1 - i;
    const T* xr = x + r * d;
    T* orow = o + r * d;
    for (long long c = lane; c < d; c += 32) {
      if (UN == 0) orow[c] = c <= i ? xr[c + sh] : T(0);
      else orow[c] = c >= sh ? xr[c - sh] : T(0);
    }
  }
  publish_late(p.out, o);
}

// fp32 rows of 4 | d floats: the same shifted row copies four columns per lane per step --
// 16-byte stores, four scalar (shifted, unaligned) loads in flight, zero columns not read.
// FUSED (planner _skew_pairs, plan kind 104): out = a + rel_skew(x), the attention logits'
// add of the skewed relative term (y operand a = q.k^T) -- the skewed [BH, T, T] tensor never
// reaches HBM.  Same per-element additions as rel_skew followed by add.
template <int UN, bool FUSED>
__global__ void __launch_bounds__(256) k_rel_skew_v4(RowParams p) {
  COEX_PDL_ENTER();
  stamp(p.ds, SK_SKEW);
  const float* x = res<float>(p.x);
  const float* a = FUSED ? res<float>(p.y) : nullptr;
  float* o = pick_out<float>(p.out, x, a);
  publish_early(p.out, o);
  count_op(p.ds);
  const int lane = threadIdx.x & 31;
  const long long warps = (long long)gridDim.x * (blockDim.x / 32);
  const int d = (int)p.d, d4 = d / 4;
  for (long long r = (long long)blockIdx.x * (blockDim.x / 32) + threadIdx.x / 32; r < p.rows; r += warps) {
    const int i = (int)(r % d), sh = d - 1 - i;
    const float* xr = x + r * d;
    float4* orow = (float4*)(o + r * d);
    const float4* ar = FUSED ? (const float4*)(a + r * d) : nullptr;
    for (int q0 = lane; q0 < d4; q0 += 128) {      // four 16-byte groups per lane in flight
      float v[4][4];
      float4 av[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int q = q0 + 32 * u;
        if (FUSED) av[u] = q < d4 ? ar[q] : make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          const int c = 4 * q + e;
          const bool in = q < d4 && (UN == 0 ? c <= i : c >= sh);
          v[u][e] = in ? xr[UN == 0 ? c + sh : c - sh] : 0.f;
        }
      }
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int q = q0 + 32 * u;
        if (q >= d4) break;
        float4 w = make_float4(v[u][0], v[u][1], v[u][2], v[u][3]);
        if (FUSED) w = make_float4(av[u].x + w.x, av[u].y + w.y, av[u].z + w.z, av[u].w + w.w);
        orow[q] = w;
        if (p.shadow) {                               // bf16 GEMM-operand copy (C5 unskew)
          __nv_bfloat162 h0 = __floats2bfloat162_rn(w.x, w.y), h1 = __floats2bfloat162_rn(w.z, w.w);
          ((uint2*)(p.shadow + r * d))[q] = make_uint2(*(uint32_t*)&h0, *(uint32_t*)&h1);
        }
      }
    }
  }
  publish_late(p.out, o);
}

// ------------------------------------------------------------------ layernorm
// One warp per row; the row is read twice (mean, then centred moments) from L1/L2.
template <typename T>
__device__ __forceinline__ void ln_row_stats(const T* xr, long long d, int lane, double& mean, double& rstd) {
  double s = 0.0;
  for (long long c = lane; c < d; c += 32) s += (double)xr[c];
  mean = warp_sum(s) / (double)d;
  double q = 0.0;
  for (long long c = lane; c < d; c += 32) {
    const double v = (double)xr[c] - mean;
    q += v * v;
  }
  rstd = 1.0 / sqrt(warp_sum(q) / (double)d + kLnEps);
}

// mode 0: y = xhat*g + b (x, g = y operand, b = z operand); mode 1: dx (x, g, dy = z)
template <typename T, int MODE>
__global__ void __launch_bounds__(256) k_layernorm(RowParams p) {
  COEX_PDL_ENTER();
  stamp(p.ds, SK_LN);
  const T* x = res<T>(p.x);
  const T* g = res<T>(p.y);
  const T* z = res<T>(p.z);
  T* o = pick_out<T>(p.out, x, g);
  publish_early(p.out, o);
  count_op(p.ds);
  const int lane = threadIdx.x & 31;
  const long long warps = (long long)gridDim.x * (blockDim.x / 32);
  if (p.d <= 768 && sizeof(T) == 4) {               // fp32 rows up to 768 held in registers
    constexpr int PER = 24;
    const long long d = p.d;
    for (long long r = (long long)blockIdx.x * (blockDim.x / 32) + threadIdx.x / 32; r < p.rows; r += warps) {
      const T* xr = x + r * d;
      float xv[PER];
      float s1 = 0.f;
#pragma unroll
      for (int j = 0; j < PER; ++j) {
        const long long c = lane + 32ll * j;
        xv[j] = c < d ? (float)xr[c] : 0.f;
        s1 += xv[j];
      }
      const float mean = warp_sum(s1) / (float)d;
      float s2 = 0.f;
#pragma unroll
      for (int j = 0; j < PER; ++j) {
        const long long c = lane + 32ll * j;
        const float t = c < d ? xv[j] - mean : 0.f;
        s2 += t * t;
      }
      const float rstd = rsqrtf(warp_sum(s2) / (float)d + (float)kLnEps);
      if (MODE == 0) {
#pragma unroll
        for (int j = 0; j < PER; ++j) {
          const long long c = lane + 32ll * j;
          if (c < d) {
            const T v = (T)(((xv[j] - mean) * rstd) * (float)g[c] + (float)z[c]);
            o[r * d + c] = v;
            if (p.shadow) p.shadow[r * d + c] = __float2bfloat16_rn((float)v);   // GEMM operand copy
          }
        }
      } else {
        const T* dyr = z + r * d;
        float gv[PER];
        float m1 = 0.f, m2 = 0.f;
#pragma unroll
        for (int j = 0; j < PER; ++j) {
          const long long c = lane + 32ll * j;
          gv[j] = c < d ? (float)dyr[c] * (float)g[c] : 0.f;
          m1 += gv[j];
          m2 += c < d ? gv[j] * ((xv[j] - mean) * rstd) : 0.f;
        }
        m1 = warp_sum(m1) / (float)d;
        m2 = warp_sum(m2) / (float)d;
#pragma unroll
        for (int j = 0; j < PER; ++j) {
          const long long c = lane + 32ll * j;
          if (c < d) o[r * d + c] = (T)(((gv[j] - m1) - ((xv[j] - mean) * rstd) * m2) * rstd);
        }
      }
    }
    publish_late(p.out, o);
    return;
  }
  for (long long r = (long long)blockIdx.x * (blockDim.x / 32) + threadIdx.x / 32; r < p.rows; r += warps) {
    const T* xr = x + r * p.d;
    double mean, rstd;
    ln_row_stats(xr, p.d, lane, mean, rstd);
    if (MODE == 0) {
      for (long long c = lane; c < p.d; c += 32) {
        const T v = (T)((((double)xr[c] - mean) * rstd) * (double)g[c] + (double)z[c]);
        o[r * p.d + c] = v;
        if (p.shadow) p.shadow[r * p.d + c] = __float2bfloat16_rn((float)v);
      }
    } else {
      const T* dy = z + r * p.d;
      double m1 = 0.0, m2 = 0.0;
      for (long long c = lane; c < p.d; c += 32) {
        const double dxh = (double)dy[c] * (double)g[c];
        m1 += dxh;
        m2 += dxh * (((double)xr[c] - mean) * rstd);
      }
      m1 = warp_sum(m1) / (double)p.d;
      m2 = warp_sum(m2) / (double)p.d;
      for (long long c = lane; c < p.d; c += 32) {
        const double xh = ((double)xr[c] - mean) * rstd;
        o[r * p.d + c] = (T)((((double)dy[c] * (double)g[c] - m1) - xh * m2) * rstd);
      }
    }
  }
  publish_late(p.out, o);
}

// fp32 rows with 4 | d <= 1024 (C4 / C5: 768 / 512): one warp per row, 16-byte accesses --
// lane l holds float4 groups l, l+32, ... (PER = d / 128 of them) -- so a row is a handful of
// coalesced 512-byte instructions per operand; the bf16 shadow leaves as 8-byte stores.
// mode 0: y = xhat*g + b (+ shadow); mode 1: dx from (x, g, dy).  Same math as k_layernorm.
template <int MODE, int PER>
__global__ void __launch_bounds__(256) k_layernorm_v4(RowParams p) {
  COEX_PDL_ENTER();
  stamp(p.ds, SK_LN);
  const float* x = res<float>(p.x);
  const float* g = res<float>(p.y);
  const float* z = res<float>(p.z);
  float* o = pick_out<float>(p.out, x, g);
  publish_early(p.out, o);
  count_op(p.ds);
  const int lane = threadIdx.x & 31;
  const long long warps = (long long)gridDim.x * (blockDim.x / 32);
  const long long d = p.d, d4 = d / 4;
  const float4* g4 = (const float4*)g;
  const float4* z4 = (const float4*)z;
  for (long long r = (long long)blockIdx.x * (blockDim.x / 32) + threadIdx.x / 32; r < p.rows; r += warps) {
    const float4* xr = (const float4*)(x + r * d);
    float4 xv[PER];
    float s1 = 0.f;
#pragma unroll
    for (int j = 0; j < PER; ++j) {
      const long long c = lane + 32ll * j;
      xv[j] = c < d4 ? __ldcs(xr + c) : make_float4(0.f, 0.f, 0.f, 0.f);
      s1 += (xv[j].x + xv[j].y) + (xv[j].z + xv[j].w);
    }
    const float mean = warp_sum(s1) / (float)d;
    float s2 = 0.f;
#pragma unroll
    for (int j = 0; j < PER; ++j) {
      const long long c = lane + 32ll * j;
      if (c < d4) {
        const float a = xv[j].x - mean, b = xv[j].y - mean, e = xv[j].z - mean, f = xv[j].w - mean;
        s2 += (a * a + b * b) + (e * e + f * f);
      }
    }
    const float rstd = rsqrtf(warp_sum(s2) / (float)d + (float)kLnEps);
    if (MODE == 0) {
      float4* orow = (float4*)(o + r * d);
      uint2* srow = p.shadow ? (uint2*)(p.shadow + r * d) : nullptr;
#pragma unroll
      for (int j = 0; j < PER; ++j) {
        const long long c = lane + 32ll * j;
        if (c < d4) {
          const float4 gg = __ldg(g4 + c), bb = __ldg(z4 + c);
          float4 v;
          v.x = ((xv[j].x - mean) * rstd) * gg.x + bb.x;
          v.y = ((xv[j].y - mean) * rstd) * gg.y + bb.y;
          v.z = ((xv[j].z - mean) * rstd) * gg.z + bb.z;
          v.w = ((xv[j].w - mean) * rstd) * gg.w + bb.w;
          orow[c] = v;
          if (srow) {
            __nv_bfloat162 w0 = __floats2bfloat162_rn(v.x, v.y), w1 = __floats2bfloat162_rn(v.z, v.w);
            srow[c] = make_uint2(*(uint32_t*)&w0, *(uint32_t*)&w1);
          }
        }
      }
    } else {
      const float4* dyr = (const float4*)(z + r * d);
      float4 gv[PER];
      float m1 = 0.f, m2 = 0.f;
#pragma unroll
      for (int j = 0; j < PER; ++j) {
        const long long c = lane + 32ll * j;
        if (c < d4) {
          const float4 dy = __ldcs(dyr + c), gg = __ldg(g4 + c);
          gv[j] = make_float4(dy.x * gg.x, dy.y * gg.y, dy.z * gg.z, dy.w * gg.w);
          m1 += (gv[j].x + gv[j].y) + (gv[j].z + gv[j].w);
          m2 += (gv[j].x * ((xv[j].x - mean) * rstd) + gv[j].y * ((xv[j].y - mean) * rstd)) +
                (gv[j].z * ((xv[j].z - mean) * rstd) + gv[j].w * ((xv[j].w - mean) * rstd));
        } else {
          gv[j] = make_float4(0.f, 0.f, 0.f, 0.f);
        }
      }
      m1 = warp_sum(m1) / (float)d;
      m2 = warp_sum(m2) / (float)d;
      float4* orow = (float4*)(o + r * d);
#pragma unroll
      for (int j = 0; j < PER; ++j) {
        const long long c = lane + 32ll * j;
        if (c < d4) {
          float4 v;
          v.x = ((gv[j].x - m1) - ((xv[j].x - mean) * rstd) * m2) * rstd;
          v.y = ((gv[j].y - m1) - ((xv[j].y - mean) * rstd) * m2) * rstd;
          v.z = ((gv[j].z - m1) - ((xv[j].z - mean) * rstd) * m2) * rstd;
          v.w = ((gv[j].w - m1) - ((xv[j].w - mean) * rstd) * m2) * rstd;
          orow[c] = v;
        }
      }
    }
  }
  publish_late(p.out, o);
}

// Fused layernorm backward (planner _bn_bwd_groups, plan kind 103): layernorm_dx(x, g, dy),
// ln_dgamma(x, dy) and sum_rows(dy) over the same (x, dy) in ONE pass -- fp32, 4 | d <= 1024.
// Warps take rows (16-byte accesses as k_layernorm_v4) and write dx; every lane keeps its
// columns' sum(dy * xhat) and sum(dy) in registers over its rows, the block combines its
// warps in shared memory (fp64), adds into kColReplicas fp64 accumulator replicas, and the
// last block sums the replicas in order, writes dgamma / dbeta and re-zeroes them.
// (out = dx, out2 = dgamma, out3 = dbeta; p.acc = 2 * kColReplicas * d doubles)
struct LnBwdParams {
  RowParams p;
  Out out_g, out_b;
};
template <int PER>
__global__ void __launch_bounds__(256) k_ln_bwd_v4(const __grid_constant__ LnBwdParams lp) {
  COEX_PDL_ENTER();
  const RowParams& p = lp.p;
  const Out& out_g = lp.out_g;
  const Out& out_b = lp.out_b;
  stamp(p.ds, SK_LN);
  __shared__ double red[2][1024];
  const float* x = res<float>(p.x);
  const float* g = res<float>(p.y);
  const float* z = res<float>(p.z);
  float* o = pick_out<float>(p.out, x, g);
  float* og = pick_out<float>(out_g, x, g);
  float* ob = pick_out<float>(out_b, x, g);
  publish_early(p.out, o);
  publish_early(out_g, og);
  publish_early(out_b, ob);
  count_op(p.ds);
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const long long warps = (long long)gridDim.x * (blockDim.x / 32);
  const long long d = p.d, d4 = d / 4;
  const float4* g4 = (const float4*)g;
  float4 ag[PER], ab[PER];
#pragma unroll
  for (int j = 0; j < PER; ++j) {
    ag[j] = make_float4(0.f, 0.f, 0.f, 0.f);
    ab[j] = make_float4(0.f, 0.f, 0.f, 0.f);
  }
  for (int i = threadIdx.x; i < 2 * 1024; i += blockDim.x) (&red[0][0])[i] = 0.0;
  for (long long r = (long long)blockIdx.x * (blockDim.x / 32) + wid; r < p.rows; r += warps) {
    const float4* xr = (const float4*)(x + r * d);
    const float4* dyr = (const float4*)(z + r * d);
    float4 xv[PER], dv[PER];
    float s1 = 0.f;
#pragma unroll
    for (int j = 0; j < PER; ++j) {
      const long long c = lane + 32ll * j;
      xv[j] = c < d4 ? __ldcs(xr + c) : make_float4(0.f, 0.f, 0.f, 0.f);
      dv[j] = c < d4 ? __ldcs(dyr + c) : make_float4(0.f, 0.f, 0.f, 0.f);
      s1 += (xv[j].x + xv[j].y) + (xv[j].z + xv[j].w);
    }
    const float mean = warp_sum(s1) / (float)d;
    float s2 = 0.f;
#pragma unroll
    for (int j = 0; j < PER; ++j) {
      const long long c = lane + 32ll * j;
      if (c < d4) {
        xv[j] = make_float4(xv[j].x - mean, xv[j].y - mean, xv[j].z - mean, xv[j].w - mean);
        s2 += (xv[j].x * xv[j].x + xv[j].y * xv[j].y) + (xv[j].z * xv[j].z + xv[j].w * xv[j].w);
      }
    }
    const float rstd = rsqrtf(warp_sum(s2) / (float)d + (float)kLnEps);
    float m1 = 0.f, m2 = 0.f;
    float4 gv[PER];
#pragma unroll
    for (int j = 0; j < PER; ++j) {
      const long long c = lane + 32ll * j;
      if (c < d4) {
        const float4 gg = __ldg(g4 + c);
        const float4 xh = make_float4(xv[j].x * rstd, xv[j].y * rstd, xv[j].z * rstd, xv[j].w * rstd);
        xv[j] = xh;
        gv[j] = make_float4(dv[j].x * gg.x, dv[j].y * gg.y, dv[j].z * gg.z, dv[j].w * gg.w);
        m1 += (gv[j].x + gv[j].y) + (gv[j].z + gv[j].w);
        m2 += (gv[j].x * xh.x + gv[j].y * xh.y) + (gv[j].z * xh.z + gv[j].w * xh.w);
        ag[j].x += dv[j].x * xh.x; ag[j].y += dv[j].y * xh.y; ag[j].z += dv[j].z * xh.z; ag[j].w += dv[j].w * xh.w;
        ab[j].x += dv[j].x; ab[j].y += dv[j].y; ab[j].z += dv[j].z; ab[j].w += dv[j].w;
      } else {
        gv[j] = make_float4(0.f, 0.f, 0.f, 0.f);
      }
    }
    m1 = warp_sum(m1) / (float)d;
    m2 = warp_sum(m2) / (float)d;
    float4* orow = (float4*)(o + r * d);
#pragma unroll
    for (int j = 0; j < PER; ++j) {
      const long long c = lane + 32ll * j;
      if (c < d4)
        orow[c] = make_float4(((gv[j].x - m1) - xv[j].x * m2) * rstd, ((gv[j].y - m1) - xv[j].y * m2) * rstd,
                              ((gv[j].z - m1) - xv[j].z * m2) * rstd, ((gv[j].w - m1) - xv[j].w * m2) * rstd);
    }
  }
  publish_late(p.out, o);
  __syncthreads();                                   // red zeroed
  // warps of the block in order (fixed order per block): fp64 column partials
  for (int w = 0; w < 8; ++w) {
    if (wid == w) {
#pragma unroll
      for (int j = 0; j < PER; ++j) {
        const long long c = lane + 32ll * j;
        if (c < d4) {
          red[0][4 * c] += ag[j].x; red[0][4 * c + 1] += ag[j].y; red[0][4 * c + 2] += ag[j].z; red[0][4 * c + 3] += ag[j].w;
          red[1][4 * c] += ab[j].x; red[1][4 * c + 1] += ab[j].y; red[1][4 * c + 2] += ab[j].z; red[1][4 * c + 3] += ab[j].w;
        }
      }
    }
    __syncthreads();
  }
  double* acc = p.acc + (long long)(blockIdx.x % kColReplicas) * 2 * d;
  for (long long c = threadIdx.x; c < d; c += blockDim.x) {
    atomicAdd(acc + c, red[0][c]);
    atomicAdd(acc + d + c, red[1][c]);
  }
  if (!last_block(p.counter)) return;
  const unsigned int nrep = gridDim.x < (unsigned)kColReplicas ? gridDim.x : (unsigned)kColReplicas;
  for (long long c = threadIdx.x; c < d; c += blockDim.x) {
    double sg = 0.0, sb = 0.0;
    for (unsigned int q = 0; q < nrep; ++q) {
      double* a = p.acc + (long long)q * 2 * d;
      sg += __ldcg(a + c);
      sb += __ldcg(a + d + c);
      a[c] = 0.0;
      a[d + c] = 0.0;
    }
    og[c] = (float)sg;
    ob[c] = (float)sb;
  }
  if (threadIdx.x == 0) *p.counter = 0u;
  __syncthreads();
  if (threadIdx.x == 0) {
    if (out_g.late != nullptr)
      for (int i = 0; i < out_g.npub; ++i) *out_g.pub[i] = og;
    if (out_b.late != nullptr)
      for (int i = 0; i < out_b.npub; ++i) *out_b.pub[i] = ob;
  }
}

// ln_dgamma: out[c] = sum over rows of dy * xhat (x, dy = y operand).  Warps take rows; each
// lane accumulates its columns in double, blocks add into kColReplicas fp64 accumulators,
// the last block sums the replicas, writes the output and re-zeroes the accumulators.
template <typename T>
__global__ void __launch_bounds__(256) k_ln_dgamma(RowParams p) {
  COEX_PDL_ENTER();
  stamp(p.ds, SK_LN);
  const T* x = res<T>(p.x);
  const T* dy = res<T>(p.y);
  T* o = pick_out<T>(p.out, x, dy);
  publish_early(p.out, o);
  count_op(p.ds);
  constexpr int MAXC = 32;                          // columns per lane (d <= 1024)
  const int lane = threadIdx.x & 31;
  double accl[MAXC];
#pragma unroll
  for (int j = 0; j < MAXC; ++j) accl[j] = 0.0;
  const long long warps = (long long)gridDim.x * (blockDim.x / 32);
  for (long long r = (long long)blockIdx.x * (blockDim.x / 32) + threadIdx.x / 32; r < p.rows; r += warps) {
    const T* xr = x + r * p.d;
    double mean, rstd;
    ln_row_stats(xr, p.d, lane, mean, rstd);
#pragma unroll
    for (int j = 0; j < MAXC; ++j) {
      const long long c = lane + 32ll * j;
      if (c < p.d) accl[j] += (double)dy[r * p.d + c] * (((double)xr[c] - mean) * rstd);
    }
  }
  double* accr = p.acc + (long long)(blockIdx.x % kColReplicas) * p.d;
#pragma unroll
  for (int j = 0; j < MAXC; ++j) {
    const long long c = lane + 32ll * j;
    if (c < p.d && accl[j] != 0.0) atomicAdd(accr + c, accl[j]);
  }
  if (!last_block(p.counter)) return;
  const unsigned int nrep = gridDim.x < (unsigned)kColReplicas ? gridDim.x : (unsigned)kColReplicas;
  for (long long c = threadIdx.x; c < p.d; c += blockDim.x) {
    double s = 0.0;
    for (unsigned int q = 0; q < nrep; ++q) {
      s += __ldcg(p.acc + (long long)q * p.d + c);
      p.acc[(long long)q * p.d + c] = 0.0;
    }
    o[c] = (T)s;
  }
  if (threadIdx.x == 0) *p.counter = 0u;
  __syncthreads();
  if (threadIdx.x == 0 && p.out.late != nullptr)
    for (int i = 0; i < p.out.npub; ++i) *p.out.pub[i] = o;
}

// ------------------------------------------------------------------ causal softmax
// One warp per row of a [T, T] block: row i keeps columns j <= i; y = exp(s*x - max) / sum.
template <typename T>
__global__ void __launch_bounds__(256) k_causal_softmax(RowParams p) {
  COEX_PDL_ENTER();
  stamp(p.ds, SK_SOFTMAX);
  const T* x = res<T>(p.x);
  T* o = pick_out<T>(p.out, x, nullptr);
  publish_early(p.out, o);
  count_op(p.ds);
  const int lane = threadIdx.x & 31;
  const long long warps = (long long)gridDim.x * (blockDim.x / 32);
  const long long d = p.d;
  typedef typename AccT<T>::type A;
  const A sc = (A)p.scale;
  if (d <= 1024) {                                  // row held in registers: one read, one write
    constexpr int PER = 32;
    for (long long r = (long long)blockIdx.x * (blockDim.x / 32) + threadIdx.x / 32; r < p.rows; r += warps) {
      const long long i = r % p.T;
      const T* xr = x + r * d;
      T* orow = o + r * d;
      A v[PER];
      A mx = -INFINITY;
#pragma unroll
      for (int j = 0; j < PER; ++j) {
        const long long c = lane + 32ll * j;
        v[j] = c <= i ? (A)xr[c] * sc : -INFINITY;
        mx = fmax(mx, v[j]);
      }
      mx = warp_max(mx);
      A sm = 0;
#pragma unroll
      for (int j = 0; j < PER; ++j) {
        const long long c = lane + 32ll * j;
        v[j] = c <= i ? ex(v[j] - mx) : (A)0;
        sm += v[j];
      }
      const A inv = (A)1 / warp_sum(sm);
#pragma unroll
      for (int j = 0; j < PER; ++j) {
        const long long c = lane + 32ll * j;
        if (c < d) {
          const A y = v[j] * inv;
          orow[c] = (T)y;
          if (p.shadow) p.shadow[r * d + c] = __float2bfloat16_rn((float)y);
        }
      }
    }
    publish_late(p.out, o);
    return;
  }
  for (long long r = (long long)blockIdx.x * (blockDim.x / 32) + threadIdx.x / 32; r < p.rows; r += warps) {
    const long long i = r % p.T;                    // row index inside its [T, T] block
    const T* xr = x + r * d;
    T* orow = o + r * d;
    A mx = -INFINITY;
    for (long long c = lane; c <= i; c += 32) mx = fmax(mx, (A)xr[c] * sc);
    mx = warp_max(mx);
    A s = 0;
    for (long long c = lane; c <= i; c += 32) s += ex((A)xr[c] * sc - mx);
    s = warp_sum(s);
    const A inv = (A)1 / s;
    for (long long c = lane; c < d; c += 32) {
      const A v = c <= i ? ex((A)xr[c] * sc - mx) * inv : (A)0;
      orow[c] = (T)v;
      if (p.shadow) p.shadow[r * d + c] = __float2bfloat16_rn((float)v);
    }
  }
  publish_late(p.out, o);
}

// dx = scale * y * (dy - sum_j dy*y)   (x = y, y = dy operand)
template <typename T>
__global__ void __launch_bounds__(256) k_softmax_grad(RowParams p) {
  COEX_PDL_ENTER();
  stamp(p.ds, SK_SOFTMAX_GRAD);
  const T* y = res<T>(p.x);
  const T* dy = res<T>(p.y);
  T* o = pick_out<T>(p.out, y, dy);
  publish_early(p.out, o);
  count_op(p.ds);
  const int lane = threadIdx.x & 31;
  const long long warps = (long long)gridDim.x * (blockDim.x / 32);
  const long long d = p.d;
  typedef typename AccT<T>::type A;
  if (d <= 1024) {                                  // rows held in registers: y and dy read once
    constexpr int PER = 32;
    for (long long r = (long long)blockIdx.x * (blockDim.x / 32) + threadIdx.x / 32; r < p.rows; r += warps) {
      const T* yr = y + r * d;
      const T* gr = dy + r * d;
      A yv[PER], gv[PER];
      A dot = 0;
#pragma unroll
      for (int j = 0; j < PER; ++j) {
        const long long c = lane + 32ll * j;
        yv[j] = c < d ? (A)yr[c] : (A)0;
        gv[j] = yv[j] != (A)0 ? (A)gr[c] : (A)0;
        dot += gv[j] * yv[j];
      }
      dot = warp_sum(dot);
#pragma unroll
      for (int j = 0; j < PER; ++j) {
        const long long c = lane + 32ll * j;
        if (c < d) {
          const A v = yv[j] != (A)0 ? (A)p.scale * (yv[j] * (gv[j] - dot)) : (A)0;
          o[r * d + c] = (T)v;
          if (p.shadow) p.shadow[r * d + c] = __float2bfloat16_rn((float)v);
        }
      }
    }
    publish_late(p.out, o);
    return;
  }
  for (long long r = (long long)blockIdx.x * (blockDim.x / 32) + threadIdx.x / 32; r < p.rows; r += warps) {
    const T* yr = y + r * d;
    const T* gr = dy + r * d;
    // entries with y == 0 (causal mask) contribute nothing and their dy is never read (the
    // planner may skip computing dy there)
    A dot = 0;
    for (long long c = lane; c < d; c += 32) {
      const A yv = (A)yr[c];
      if (yv != (A)0) dot += (A)gr[c] * yv;
    }
    dot = warp_sum(dot);
    for (long long c = lane; c < d; c += 32) {
      const A yv = (A)yr[c];
      const A v = yv != (A)0 ? (A)p.scale * (yv * ((A)gr[c] - dot)) : (A)0;
      o[r * d + c] = (T)v;
      if (p.shadow) p.shadow[r * d + c] = __float2bfloat16_rn((float)v);
    }
  }
  publish_late(p.out, o);
}

// ------------------------------------------------------------------ cross-entropy
// One block per row (vocabulary-wide rows).  MODE 0: loss row values into p.acc, the last
// block writes their mean (ordered sum: deterministic); MODE 1: (softmax - onehot) / rows.
template <typename T, int MODE>
__global__ void __launch_bounds__(256) k_cross_entropy(RowParams p) {
  COEX_PDL_ENTER();
  stamp(p.ds, SK_CE);
  typedef typename AccT<T>::type A;
  const T* lg = res<T>(p.x);
  const T* ids = res<T>(p.y);
  T* o = pick_out<T>(p.out, lg, ids);
  if (MODE == 1) publish_early(p.out, o);
  count_op(p.ds);
  __shared__ A redm[32], reds[32];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
  const long long V = p.d;
  for (long long r = blockIdx.x; r < p.rows; r += gridDim.x) {
    const T* row = lg + r * V;
    // online max / sum of exponentials in one pass (rescaling the partial sum on a new max)
    // groups of 4 independent loads per thread (memory-level parallelism), merged online
    A mx = -INFINITY, sm = 0;
    const long long step = blockDim.x;
    long long c = threadIdx.x;
    for (; c + 3 * step < V; c += 4 * step) {
      const A v0 = (A)row[c], v1 = (A)row[c + step], v2 = (A)row[c + 2 * step], v3 = (A)row[c + 3 * step];
      const A m4 = fmax(fmax(v0, v1), fmax(v2, v3));
      if (m4 > mx) {
        sm = mx == -INFINITY ? (A)0 : sm * ex(mx - m4);
        mx = m4;
      }
      sm += (ex(v0 - mx) + ex(v1 - mx)) + (ex(v2 - mx) + ex(v3 - mx));
    }
    for (; c < V; c += step) {
      const A v = (A)row[c];
      if (v > mx) {
        sm = mx == -INFINITY ? (A)1 : sm * ex(mx - v) + (A)1;
        mx = v;
      } else {
        sm += ex(v - mx);
      }
    }
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) {
      const A om = __shfl_xor_sync(0xffffffffu, mx, off), os = __shfl_xor_sync(0xffffffffu, sm, off);
      const A nm = fmax(mx, om);
      sm = (mx == -INFINITY ? (A)0 : sm * ex(mx - nm)) + (om == -INFINITY ? (A)0 : os * ex(om - nm));
      mx = nm;
    }
    if (lane == 0) { redm[wid] = mx; reds[wid] = sm; }
    __syncthreads();
    A gm = redm[0];
    for (int w = 1; w < nw; ++w) gm = fmax(gm, redm[w]);
    A gs = 0;
    for (int w = 0; w < nw; ++w) gs += redm[w] == -INFINITY ? (A)0 : reds[w] * ex(redm[w] - gm);
    __syncthreads();
    double f = floor((double)ids[r]);
    const long long id = f < 0 ? 0 : (f > (double)(V - 1) ? V - 1 : (long long)f);
    if (MODE == 0) {
      if (threadIdx.x == 0) p.acc[r] = ((double)log(gs) + (double)gm) - (double)row[id];
    } else {
      const A inv = (A)1 / gs, invr = (A)(1.0 / (p.scale > 0.0 ? p.scale : (double)p.rows));   // scale: global rows
      T* orow = o + r * V;
#pragma unroll 4
      for (long long c2 = threadIdx.x; c2 < V; c2 += blockDim.x) {
        A g = ex((A)row[c2] - gm) * inv;
        if (c2 == id) g -= (A)1;
        orow[c2] = (T)(g * invr);
      }
    }
  }
  if (MODE == 1) {
    publish_late(p.out, o);
    return;
  }
  if (!last_block(p.counter)) return;
  if (threadIdx.x == 0) {
    double acc = 0.0;
    for (long long r = 0; r < p.rows; ++r) acc += __ldcg(p.acc + r);
    o[0] = (T)(acc / (double)p.rows);
    *p.counter = 0u;
    for (int i = 0; i < p.out.npub; ++i) *p.out.pub[i] = o;
  }
}

// Fused cross-entropy (planner: cross_entropy + cross_entropy_grad of the same logits and
// ids; tolerance modes).  One block per row; the row is staged in shared memory on its one
// HBM read (max on the fly), its exponentials cached in place, and the gradient
// (softmax - onehot) / rows written from shared memory -- in fp32 (unless no reader needs
// it) and as the bf16 GEMM-operand shadow [rows][spitch] the LM-head weight / input
// gradient GEMMs read.  Row losses go to acc; the last block writes their mean in row order.
// HBM: logits once in, gradient out (vs. two full reads and a conversion pass unfused).
template <int NT>
__device__ __forceinline__ float block_reduce(float v, bool is_max, float* red) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) {
    const float o = __shfl_xor_sync(0xffffffffu, v, off);
    v = is_max ? fmaxf(v, o) : v + o;
  }
  if (lane == 0) red[wid] = v;
  __syncthreads();
  float r = red[0];
  for (int w = 1; w < NT / 32; ++w) r = is_max ? fmaxf(r, red[w]) : r + red[w];
  __syncthreads();
  return r;
}

template <int NT>
__global__ void __launch_bounds__(NT) k_ce_fused(RowParams p) {
  COEX_PDL_ENTER();
  stamp(p.ds, SK_CE);
  extern __shared__ float srow[];
  __shared__ float red[NT / 32];
  const float* lg = res<float>(p.x);
  const float* ids = res<float>(p.y);
  float* o = pick_out<float>(p.out, lg, ids);
  float* lo = pick_out<float>(p.out2, lg, ids);
  publish_early(p.out, o);
  count_op(p.ds);
  const long long V = p.d;
  const float invr = (float)(1.0 / (p.scale > 0.0 ? p.scale : (double)p.rows));   // scale: global rows
  for (long long r = blockIdx.x; r < p.rows; r += gridDim.x) {
    const float* row = lg + r * V;
    float mx = -INFINITY;
    long long c = threadIdx.x;
    for (; c + 7 * NT < V; c += 8 * NT) {            // eight independent loads in flight
      float v[8];
#pragma unroll
      for (int q = 0; q < 8; ++q) v[q] = __ldcs(row + c + q * NT);
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        srow[c + q * NT] = v[q];
        mx = fmaxf(mx, v[q]);
      }
    }
    for (; c < V; c += NT) {
      const float v = __ldcs(row + c);
      srow[c] = v;
      mx = fmaxf(mx, v);
    }
    const float gm = block_reduce<NT>(mx, true, red);
    float sm = 0.f;
    for (long long k = threadIdx.x; k < V; k += NT) {
      const float e = __expf(srow[k] - gm);
      srow[k] = e;
      sm += e;
    }
    const float gs = block_reduce<NT>(sm, false, red);
    const double f = floor((double)ids[r]);
    const long long id = f < 0 ? 0 : (f > (double)(V - 1) ? V - 1 : (long long)f);
    if (threadIdx.x == 0) p.acc[r] = ((double)logf(gs) + (double)gm) - (double)row[id];
    const float inv = 1.f / gs;
    float* orow = o + r * V;
    __nv_bfloat16* srow16 = p.shadow ? p.shadow + r * p.spitch : nullptr;
    for (long long k = threadIdx.x; k < V; k += NT) {
      float g = srow[k] * inv;
      if (k == id) g -= 1.f;
      g *= invr;
      if (!p.skip_f32) __stcs(orow + k, g);
      if (srow16) srow16[k] = __float2bfloat16_rn(g);
    }
    if (srow16)
      for (long long k = V + threadIdx.x; k < p.spitch; k += NT) srow16[k] = __float2bfloat16_rn(0.f);
    __syncthreads();                                  // srow reused by the next row
  }
  publish_late(p.out, o);
  if (!last_block(p.counter)) return;
  if (threadIdx.x == 0) {
    double acc = 0.0;
    for (long long r = 0; r < p.rows; ++r) acc += __ldcg(p.acc + r);
    lo[0] = (float)(acc / (double)p.rows);
    *p.counter = 0u;
    for (int i = 0; i < p.out2.npub; ++i) *p.out2.pub[i] = lo;
  }
}

// Fused cross-entropy over a CTA PAIR per row (wide vocabularies, C4: 50257): each CTA of a
// 2-CTA cluster stages one half of the row in shared memory (100 KB, so two CTAs -- two rows
// -- are resident per SM and one row's load phase overlaps the other's exp / store phases,
// where the one-CTA-per-row kernel leaves HBM idle); the pair combines its max and sum of
// exponentials through distributed shared memory (two cluster barriers per row).  Same
// arithmetic per element as k_ce_fused; the row sum is the two halves' sums added.
template <int NT>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(NT) k_ce_pair(RowParams p) {
  COEX_PDL_ENTER();
  stamp(p.ds, SK_CE);
  extern __shared__ float srow[];
  __shared__ float red[NT / 32];
  __shared__ float xch[2];                          // this CTA's (max, sum) for the peer
  __shared__ __align__(8) uint64_t lbar;            // bulk-copy completion of the staged half row
  namespace cg = cooperative_groups;
  cg::cluster_group cl = cg::this_cluster();
  const unsigned crank = cl.block_rank();
  const float* peer = cl.map_shared_rank(&xch[0], crank ^ 1u);
  const float* lg = res<float>(p.x);
  const float* ids = res<float>(p.y);
  float* o = pick_out<float>(p.out, lg, ids);
  float* lo = pick_out<float>(p.out2, lg, ids);
  publish_early(p.out, o);
  count_op(p.ds);
  const long long V = p.d, half = (V + 1) / 2;
  const long long c0 = crank * half, cn = (c0 + half < V ? c0 + half : V) - c0;
  const float invr = (float)(1.0 / (p.scale > 0.0 ? p.scale : (double)p.rows));
  const long long pairs = gridDim.x / 2;
  uint32_t lphase = 0;
  if (threadIdx.x == 0) {
    mbar_init(&lbar, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  for (long long r = blockIdx.x / 2; r < p.rows; r += pairs) {
    // stage the half row: its 16-byte-aligned body by ONE bulk copy (the copy engine keeps
    // the whole 100 KB in flight; the other resident CTA computes meanwhile), the <= 3 head /
    // tail scalars by plain loads.  Element k lives at srow[k + sh], sh = 4 - head, so the
    // body lands 16-byte aligned at srow[4].
    const float* row = lg + r * V + c0;
    const int head = (int)(((16 - ((uintptr_t)row & 15)) & 15) / 4) < cn ? (int)(((16 - ((uintptr_t)row & 15)) & 15) / 4)
                                                                           : (int)cn;
    const long long nb4 = (cn - head) / 4;            // 16-byte body groups
    const int sh = 4 - head;
    float* st = srow + sh;
    if (threadIdx.x == 0 && nb4 > 0) {
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");   // generic smem use of the last row
      mbar_expect_tx(&lbar, (uint32_t)(nb4 * 16));
      asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                       smem_u32(srow + 4)),
                   "l"(row + head), "r"((uint32_t)(nb4 * 16)), "r"(smem_u32(&lbar))
                   : "memory");
    }
    if (threadIdx.x < head) st[threadIdx.x] = __ldcs(row + threadIdx.x);
    for (long long k = head + nb4 * 4 + threadIdx.x; k < cn; k += NT) st[k] = __ldcs(row + k);
    if (nb4 > 0) {
      mbar_wait(&lbar, lphase);
      lphase ^= 1u;
    }
    __syncthreads();
    // smem passes over the staged half: the aligned body as float4 (srow[4 ..]), the head
    // (srow[sh .. 3]) and tail scalars apart -- a quarter of the instructions per element
    const int n4 = (int)nb4;
    const int tail0 = head + 4 * n4, ncn = (int)cn;
    float4* body4 = (float4*)(srow + 4);
    float mx = -INFINITY;
    for (int q = threadIdx.x; q < n4; q += NT) {
      const float4 v = body4[q];
      mx = fmaxf(mx, fmaxf(fmaxf(v.x, v.y), fmaxf(v.z, v.w)));
    }
    if (threadIdx.x < head) mx = fmaxf(mx, st[threadIdx.x]);
    for (int k = tail0 + threadIdx.x; k < ncn; k += NT) mx = fmaxf(mx, st[k]);
    float lm = block_reduce<NT>(mx, true, red);
    if (threadIdx.x == 0) xch[0] = lm;
    cl.sync();
    const float gm = fmaxf(lm, peer[0]);
    float sm = 0.f;
    for (int q = threadIdx.x; q < n4; q += NT) {
      float4 v = body4[q];
      v.x = __expf(v.x - gm); v.y = __expf(v.y - gm); v.z = __expf(v.z - gm); v.w = __expf(v.w - gm);
      body4[q] = v;
      sm += (v.x + v.y) + (v.z + v.w);
    }
    if (threadIdx.x < head) {
      const float e = __expf(st[threadIdx.x] - gm);
      st[threadIdx.x] = e;
      sm += e;
    }
    for (int k = tail0 + threadIdx.x; k < ncn; k += NT) {
      const float e = __expf(st[k] - gm);
      st[k] = e;
      sm += e;
    }
    const float ls = block_reduce<NT>(sm, false, red);
    if (threadIdx.x == 0) xch[1] = ls;
    cl.sync();
    const float gs = crank == 0 ? ls + peer[1] : peer[1] + ls;   // same order on both CTAs
    const double f = floor((double)ids[r]);
    const long long id = f < 0 ? 0 : (f > (double)(V - 1) ? V - 1 : (long long)f);
    if (crank == 0 && threadIdx.x == 0) p.acc[r] = ((double)logf(gs) + (double)gm) - (double)lg[r * V + id];
    const float inv = 1.f / gs;
    float* orow = o + r * V + c0;
    __nv_bfloat16* srow16 = p.shadow ? p.shadow + r * p.spitch + c0 : nullptr;
    const long long lid = id - c0;
    auto grad = [&](int k) {
      float g = st[k] * inv;
      if (k == lid) g -= 1.f;
      return g * invr;
    };
    if (!p.skip_f32)
      for (int k = threadIdx.x; k < ncn; k += NT) __stcs(orow + k, grad(k));
    if (srow16) {
      // bf16 shadow as 4-byte column pairs on even absolute columns (the shadow row pitch
      // is a multiple of 8); an odd first / last column of this half goes alone
      const int k0 = (int)(c0 & 1);                  // first k whose absolute column is even
      if (k0 && threadIdx.x == 0) srow16[0] = __float2bfloat16_rn(grad(0));
      for (int k = k0 + 2 * threadIdx.x; k + 1 < ncn; k += 2 * NT)
        *(__nv_bfloat162*)(srow16 + k) = __floats2bfloat162_rn(grad(k), grad(k + 1));
      if (((ncn - k0) & 1) && threadIdx.x == 0) srow16[ncn - 1] = __float2bfloat16_rn(grad(ncn - 1));
    }
    if (srow16 && crank == 1)
      for (long long k = cn + threadIdx.x; k < p.spitch - c0; k += NT) srow16[k] = __float2bfloat16_rn(0.f);
    __syncthreads();                                  // srow reused by the next row
  }
  cl.sync();                                          // no CTA leaves while its peer reads xch
  publish_late(p.out, o);
  if (!last_block(p.counter)) return;
  if (threadIdx.x == 0) {
    double acc = 0.0;
    for (long long r = 0; r < p.rows; ++r) acc += __ldcg(p.acc + r);
    lo[0] = (float)(acc / (double)p.rows);
    *p.counter = 0u;
    for (int i = 0; i < p.out2.npub; ++i) *p.out2.pub[i] = lo;
  }
}

// Streaming fused cross-entropy for wide vocabularies (C4: 50257): no shared-memory row --
// pass 1 reads the row once with 16-byte loads (online max / sum of exponentials per thread,
// merged across the block), pass 2 re-reads it (L2-resident: a few rows per SM in flight)
// and writes the gradient 8 columns per thread: the bf16 shadow as one 16-byte store, the
// fp32 gradient only when a reader needs it.  256 threads per row, several rows per SM, so
// HBM latency hides behind other rows instead of behind one 200 KB staging copy.
__device__ __forceinline__ void ce_merge(float& m, float& s, float m2, float s2) {
  const float mn = fmaxf(m, m2);
  s = (m == -INFINITY ? 0.f : s * __expf(m - mn)) + (m2 == -INFINITY ? 0.f : s2 * __expf(m2 - mn));
  m = mn;
}
__global__ void __launch_bounds__(256) k_ce_stream(RowParams p) {
  COEX_PDL_ENTER();
  stamp(p.ds, SK_CE);
  __shared__ float red_m[8], red_s[8];
  const float* lg = res<float>(p.x);
  const float* ids = res<float>(p.y);
  float* o = pick_out<float>(p.out, lg, ids);
  float* lo = pick_out<float>(p.out2, lg, ids);
  publish_early(p.out, o);
  count_op(p.ds);
  const long long V = p.d;
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  const float invr = (float)(1.0 / (p.scale > 0.0 ? p.scale : (double)p.rows));
  for (long long r = blockIdx.x; r < p.rows; r += gridDim.x) {
    const float* row = lg + r * V;
    // ---- pass 1: online (max, sum exp) over the row; 16-byte aligned body
    const int head = (int)((16 - ((uintptr_t)row & 15)) & 15) / 4;   // scalars before alignment
    const long long h = head < V ? head : V;
    const long long nv = (V - h) / 4;
    float m = -INFINITY, sm = 0.f;
    if (tid < h) {
      const float v = __ldcs(row + tid);
      m = v;
      sm = 1.f;
    }
    const float4* body = (const float4*)(row + h);
    long long i = tid;
    for (; i + 3 * 256 < nv; i += 4 * 256) {           // four 16-byte loads in flight
      float4 q[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) q[u] = __ldcs(body + i + u * 256);
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const float mx = fmaxf(fmaxf(q[u].x, q[u].y), fmaxf(q[u].z, q[u].w));
        const float s4 = __expf(q[u].x - mx) + __expf(q[u].y - mx) + __expf(q[u].z - mx) + __expf(q[u].w - mx);
        ce_merge(m, sm, mx, s4);
      }
    }
    for (; i < nv; i += 256) {
      const float4 q = __ldcs(body + i);
      const float mx = fmaxf(fmaxf(q.x, q.y), fmaxf(q.z, q.w));
      ce_merge(m, sm, mx, __expf(q.x - mx) + __expf(q.y - mx) + __expf(q.z - mx) + __expf(q.w - mx));
    }
    for (long long k = h + nv * 4 + tid; k < V; k += 256) ce_merge(m, sm, __ldcs(row + k), 1.f);
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) {
      const float m2 = __shfl_xor_sync(0xffffffffu, m, off), s2 = __shfl_xor_sync(0xffffffffu, sm, off);
      ce_merge(m, sm, m2, s2);
    }
    if (lane == 0) {
      red_m[wid] = m;
      red_s[wid] = sm;
    }
    __syncthreads();
    float gm = red_m[0], gs = red_s[0];
    for (int w = 1; w < 8; ++w) ce_merge(gm, gs, red_m[w], red_s[w]);
    __syncthreads();                                   // red_* reused by the next row
    const double f = floor((double)ids[r]);
    const long long id = f < 0 ? 0 : (f > (double)(V - 1) ? V - 1 : (long long)f);
    if (tid == 0) p.acc[r] = ((double)logf(gs) + (double)gm) - (double)row[id];
    // ---- pass 2: gradient, 8 columns per thread (one 16-byte bf16 shadow store)
    const float inv = 1.f / gs;
    float* orow = o + r * V;
    __nv_bfloat16* srow16 = p.shadow ? p.shadow + r * p.spitch : nullptr;
    const long long pitch = p.shadow ? p.spitch : (V + 7) / 8 * 8;
    // four 8-column chunks per iteration: all 32 loads issued before any use (L2 latency
    // overlapped instead of paid once per chunk)
    for (long long k00 = (long long)tid * 8; k00 < pitch; k00 += 4 * 256 * 8) {
      float g[4][8];
#pragma unroll
      for (int q = 0; q < 4; ++q)
#pragma unroll
        for (int u = 0; u < 8; ++u) {
          const long long k = k00 + q * 2048 + u;
          g[q][u] = k < V ? __ldg(row + k) : 0.f;
        }
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const long long k0 = k00 + q * 2048;
        if (k0 >= pitch) break;
#pragma unroll
        for (int u = 0; u < 8; ++u) {
          const long long k = k0 + u;
          float v = 0.f;
          if (k < V) {
            v = __expf(g[q][u] - gm) * inv;
            if (k == id) v -= 1.f;
            v *= invr;
            if (!p.skip_f32) __stcs(orow + k, v);
          }
          g[q][u] = v;
        }
        if (srow16) {
          __nv_bfloat162 w0 = __floats2bfloat162_rn(g[q][0], g[q][1]), w1 = __floats2bfloat162_rn(g[q][2], g[q][3]);
          __nv_bfloat162 w2 = __floats2bfloat162_rn(g[q][4], g[q][5]), w3 = __floats2bfloat162_rn(g[q][6], g[q][7]);
          uint4 pk;
          pk.x = *(uint32_t*)&w0; pk.y = *(uint32_t*)&w1; pk.z = *(uint32_t*)&w2; pk.w = *(uint32_t*)&w3;
          *(uint4*)(srow16 + k0) = pk;
        }
      }
    }
  }
  publish_late(p.out, o);
  if (!last_block(p.counter)) return;
  if (threadIdx.x == 0) {
    double acc = 0.0;
    for (long long r = 0; r < p.rows; ++r) acc += __ldcg(p.acc + r);
    lo[0] = (float)(acc / (double)p.rows);
    *p.counter = 0u;
    for (int i = 0; i < p.out2.npub; ++i) *p.out2.pub[i] = lo;
  }
}

// ------------------------------------------------------------------ wide column sums
// sum_rows for wide rows (C > 1024, e.g. the position-embedding gradient [B, T*d] or the MLP
// bias gradient [B*T, 4d]): each thread owns one column and adds a chunk of rows in order;
// one chunk -> written directly, several chunks (grid.y) -> fp64 atomics into p.acc and a
// k_acc_out pass.   (x operand, rows x d)
template <typename T>
__global__ void __launch_bounds__(256) k_colsum_wide(RowParams p) {
  COEX_PDL_ENTER();
  stamp(p.ds, SK_COLSUM);
  const T* x = res<T>(p.x);
  T* o = pick_out<T>(p.out, x, nullptr);
  if (gridDim.y == 1) publish_early(p.out, o);
  if (blockIdx.y == 0) count_op(p.ds);
  const long long c = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  const long long r0 = p.rows * blockIdx.y / gridDim.y, r1 = p.rows * (blockIdx.y + 1) / gridDim.y;
  if (c < p.d) {
    // four independent accumulators (combined in a fixed order) keep four loads in flight
    double a0 = 0.0, a1 = 0.0, a2 = 0.0, a3 = 0.0;
    long long r = r0;
    for (; r + 3 < r1; r += 4) {
      const double v0 = (double)x[r * p.d + c], v1 = (double)x[(r + 1) * p.d + c];
      const double v2 = (double)x[(r + 2) * p.d + c], v3 = (double)x[(r + 3) * p.d + c];
      a0 += v0; a1 += v1; a2 += v2; a3 += v3;
    }
    for (; r < r1; ++r) a0 += (double)x[r * p.d + c];
    const double acc = (a0 + a1) + (a2 + a3);
    if (gridDim.y == 1) o[c] = (T)acc;
    else atomicAdd(p.acc + c, acc);
  }
  if (gridDim.y == 1) publish_late(p.out, o);
}

// fp32, 4 | d: each thread owns FOUR columns (one 16-byte load per row) and a quarter of the
// block's rows (4 row lanes x 64 column groups = 256 columns per block), eight loads in
// flight; fp64 accumulation, the four row lanes combined in shared memory in a fixed order,
// then written (one row chunk) or added with fp64 atomics into p.acc (k_acc_out pass).
__global__ void __launch_bounds__(256) k_colsum_v4(RowParams p) {
  COEX_PDL_ENTER();
  stamp(p.ds, SK_COLSUM);
  __shared__ double part[4][64][4];
  const float* x = res<float>(p.x);
  float* o = pick_out<float>(p.out, x, nullptr);
  if (gridDim.y == 1) publish_early(p.out, o);
  if (blockIdx.y == 0 && blockIdx.x == 0) count_op(p.ds);
  const int cg = threadIdx.x & 63, rl = threadIdx.x >> 6;
  const long long c = ((long long)blockIdx.x * 64 + cg) * 4;
  const long long r0 = p.rows * blockIdx.y / gridDim.y, r1 = p.rows * (blockIdx.y + 1) / gridDim.y;
  double a0 = 0.0, a1 = 0.0, a2 = 0.0, a3 = 0.0;
  if (c < p.d) {
    const float* col = x + c;
    long long r = r0 + rl;
    for (; r + 28 < r1; r += 32) {                   // eight rows of this lane in flight
      float4 q[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) q[u] = __ldcs((const float4*)(col + (r + 4 * u) * p.d));
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        a0 += (double)q[u].x; a1 += (double)q[u].y; a2 += (double)q[u].z; a3 += (double)q[u].w;
      }
    }
    for (; r < r1; r += 4) {
      const float4 q = __ldcs((const float4*)(col + r * p.d));
      a0 += (double)q.x; a1 += (double)q.y; a2 += (double)q.z; a3 += (double)q.w;
    }
  }
  part[rl][cg][0] = a0;
  part[rl][cg][1] = a1;
  part[rl][cg][2] = a2;
  part[rl][cg][3] = a3;
  __syncthreads();
  if (rl == 0 && c < p.d) {
    for (int k = 0; k < 4; ++k) {
      const double v = (part[0][cg][k] + part[1][cg][k]) + (part[2][cg][k] + part[3][cg][k]);
      if (gridDim.y == 1) o[c + k] = (float)v;
      else atomicAdd(p.acc + c + k, v);
    }
  }
  if (gridDim.y == 1) {
    publish_late(p.out, o);
    return;
  }
  // several row chunks: the last block to finish writes the output from the fp64
  // accumulators and re-zeroes them (no separate k_acc_out launch)
  __shared__ unsigned int last;
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    last = atomicAdd(p.counter, 1u) == gridDim.x * gridDim.y - 1 ? 1u : 0u;
    if (last) __threadfence();
  }
  __syncthreads();
  if (!last) return;
  for (long long k = threadIdx.x; k < p.d; k += blockDim.x) {
    o[k] = (float)__ldcg(p.acc + k);
    p.acc[k] = 0.0;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    *p.counter = 0u;
    __threadfence();
    for (int i = 0; i < p.out.npub; ++i) *p.out.pub[i] = o;
  }
}

template <typename T>
__global__ void __launch_bounds__(256) k_acc_out(RowParams p) {
  COEX_PDL_ENTER();
  T* o = pick_out<T>(p.out, res<T>(p.x), nullptr);
  publish_early(p.out, o);
  for (long long c = (long long)blockIdx.x * blockDim.x + threadIdx.x; c < p.d; c += (long long)gridDim.x * blockDim.x) {
    o[c] = (T)p.acc[c];
    p.acc[c] = 0.0;                                  // re-zero for the next launch
  }
  publish_late(p.out, o);
}

// ------------------------------------------------------------------ axis ops (general)
// x viewed as [outer][A][inner] around the axis.  slice: out[o][j][i] = x[o][start + j][i];
// concat: out[o][j][i] = j < A ? a[o][j][i] : b[o][j - A][i]; sum_axis: out[o][i] = sequential
// sum over j from +0 (thread per output element, coalesced over i).
struct AxisParams {
  DevState* ds;
  In a, b;
  Out out;
  long long outer, A, A2, inner, start, length;
  int mode;                  // 0 slice, 1 concat, 2 sum_axis
};

template <typename T>
__global__ void __launch_bounds__(256) k_axis(AxisParams p) {
  COEX_PDL_ENTER();
  stamp(p.ds, SK_AXIS);
  const T* a = res<T>(p.a);
  const T* b = p.mode == 1 ? res<T>(p.b) : nullptr;
  T* o = pick_out<T>(p.out, a, b);
  publish_early(p.out, o);
  count_op(p.ds);
  const long long stride = (long long)gridDim.x * blockDim.x;
  if (p.mode == 2) {
    const long long total = p.outer * p.inner;
    for (long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x; e < total; e += stride) {
      const long long i = e % p.inner, ob = e / p.inner;
      const T* src = a + ob * p.A * p.inner + i;
      T acc = (T)0;
      for (long long j = 0; j < p.A; ++j) acc = acc + src[j * p.inner];
      o[e] = acc + (T)0;
    }
  } else {
    const long long L = p.mode == 0 ? p.length : p.A + p.A2;
    const long long total = p.outer * L * p.inner;
    for (long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x; e < total; e += stride) {
      const long long i = e % p.inner, t = e / p.inner, j = t % L, ob = t / L;
      if (p.mode == 0) o[e] = a[(ob * p.A + p.start + j) * p.inner + i];
      else o[e] = j < p.A ? a[(ob * p.A + j) * p.inner + i] : b[(ob * p.A2 + j - p.A) * p.inner + i];
    }
  }
  publish_late(p.out, o);
}

}  // namespace coex
