// kernels.cuh -- sm_100a device code of the B200 symbolic-execution backend.
//
// Every compute kernel serves both execution paths:
//   * eager (coex_exec_op: imperative / tracing / replay steps) -- operands are
//     passed as direct device pointers;
//   * graph (one CUDA Graph per SymProgram specialisation) -- operands are read
//     through *cells*: device words holding the pointer of the latest execution
//     of the producing node (phi semantics for branch merges / loop-carried
//     values).
// Reference semantics (float64, pinned orders) are in pkg/src/coex/tensor.py;
// each kernel cites the lines it reproduces.
#pragma once
#include <cuda_runtime.h>
#include <cuda_bf16.h>
#include <stdint.h>

namespace coex {

// Programmatic dependent launch: every kernel of a pass graph is linked to its predecessor by a
// programmatic edge (runtime.cu add_kernel), so it is scheduled while the predecessor's last
// wave drains; it waits here until the predecessor grid has completed and its writes are
// visible, then lets its own successor launch early.  Outside PDL both are no-ops.
#define COEX_PDL_ENTER()                                        \
  do {                                                          \
    asm volatile("griddepcontrol.wait;" ::: "memory");          \
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); \
  } while (0)

constexpr int kMaxRank = 8;
constexpr int kMaxDevVars = 1024;   // variables per context (runtime.cu kMaxVars)
constexpr int kMaxPub = 6;

// ------------------------------------------------------------------ pass state
// One per context, in device memory.  Reset by k_pass_begin.
struct DevState {
  int cancelled;                  // spinners stop, conditionals skip, no commit
  int status;                     // coex_status of a device-detected failure
  unsigned long long pass_id;
  long long dec_head;             // decisions consumed this pass
  long long feed_head;            // feeds consumed this pass
  long long fetch_head;           // fetch entries published this pass
  unsigned long long fetch_bytes; // fetch payload arena bump pointer
  unsigned long long stall_ns;    // time spent spinning on the host
  long long ops;                  // compute kernels executed (not skipped)
  unsigned long long t_begin;
  unsigned long long* trace;      // optional per-kernel stamps: (globaltimer, kind) pairs
  int trace_cap;
  int trace_n;
};

// Kernel kinds recorded by stamp() (profiling: share of each kernel kind in a pass).
enum StampKind {
  SK_BEGIN = 0, SK_EW = 1, SK_REDUCE = 2, SK_TRANSPOSE = 3, SK_MATMUL = 4, SK_PTR = 5, SK_DECIDE = 6,
  SK_FEED_WAIT = 7, SK_FEED_FILL = 8, SK_FETCH = 9, SK_GATE = 10, SK_COMMIT = 11, SK_END = 12,
  SK_AFTER_WAIT = 64, SK_FUSED = 13, SK_IM2COL = 14, SK_COL2IM = 15, SK_CVT = 16, SK_COLSTATS = 17,
  SK_BNAPPLY = 18, SK_SPLITK = 19, SK_SOFTMAX = 20, SK_SOFTMAX_GRAD = 21, SK_CE = 22, SK_BIAS = 23, SK_LN = 24,
  SK_EMBED = 25, SK_COLSUM = 26, SK_SKEW = 27, SK_POOL = 28, SK_AXIS = 29, SK_GUARD = 30, SK_ATTN = 31,
  SK_ATTN_DELTA = 32, SK_ATTN_KV = 33, SK_ATTN_Q = 34, SK_NVLS = 35
};

// Host <-> device rings in pinned, mapped host memory.
constexpr int kDecCap = 1024;
constexpr int kFeedCap = 1024;
constexpr int kFetchCap = 4096;

struct DecEntry {
  volatile unsigned long long seq;
  long long id;
  int kind;     // 0 = case, 1 = loop
  int value;    // case index / continue flag
};

enum FeedType { FEED_SCALAR = 0, FEED_HOST = 1, FEED_SYNTH = 2, FEED_DEVICE = 3, FEED_MAPPED = 4 };

struct FeedEntry {
  volatile unsigned long long seq;
  long long slot;
  int type;
  int ndim;
  long long shape[kMaxRank];
  unsigned long long state;    // FEED_SYNTH generator state
  double scalar;               // FEED_SCALAR value
  unsigned long long off;      // FEED_HOST payload offset in the feed arena (doubles)
  const void* dptr;            // FEED_DEVICE pointer (context precision) / FEED_MAPPED host f64 payload
};

struct FetchEntry {
  volatile unsigned long long seq;
  long long node;
  unsigned long long off;      // payload offset (bytes) in the fetch arena
  long long numel;
  int ndim;
  int pad;
  long long shape[kMaxRank];
};

struct Mailbox {
  volatile unsigned long long pass_id;   // host: set before launch
  volatile unsigned long long cancel;    // host: = pass_id to cancel
  volatile unsigned long long done;      // device: = pass_id when the pass ended
  volatile int status;
  volatile int committed;
  volatile long long dec_consumed;
  volatile long long feed_consumed;
  volatile unsigned long long exec_ns;
  volatile unsigned long long stall_ns;
  volatile long long ops;
  volatile long long fetches;
  volatile unsigned long long dirty_mask;        // first 64 variables (coex_pass_stats)
  volatile unsigned long long dirty[kMaxDevVars / 64];   // every variable committed by the pass
  volatile int var_shape_id[kMaxDevVars];
  DecEntry dec[kDecCap];
  FeedEntry feed[kFeedCap];
  FetchEntry fetch[kFetchCap];
};

__device__ __forceinline__ unsigned long long ld_acquire_sys(const volatile unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release_sys(volatile unsigned long long* p, unsigned long long v) {
  asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ unsigned long long globaltimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

__device__ __forceinline__ void stamp(DevState* ds, int kind) {
  if (ds != nullptr && blockIdx.x == 0 && threadIdx.x == 0 && threadIdx.y == 0 && ds->trace != nullptr) {
    int i = ds->trace_n;
    if (i < ds->trace_cap) {
      ds->trace[2 * i] = globaltimer();
      ds->trace[2 * i + 1] = (unsigned long long)kind;
      ds->trace_n = i + 1;
    }
  }
}

__host__ __device__ __forceinline__ unsigned long long seq_of(unsigned long long pass_id, long long idx) {
  return (pass_id << 24) + (unsigned long long)idx + 1ull;
}

// ------------------------------------------------------------------ operands
struct In {
  const void* direct;
  void* const* cell;
  void* const* ovl;      // variable operand: overlay slot (set by an in-pass AssignVar) read first
};
template <typename T>
__device__ __forceinline__ const T* res(const In& x) {
  if (x.ovl != nullptr) {
    const void* o = *x.ovl;
    if (o != nullptr) return (const T*)o;
  }
  return (const T*)(x.cell ? *x.cell : x.direct);
}

struct Out {
  void* buf[2];          // buf[1] used only when pingpong
  int pingpong;          // node may read its own previous output
  int npub;
  void** pub[kMaxPub];   // cells that receive the chosen output pointer
  unsigned int* late;    // non-null: publish from the last block (node reads a cell it publishes)
};

template <typename T>
__device__ __forceinline__ T* pick_out(const Out& o, const void* a, const void* b) {
  if (!o.pingpong) return (T*)o.buf[0];
  return (T*)((a == o.buf[0] || b == o.buf[0]) ? o.buf[1] : o.buf[0]);
}

// Early publication: block 0 / thread 0, before compute (safe when no block reads a published cell).
__device__ __forceinline__ void publish_early(const Out& o, void* out) {
  if (o.late == nullptr && blockIdx.x == 0 && threadIdx.x == 0)
    for (int i = 0; i < o.npub; ++i) *o.pub[i] = out;
}
// Late publication: the last block to finish writes the cells.
__device__ __forceinline__ void publish_late(const Out& o, void* out) {
  if (o.late == nullptr) return;
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    unsigned int prev = atomicAdd(o.late, 1u);
    if (prev == gridDim.x * gridDim.y * gridDim.z - 1) {
      for (int i = 0; i < o.npub; ++i) *o.pub[i] = out;
      *o.late = 0u;
    }
  }
}

// Cancellation ("after cancel the pass stops within one kernel execution"):
// the spinners (decisions, feeds, fetches) stop waiting, conditional nodes then run no body,
// the commit is skipped and AssignVar leaves the overlay alone (k_ptr and the feed kernels
// test the flag).  Compute kernels do not test it themselves (a dependent flag load at every
// launch cost ~5 % of the C2 step); instead the builder cuts every straight-line list into
// guarded segments: a one-thread k_guard reads the host's cancel word and sets an IF
// conditional whose body is the next segment (COEX_CANCEL_EVERY kernels, default 64), so a
// cancelled pass skips every later segment and runs at most the one in flight.  Cells start
// each pass at their build-time values (a buffer of the right size, or the program's
// zero-filled spare buffer of the largest size), so any prefix of kernels reads valid memory.
__device__ __forceinline__ bool skip(const DevState* ds) {
  return ds != nullptr && *(volatile const int*)&ds->cancelled;
}
__device__ __forceinline__ void count_op(DevState* ds) {
  if (ds != nullptr && blockIdx.x == 0 && threadIdx.x == 0) ds->ops += 1;
}

// ------------------------------------------------------------------ elementwise
// ADD/SUB/MUL with rank-0 broadcast (tensor.py:121-128, 261-263); NEG/RELU/SIGMOID (tensor.py:264-270).
// Extension elementwise ops (configs C2-C5, oracle/kernels.py ext_kernel): TANH, LEAKY_RELU
// (slope 0.2), RELU_GRAD(x, dy), LEAKY_RELU_GRAD(x, dy), BCE_TERM(x, t).
enum EwOp { EW_ADD = 0, EW_SUB = 1, EW_MUL = 2, EW_NEG = 3, EW_RELU = 4, EW_SIGMOID = 5, EW_COPY = 6,
            EW_TANH = 7, EW_LRELU = 8, EW_RELU_GRAD = 9, EW_LRELU_GRAD = 10, EW_BCE = 11,
            EW_TO_INDEX = 12, EW_GELU_GRAD = 13, EW_GELU = 14, EW_SQRT = 15, EW_DIV = 16 };
constexpr double kGeluK = 0.7978845608028654;   // sqrt(2/pi)
constexpr double kLeakySlope = 0.2;

__host__ __device__ __forceinline__ bool ew_binary(int op) {
  return op <= EW_MUL || (op >= EW_RELU_GRAD && op <= EW_GELU_GRAD) || op == EW_DIV;
}

__device__ __forceinline__ double ew_apply(int op, double a, double b) {
  switch (op) {
    case EW_ADD: return __dadd_rn(a, b);
    case EW_SUB: return __dsub_rn(a, b);
    case EW_MUL: return __dmul_rn(a, b);
    case EW_NEG: return -a;
    case EW_RELU: return (a > 0.0 || a != a) ? a : 0.0;        // np.maximum(x, 0): NaN kept, -0 -> +0
    case EW_SIGMOID: return __ddiv_rn(1.0, __dadd_rn(1.0, exp(-a)));
    case EW_TANH: return tanh(a);
    case EW_LRELU: return a > 0.0 ? a : __dmul_rn(a, kLeakySlope);
    case EW_RELU_GRAD: return a > 0.0 ? b : 0.0;
    case EW_LRELU_GRAD: return a > 0.0 ? b : __dmul_rn(b, kLeakySlope);
    case EW_BCE: return __dadd_rn(__dsub_rn(a > 0.0 ? a : 0.0, __dmul_rn(a, b)), log1p(exp(-fabs(a))));
    case EW_TO_INDEX: {
      const double v = floor((a + 1.0) * 0.5 * b);
      return v < 0.0 ? 0.0 : (v > b - 1.0 ? b - 1.0 : v);
    }
    case EW_GELU: return 0.5 * a * (1.0 + tanh(kGeluK * (a + 0.044715 * a * a * a)));
    case EW_GELU_GRAD: {
      const double t = tanh(kGeluK * (a + 0.044715 * a * a * a));
      return b * (0.5 * (1.0 + t) + 0.5 * a * (1.0 - t * t) * kGeluK * (1.0 + 3.0 * 0.044715 * a * a));
    }
    case EW_SQRT: return __dsqrt_rn(a);
    case EW_DIV: return __ddiv_rn(a, b);
    default: return a;
  }
}
__device__ __forceinline__ float ew_apply(int op, float a, float b) {
  switch (op) {
    case EW_ADD: return __fadd_rn(a, b);
    case EW_SUB: return __fsub_rn(a, b);
    case EW_MUL: return __fmul_rn(a, b);
    case EW_NEG: return -a;
    case EW_RELU: return (a > 0.0f || a != a) ? a : 0.0f;
    case EW_SIGMOID: return __fdiv_rn(1.0f, __fadd_rn(1.0f, expf(-a)));
    case EW_TANH: return tanhf(a);
    case EW_LRELU: return a > 0.0f ? a : __fmul_rn(a, (float)kLeakySlope);
    case EW_RELU_GRAD: return a > 0.0f ? b : 0.0f;
    case EW_LRELU_GRAD: return a > 0.0f ? b : __fmul_rn(b, (float)kLeakySlope);
    case EW_BCE: return __fadd_rn(__fsub_rn(a > 0.0f ? a : 0.0f, __fmul_rn(a, b)), log1pf(expf(-fabsf(a))));
    case EW_TO_INDEX: {
      const float v = floorf((a + 1.0f) * 0.5f * b);
      return v < 0.0f ? 0.0f : (v > b - 1.0f ? b - 1.0f : v);
    }
    case EW_GELU: return 0.5f * a * (1.0f + tanhf((float)kGeluK * (a + 0.044715f * a * a * a)));
    case EW_GELU_GRAD: {
      const float t = tanhf((float)kGeluK * (a + 0.044715f * a * a * a));
      return b * (0.5f * (1.0f + t) + 0.5f * a * (1.0f - t * t) * (float)kGeluK * (1.0f + 3.0f * 0.044715f * a * a));
    }
    case EW_SQRT: return __fsqrt_rn(a);
    case EW_DIV: return __fdiv_rn(a, b);
    default: return a;
  }
}

struct EwParams {
  DevState* ds;
  In a, b;
  int op;
  int a_scalar, b_scalar;   // broadcast rank-0 operand
  long long n;
  Out out;
  __nv_bfloat16* shadow;    // bf16 mode: also write the bf16 copy later GEMMs read (GELU / GELU_GRAD)
  int skip_f32;             // the fp32 output has no reader (only GEMMs, through the shadow)
};

// fp32 float4 body with the op fixed at compile time (no per-element dispatch)
template <int OP>
__device__ __forceinline__ void ew_body4(const EwParams& p, const float* a, const float* b, float* o, float as,
                                         float bs, long long n4, long long stride) {
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n4; i += stride) {
    const float4 x4 = p.a_scalar ? make_float4(as, as, as, as) : ((const float4*)a)[i];
    float4 y4 = make_float4(bs, bs, bs, bs);
    if (b != nullptr && !p.b_scalar) y4 = ((const float4*)b)[i];
    float4 r;
    r.x = ew_apply(OP, x4.x, y4.x);
    r.y = ew_apply(OP, x4.y, y4.y);
    r.z = ew_apply(OP, x4.z, y4.z);
    r.w = ew_apply(OP, x4.w, y4.w);
    if (!p.skip_f32) ((float4*)o)[i] = r;
    if (p.shadow) {
      __nv_bfloat162 h0 = __floats2bfloat162_rn(r.x, r.y), h1 = __floats2bfloat162_rn(r.z, r.w);
      ((uint2*)p.shadow)[i] = make_uint2(*(uint32_t*)&h0, *(uint32_t*)&h1);
    }
  }
}

template <typename T>
__global__ void __launch_bounds__(256) k_elementwise(EwParams p) {
  COEX_PDL_ENTER();
  stamp(p.ds, SK_EW);
  const T* a = res<T>(p.a);
  const T* b = ew_binary(p.op) ? res<T>(p.b) : nullptr;
  T* o = pick_out<T>(p.out, a, b);
  publish_early(p.out, o);
  count_op(p.ds);
  const long long n = p.n;
  const long long stride = (long long)gridDim.x * blockDim.x;
  const T as = p.a_scalar ? a[0] : T(0);
  const T bs = (b != nullptr && p.b_scalar) ? b[0] : T(0);
  if constexpr (sizeof(T) == 4) {
    // float4 path: four independent elements per thread (same per-element rounding)
    const bool va = p.a_scalar || (((uintptr_t)a & 15) == 0);
    const bool vb = b == nullptr || p.b_scalar || (((uintptr_t)b & 15) == 0);
    if ((n & 3) == 0 && va && vb && (((uintptr_t)o & 15) == 0)) {
      const float* af = (const float*)a;
      const float* bf = (const float*)b;
      float* of = (float*)o;
      bool done = true;
      switch (p.op) {                                // hot ops: op-specialised loops
        case EW_ADD: ew_body4<EW_ADD>(p, af, bf, of, (float)as, (float)bs, n / 4, stride); break;
        case EW_SUB: ew_body4<EW_SUB>(p, af, bf, of, (float)as, (float)bs, n / 4, stride); break;
        case EW_MUL: ew_body4<EW_MUL>(p, af, bf, of, (float)as, (float)bs, n / 4, stride); break;
        case EW_GELU: ew_body4<EW_GELU>(p, af, bf, of, (float)as, (float)bs, n / 4, stride); break;
        case EW_GELU_GRAD: ew_body4<EW_GELU_GRAD>(p, af, bf, of, (float)as, (float)bs, n / 4, stride); break;
        default: done = false;
      }
      if (done) {
        publish_late(p.out, o);
        return;
      }
      for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n / 4; i += stride) {
        const float4 x4 = p.a_scalar ? make_float4(as, as, as, as) : ((const float4*)a)[i];
        float4 y4 = make_float4(bs, bs, bs, bs);
        if (b != nullptr && !p.b_scalar) y4 = ((const float4*)b)[i];
        float4 r;
        r.x = ew_apply(p.op, x4.x, y4.x);
        r.y = ew_apply(p.op, x4.y, y4.y);
        r.z = ew_apply(p.op, x4.z, y4.z);
        r.w = ew_apply(p.op, x4.w, y4.w);
        if (!p.skip_f32) ((float4*)o)[i] = r;
        if (p.shadow) {
          __nv_bfloat162 h0 = __floats2bfloat162_rn(r.x, r.y), h1 = __floats2bfloat162_rn(r.z, r.w);
          ((uint2*)p.shadow)[i] = make_uint2(*(uint32_t*)&h0, *(uint32_t*)&h1);
        }
      }
      publish_late(p.out, o);
      return;
    }
  }
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
    T x = p.a_scalar ? as : a[i];
    T y = (b == nullptr) ? T(0) : (p.b_scalar ? bs : b[i]);
    const T v = ew_apply(p.op, x, y);
    if (!p.skip_f32) o[i] = v;
    if (p.shadow) p.shadow[i] = __float2bfloat16_rn((float)v);
  }
  publish_late(p.out, o);
}

// ------------------------------------------------------------------ reductions
// SUM / MEAN (tensor.py:239-243, 271-277): sequential row-major sum from +0.0.
struct ReduceParams {
  DevState* ds;
  In a;
  long long n;
  int mean;
  Out out;
  double* part;              // k_reduce_multi: per-block partials (context scratch)
  unsigned int* counter;     // k_reduce_multi: last-block election
};

// Parity path: one warp streams the data, lane 0 accumulates strictly in order.
template <typename T>
__global__ void __launch_bounds__(32) k_reduce_seq(ReduceParams p) {
  COEX_PDL_ENTER();
  stamp(p.ds, SK_REDUCE);
  const T* a = res<T>(p.a);
  T* o = pick_out<T>(p.out, a, nullptr);
  publish_early(p.out, o);
  count_op(p.ds);
  const int lane = threadIdx.x;
  double acc = 0.0;
  for (long long base = 0; base < p.n; base += 32) {
    long long i = base + lane;
    double v = (i < p.n) ? (double)a[i] : 0.0;
    int cnt = (int)min(32ll, p.n - base);
    for (int j = 0; j < cnt; ++j) {
      double x = __shfl_sync(0xffffffffu, v, j);
      acc = __dadd_rn(acc, x);
    }
  }
  if (lane == 0) o[0] = (T)(p.mean ? __ddiv_rn(acc, (double)p.n) : acc);
  publish_late(p.out, o);
}

// Tolerance path, large inputs: every block sums a contiguous chunk in double (16-byte loads
// when aligned) into part[block]; the last block to finish adds the partials in block order
// (deterministic for a given grid) and re-arms the counter.  The context owns part / counter
// (kernels of one context run in stream order; PDL dependents wait for the grid).
constexpr int kReduceMaxBlocks = 1024;
template <typename T>
__global__ void __launch_bounds__(256) k_reduce_multi(ReduceParams p) {
  COEX_PDL_ENTER();
  stamp(p.ds, SK_REDUCE);
  const T* a = res<T>(p.a);
  T* o = pick_out<T>(p.out, a, nullptr);
  publish_early(p.out, o);
  count_op(p.ds);
  __shared__ double red[8];
  __shared__ unsigned int last;
  const long long lo = p.n * blockIdx.x / gridDim.x, hi = p.n * (blockIdx.x + 1) / gridDim.x;
  double acc = 0.0;
  long long i = lo + threadIdx.x;
  if constexpr (sizeof(T) == 4) {
    const long long a0 = (lo + 3) & ~3ll, a1 = hi & ~3ll;      // 16-byte aligned body (a is)
    if (((uintptr_t)a & 15) == 0 && a1 > a0) {
      for (long long j = lo + threadIdx.x; j < a0; j += blockDim.x) acc += (double)a[j];
      const float4* a4 = (const float4*)(a + a0);
      const long long n4 = (a1 - a0) / 4;
      for (long long q = threadIdx.x; q < n4; q += blockDim.x) {
        const float4 v = __ldcs(a4 + q);
        acc += ((double)v.x + (double)v.y) + ((double)v.z + (double)v.w);
      }
      i = a1 + threadIdx.x;
    }
  }
  for (; i < hi; i += blockDim.x) acc += (double)a[i];
  for (int s = 16; s > 0; s >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, s);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = acc;
  __syncthreads();
  if (threadIdx.x == 0) {
    double b = 0.0;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) b += red[w];
    p.part[blockIdx.x] = b;
    __threadfence();
    last = atomicAdd(p.counter, 1u) == gridDim.x - 1 ? 1u : 0u;
    if (last) {
      __threadfence();
      double s = 0.0;
      for (unsigned int k = 0; k < gridDim.x; ++k) s += __ldcg(p.part + k);
      o[0] = (T)(p.mean ? s / (double)p.n : s);
      *p.counter = 0u;
    }
  }
  __syncthreads();
  if (last) publish_late(p.out, o);
}

// Tolerance path (fp32 / bf16 contexts): warp-shuffle tree in double, one block.
template <typename T>
__global__ void __launch_bounds__(1024) k_reduce_tree(ReduceParams p) {
  COEX_PDL_ENTER();
  stamp(p.ds, SK_REDUCE);
  const T* a = res<T>(p.a);
  T* o = pick_out<T>(p.out, a, nullptr);
  publish_early(p.out, o);
  count_op(p.ds);
  __shared__ double part[32];
  double acc = 0.0;
  for (long long i = threadIdx.x; i < p.n; i += blockDim.x) acc += (double)a[i];
  for (int s = 16; s > 0; s >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, s);
  if ((threadIdx.x & 31) == 0) part[threadIdx.x >> 5] = acc;
  __syncthreads();
  if (threadIdx.x < 32) {
    double v = (threadIdx.x < (blockDim.x >> 5)) ? part[threadIdx.x] : 0.0;
    for (int s = 16; s > 0; s >>= 1) v += __shfl_xor_sync(0xffffffffu, v, s);
    if (threadIdx.x == 0) o[0] = (T)(p.mean ? v / (double)p.n : v);
  }
  publish_late(p.out, o);
}

// ------------------------------------------------------------------ transpose
// TRANSPOSE (tensor.py:156-161, 278-279): out[o] = in[sum idx_d * in_stride[perm[d]]], materialised.
struct TransposeParams {
  DevState* ds;
  In a;
  int rank;
  long long n;
  long long out_shape[kMaxRank];
  long long src_stride[kMaxRank];   // input stride of the axis that out-dim d reads
  Out out;
};

template <typename T>
__global__ void __launch_bounds__(256) k_transpose(TransposeParams p) {
  COEX_PDL_ENTER();
  stamp(p.ds, SK_TRANSPOSE);
  const T* a = res<T>(p.a);
  T* o = pick_out<T>(p.out, a, nullptr);
  publish_early(p.out, o);
  count_op(p.ds);
  const long long stride = (long long)gridDim.x * blockDim.x;
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < p.n; i += stride) {
    long long rem = i, src = 0;
    for (int d = p.rank - 1; d >= 0; --d) {
      long long q = rem / p.out_shape[d];
      long long r = rem - q * p.out_shape[d];
      src += r * p.src_stride[d];
      rem = q;
    }
    o[i] = a[src];
  }
  publish_late(p.out, o);
}

// Transpose that keeps the innermost axis (e.g. the attention head split [B,T,H,hd] ->
// [B,H,T,hd]): whole rows of `inner` contiguous elements move, 16-byte vectors per thread,
// 32-bit index arithmetic per row (rank <= 4 outer axes).
template <typename T>
__global__ void __launch_bounds__(256) k_transpose_rows(TransposeParams p) {
  COEX_PDL_ENTER();
  stamp(p.ds, SK_TRANSPOSE);
  const T* a = res<T>(p.a);
  T* o = pick_out<T>(p.out, a, nullptr);
  publish_early(p.out, o);
  count_op(p.ds);
  constexpr int V = 16 / sizeof(T);
  const long long inner = p.out_shape[p.rank - 1];
  const long long vpr = inner / V;                 // vectors per row
  const long long rows = p.n / inner;
  const long long stride = (long long)gridDim.x * blockDim.x;
  if (rows * vpr < (1ll << 31) && p.n < (1ll << 31)) {
    // 32-bit index arithmetic (the 64-bit div / mod chain per 16 bytes made the copy
    // instruction-bound: C5 head splits at ~40 % of HBM)
    const unsigned total = (unsigned)(rows * vpr), uv = (unsigned)vpr, uin = (unsigned)inner;
    for (unsigned u = blockIdx.x * blockDim.x + threadIdx.x; u < total; u += (unsigned)stride) {
      const unsigned r = u / uv, e = (u - r * uv) * V;
      unsigned rem = r, src = 0;
      for (int d = p.rank - 2; d >= 0; --d) {
        const unsigned sd = (unsigned)p.out_shape[d];
        const unsigned q = rem / sd;
        src += (rem - q * sd) * (unsigned)p.src_stride[d];
        rem = q;
      }
      *(uint4*)(o + (size_t)r * uin + e) = *(const uint4*)(a + src + e);
    }
    publish_late(p.out, o);
    return;
  }
  for (long long u = (long long)blockIdx.x * blockDim.x + threadIdx.x; u < rows * vpr; u += stride) {
    const long long r = u / vpr, e = (u - r * vpr) * V;
    long long rem = r, src = 0;
    for (int d = p.rank - 2; d >= 0; --d) {
      const long long idx = rem % p.out_shape[d];
      rem /= p.out_shape[d];
      src += idx * p.src_stride[d];
    }
    *(uint4*)(o + r * inner + e) = *(const uint4*)(a + src + e);
  }
  publish_late(p.out, o);
}

// 2-D transpose through a padded shared-memory tile (coalesced on both sides).
template <typename T>
__global__ void __launch_bounds__(256) k_transpose2d(TransposeParams p) {
  COEX_PDL_ENTER();
  stamp(p.ds, SK_TRANSPOSE);
  const T* a = res<T>(p.a);
  T* o = pick_out<T>(p.out, a, nullptr);
  publish_early(p.out, o);
  count_op(p.ds);
  __shared__ T tile[32][33];
  const long long R = p.out_shape[1], C = p.out_shape[0];   // input is R x C, output C x R
  const long long tiles_c = (C + 31) / 32;
  for (long long t = blockIdx.x; t < ((R + 31) / 32) * tiles_c; t += gridDim.x) {
    long long r0 = (t / tiles_c) * 32, c0 = (t % tiles_c) * 32;
    for (int k = threadIdx.y; k < 32; k += blockDim.y) {
      long long r = r0 + k, c = c0 + threadIdx.x;
      if (r < R && c < C) tile[k][threadIdx.x] = a[r * C + c];
    }
    __syncthreads();
    for (int k = threadIdx.y; k < 32; k += blockDim.y) {
      long long c = c0 + k, r = r0 + threadIdx.x;
      if (r < R && c < C) o[c * R + r] = tile[threadIdx.x][k];
    }
    __syncthreads();
  }
  publish_late(p.out, o);
}

// ------------------------------------------------------------------ matmul
// MATMUL (tensor.py:228-236): out[i,j] = (((+0 + a[i,0]*b[0,j]) + a[i,1]*b[1,j]) + ...),
// every product and every sum rounded separately, k strictly increasing.
// Parity SIMT kernel: a k-panel of A and B is staged in shared memory; each
// thread owns RM x RN outputs and walks k in order -> bitwise equal to the
// reference for any tiling.  ``trans_a``/``trans_b`` read a transposed operand
// in place (TRANSPOSE folded into the consumer).
struct MatmulParams {
  DevState* ds;
  In a, b;
  long long M, N, K;
  int trans_a, trans_b;
  long long lda, ldb;       // row stride of the stored operand
  Out out;
  long long sa, sb, sc;     // batched (blockIdx.y = batch): element strides of A, B, C per batch
};

template <typename T, int BM, int BN, int BK, int RM, int RN, bool EXACT>
__global__ void __launch_bounds__((BM / RM) * (BN / RN)) k_matmul_simt(MatmulParams p) {
  COEX_PDL_ENTER();
  stamp(p.ds, SK_MATMUL);
  const T* A = res<T>(p.a);
  const T* B = res<T>(p.b);
  T* C = pick_out<T>(p.out, A, B);
  publish_early(p.out, C);
  count_op(p.ds);
  constexpr int TX = BN / RN, TY = BM / RM, NT = TX * TY;
  __shared__ T sA[BK][BM + 1];
  __shared__ T sB[BK][BN + 1];
  const int tx = threadIdx.x % TX, ty = threadIdx.x / TX;
  const long long tiles_n = (p.N + BN - 1) / BN;
  const long long tiles = ((p.M + BM - 1) / BM) * tiles_n;
  for (long long tile = blockIdx.x; tile < tiles; tile += gridDim.x) {
    const long long m0 = (tile / tiles_n) * BM, n0 = (tile % tiles_n) * BN;
    T acc[RM][RN];
#pragma unroll
    for (int i = 0; i < RM; ++i)
#pragma unroll
      for (int j = 0; j < RN; ++j) acc[i][j] = T(0);
    for (long long k0 = 0; k0 < p.K; k0 += BK) {
      for (int e = threadIdx.x; e < BM * BK; e += NT) {
        int mm, kk;
        if (p.trans_a) { mm = e % BM; kk = e / BM; } else { kk = e % BK; mm = e / BK; }
        long long gm = m0 + mm, gk = k0 + kk;
        T v = T(0);
        if (gm < p.M && gk < p.K) v = p.trans_a ? A[gk * p.lda + gm] : A[gm * p.lda + gk];
        sA[kk][mm] = v;
      }
      for (int e = threadIdx.x; e < BK * BN; e += NT) {
        int kk, nn;
        if (p.trans_b) { kk = e % BK; nn = e / BK; } else { nn = e % BN; kk = e / BN; }
        long long gk = k0 + kk, gn = n0 + nn;
        T v = T(0);
        if (gk < p.K && gn < p.N) v = p.trans_b ? B[gn * p.ldb + gk] : B[gk * p.ldb + gn];
        sB[kk][nn] = v;
      }
      __syncthreads();
      const int kmax = (int)min((long long)BK, p.K - k0);
      for (int kk = 0; kk < kmax; ++kk) {
        T av[RM], bv[RN];
#pragma unroll
        for (int i = 0; i < RM; ++i) av[i] = sA[kk][ty + i * TY];
#pragma unroll
        for (int j = 0; j < RN; ++j) bv[j] = sB[kk][tx + j * TX];
#pragma unroll
        for (int i = 0; i < RM; ++i)
#pragma unroll
          for (int j = 0; j < RN; ++j) {
            if constexpr (EXACT) {
              acc[i][j] = ew_apply(EW_ADD, acc[i][j], ew_apply(EW_MUL, av[i], bv[j]));
            } else {
              acc[i][j] = fma(av[i], bv[j], acc[i][j]);
            }
          }
      }
      __syncthreads();
    }
#pragma unroll
    for (int i = 0; i < RM; ++i)
#pragma unroll
      for (int j = 0; j < RN; ++j) {
        long long gm = m0 + ty + i * TY, gn = n0 + tx + j * TX;
        if (gm < p.M && gn < p.N) C[gm * p.N + gn] = acc[i][j];
      }
  }
  publish_late(p.out, C);
}

// Pipelined variant: STAGES-deep cp.async ring of k-panels so the global loads
// of panel t+STAGES-1 overlap the (sequential-k) arithmetic on panel t.  Same
// per-output accumulation order as k_matmul_simt -> bitwise identical.
__device__ __forceinline__ void cp_async_el(void* smem, const void* gmem, bool valid, int bytes) {
  unsigned s = (unsigned)__cvta_generic_to_shared(smem);
  int src = valid ? bytes : 0;
  if (bytes == 8)
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;" ::"r"(s), "l"(gmem), "r"(src) : "memory");
  else
    asm volatile("cp.async.ca.shared.global [%0], [%1], 4, %2;" ::"r"(s), "l"(gmem), "r"(src) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory"); }

template <typename T, int BM, int BN, int BK, int RM, int RN, bool EXACT, int STAGES>
__global__ void __launch_bounds__((BM / RM) * (BN / RN)) k_matmul_pipe(MatmulParams p) {
  COEX_PDL_ENTER();
  stamp(p.ds, SK_MATMUL);
  const T* A0 = res<T>(p.a);
  const T* B0 = res<T>(p.b);
  T* C0 = pick_out<T>(p.out, A0, B0);
  publish_early(p.out, C0);
  if (blockIdx.y == 0) count_op(p.ds);
  const T* A = A0 + blockIdx.y * p.sa;
  const T* B = B0 + blockIdx.y * p.sb;
  T* C = C0 + blockIdx.y * p.sc;
  constexpr int TX = BN / RN, TY = BM / RM, NT = TX * TY;
  __shared__ __align__(16) T sA[STAGES][BK][BM + 1];
  __shared__ __align__(16) T sB[STAGES][BK][BN + 1];
  const int tx = threadIdx.x % TX, ty = threadIdx.x / TX;
  const long long tiles_n = (p.N + BN - 1) / BN;
  const long long tiles = ((p.M + BM - 1) / BM) * tiles_n;
  const long long nk = (p.K + BK - 1) / BK;
  const T* zero_src = A != nullptr ? A : B;
  for (long long tile = blockIdx.x; tile < tiles; tile += gridDim.x) {
    const long long m0 = (tile / tiles_n) * BM, n0 = (tile % tiles_n) * BN;
    auto load = [&](int st, long long k0) {
      for (int e = threadIdx.x; e < BM * BK; e += NT) {
        int mm, kk;
        if (p.trans_a) { mm = e % BM; kk = e / BM; } else { kk = e % BK; mm = e / BK; }
        long long gm = m0 + mm, gk = k0 + kk;
        bool ok = gm < p.M && gk < p.K;
        const T* src = ok ? (p.trans_a ? A + gk * p.lda + gm : A + gm * p.lda + gk) : zero_src;
        cp_async_el(&sA[st][kk][mm], src, ok, (int)sizeof(T));
      }
      for (int e = threadIdx.x; e < BK * BN; e += NT) {
        int kk, nn;
        if (p.trans_b) { kk = e % BK; nn = e / BK; } else { nn = e % BN; kk = e / BN; }
        long long gk = k0 + kk, gn = n0 + nn;
        bool ok = gk < p.K && gn < p.N;
        const T* src = ok ? (p.trans_b ? B + gn * p.ldb + gk : B + gk * p.ldb + gn) : zero_src;
        cp_async_el(&sB[st][kk][nn], src, ok, (int)sizeof(T));
      }
      cp_async_commit();
    };
    T acc[RM][RN];
#pragma unroll
    for (int i = 0; i < RM; ++i)
#pragma unroll
      for (int j = 0; j < RN; ++j) acc[i][j] = T(0);
#pragma unroll
    for (int st = 0; st < STAGES - 1; ++st) {
      if (st < nk) load(st, st * BK);
      else cp_async_commit();
    }
    for (long long t = 0; t < nk; ++t) {
      cp_async_wait<STAGES - 2>();
      __syncthreads();
      if (t + STAGES - 1 < nk) load((int)((t + STAGES - 1) % STAGES), (t + STAGES - 1) * BK);
      else cp_async_commit();
      const int st = (int)(t % STAGES);
      const long long k0 = t * BK;
      auto step = [&](int kk) {
        T av[RM], bv[RN];
#pragma unroll
        for (int i = 0; i < RM; ++i) av[i] = sA[st][kk][ty + i * TY];
#pragma unroll
        for (int j = 0; j < RN; ++j) bv[j] = sB[st][kk][tx + j * TX];
#pragma unroll
        for (int i = 0; i < RM; ++i)
#pragma unroll
          for (int j = 0; j < RN; ++j) {
            if constexpr (EXACT) acc[i][j] = ew_apply(EW_ADD, acc[i][j], ew_apply(EW_MUL, av[i], bv[j]));
            else acc[i][j] = fma(av[i], bv[j], acc[i][j]);
          }
      };
      if constexpr (RM == 1 && RN == 1) {
        // One output per thread: form all BK products first (independent, fully
        // pipelined), then add them in k order.  Zero-filled padding contributes
        // +0 products, and the accumulator (started at +0.0) can never be -0.0,
        // so adding them is exact -- same bits as the reference's k loop.
        T prod[BK];
#pragma unroll
        for (int kk = 0; kk < BK; ++kk) {
          if constexpr (EXACT) prod[kk] = ew_apply(EW_MUL, sA[st][kk][ty], sB[st][kk][tx]);
          else prod[kk] = sA[st][kk][ty] * sB[st][kk][tx];
        }
#pragma unroll
        for (int kk = 0; kk < BK; ++kk) {
          if constexpr (EXACT) acc[0][0] = ew_apply(EW_ADD, acc[0][0], prod[kk]);
          else acc[0][0] += prod[kk];
        }
      } else if (k0 + BK <= p.K) {
#pragma unroll
        for (int kk = 0; kk < BK; ++kk) step(kk);
      } else {
        const int kmax = (int)(p.K - k0);
        for (int kk = 0; kk < kmax; ++kk) step(kk);
      }
    }
    cp_async_wait<0>();
    __syncthreads();
#pragma unroll
    for (int i = 0; i < RM; ++i)
#pragma unroll
      for (int j = 0; j < RN; ++j) {
        long long gm = m0 + ty + i * TY, gn = n0 + tx + j * TX;
        if (gm < p.M && gn < p.N) C[gm * p.N + gn] = acc[i][j];
      }
  }
  publish_late(p.out, C0);
}

// Parity SUM / MEAN with shared-memory staging: all threads stream 2048-element
// chunks into a double buffer while thread 0 adds the previous chunk strictly in
// order (unrolled so loads run ahead of the dependent add chain).
template <typename T>
__global__ void __launch_bounds__(256) k_reduce_seq_smem(ReduceParams p) {
  COEX_PDL_ENTER();
  stamp(p.ds, SK_REDUCE);
  constexpr int CH = 2048;
  __shared__ T buf[2][CH];
  const T* a = res<T>(p.a);
  T* o = pick_out<T>(p.out, a, nullptr);
  publish_early(p.out, o);
  count_op(p.ds);
  double acc = 0.0;
  const long long nch = (p.n + CH - 1) / CH;
  for (int i = threadIdx.x; i < CH; i += blockDim.x) buf[0][i] = (i < p.n) ? a[i] : T(0);
  __syncthreads();
  for (long long c = 0; c < nch; ++c) {
    const int cur = (int)(c & 1);
    if (c + 1 < nch) {
      const long long base = (c + 1) * CH;
      for (int i = threadIdx.x; i < CH; i += blockDim.x)
        buf[cur ^ 1][i] = (base + i < p.n) ? a[base + i] : T(0);
    }
    if (threadIdx.x == 0) {
      const int cnt = (int)min((long long)CH, p.n - c * CH);
      int i = 0;
      for (; i + 8 <= cnt; i += 8) {
        double v0 = buf[cur][i], v1 = buf[cur][i + 1], v2 = buf[cur][i + 2], v3 = buf[cur][i + 3];
        double v4 = buf[cur][i + 4], v5 = buf[cur][i + 5], v6 = buf[cur][i + 6], v7 = buf[cur][i + 7];
        acc = __dadd_rn(acc, v0); acc = __dadd_rn(acc, v1); acc = __dadd_rn(acc, v2); acc = __dadd_rn(acc, v3);
        acc = __dadd_rn(acc, v4); acc = __dadd_rn(acc, v5); acc = __dadd_rn(acc, v6); acc = __dadd_rn(acc, v7);
      }
      for (; i < cnt; ++i) acc = __dadd_rn(acc, (double)buf[cur][i]);
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) o[0] = (T)(p.mean ? __ddiv_rn(acc, (double)p.n) : acc);
  publish_late(p.out, o);
}

// ------------------------------------------------------------------ fused chains
// A run of consecutive elementwise ExecOps of one element count, optionally
// closed by SUM / MEAN, executed as ONE kernel: a micro-op program interpreted
// per element over a small register file.  Each op rounds exactly like its
// standalone kernel (ew_apply), and every element is read and written by one
// thread in program order, so fusion is bit-identical to the unfused sequence
// (in-place reuse of a node's buffer is safe element by element).
constexpr int kChainIn = 8, kChainOps = 16, kChainOut = 8, kChainPub = 4, kChainRegs = 16;

struct ChainOp {
  unsigned char op, dst, a, b;   // a, b: < 16 register, >= 16 input (x - 16)
};
struct ChainParams {
  DevState* ds;
  long long n;
  int nin, nops, nout;
  In in[kChainIn];
  unsigned char in_scalar[kChainIn];
  ChainOp ops[kChainOps];
  unsigned char out_reg[kChainOut];
  void* out_buf[kChainOut];
  unsigned char npub[kChainOut];
  void** pub[kChainOut][kChainPub];
  unsigned int* late;            // non-null: publish after every block read its inputs
  int red;                       // 0 = none, 1 = SUM, 2 = MEAN of register red_reg
  int red_reg;
  void* red_buf;
  int red_npub;
  void** red_pub[kChainPub];
};

// The chain program, its operand pointers and every thread's register file live in shared
// memory: the interpreter indexes them dynamically, which on registers / kernel parameters
// would force per-thread local-memory copies.  Register file layout [reg][thread].
template <typename T>
struct ChainSmem {
  ChainOp ops[kChainOps];
  const T* ip[kChainIn];
  T sv[kChainIn];
  unsigned char in_scalar[kChainIn];
  unsigned char out_reg[kChainOut];
  T* out_buf[kChainOut];
  // fp32 update fast path: the program is  t = g * s ; y = w - t  (every parameter's SGD step):
  // axpy = 1, ax_w / ax_g = vector inputs, ax_s = the scalar input; 16-byte aligned, 4 | n
  int axpy, ax_w, ax_g, ax_s;
  T r[kChainRegs][256];
};

template <typename T>
__device__ __forceinline__ void chain_load(const ChainParams& p, ChainSmem<T>& S) {
  if (threadIdx.x == 0) {
#pragma unroll
    for (int k = 0; k < kChainOps; ++k) S.ops[k] = p.ops[k];
#pragma unroll
    for (int k = 0; k < kChainIn; ++k) {
      const T* ptr = k < p.nin ? res<T>(p.in[k]) : nullptr;
      S.ip[k] = ptr;
      S.in_scalar[k] = p.in_scalar[k];
      S.sv[k] = (k < p.nin && p.in_scalar[k]) ? ptr[0] : T(0);
    }
#pragma unroll
    for (int j = 0; j < kChainOut; ++j) {
      S.out_reg[j] = p.out_reg[j];
      S.out_buf[j] = (T*)p.out_buf[j];
    }
    S.axpy = 0;
    if (sizeof(T) == 4 && p.nops == 2 && p.nout == 1 && (p.n & 3) == 0 && p.ops[0].op == EW_MUL &&
        p.ops[1].op == EW_SUB && p.ops[1].b == p.ops[0].dst && p.out_reg[0] == p.ops[1].dst &&
        p.ops[1].a >= kChainRegs && p.ops[0].a >= kChainRegs && p.ops[0].b >= kChainRegs) {
      const int w = p.ops[1].a - kChainRegs, x = p.ops[0].a - kChainRegs, y = p.ops[0].b - kChainRegs;
      const int g = p.in_scalar[x] ? y : x, sc = p.in_scalar[x] ? x : y;
      if (!p.in_scalar[w] && !p.in_scalar[g] && p.in_scalar[sc] && !(((uintptr_t)S.ip[w] | (uintptr_t)S.ip[g] |
                                                                      (uintptr_t)S.out_buf[0]) & 15)) {
        S.axpy = 1;
        S.ax_w = w;
        S.ax_g = g;
        S.ax_s = sc;
      }
    }
  }
  __syncthreads();
}

template <typename T>
__device__ __forceinline__ T chain_src(const ChainSmem<T>& S, int x, long long i) {
  if (x < kChainRegs) return S.r[x][threadIdx.x];
  const int k = x - kChainRegs;
  return S.in_scalar[k] ? S.sv[k] : S.ip[k][i];
}

template <typename T>
__device__ __forceinline__ void chain_eval(const ChainSmem<T>& Sc, int nops, long long i) {
  ChainSmem<T>& S = const_cast<ChainSmem<T>&>(Sc);
  for (int k = 0; k < nops; ++k) {
    const ChainOp o = S.ops[k];
    S.r[o.dst][threadIdx.x] = ew_apply((int)o.op, chain_src(S, o.a, i), ew_binary(o.op) ? chain_src(S, o.b, i) : T(0));
  }
}

__device__ __forceinline__ void chain_publish(const ChainParams& p) {
#pragma unroll
  for (int j = 0; j < kChainOut; ++j)
#pragma unroll
    for (int q = 0; q < kChainPub; ++q)
      if (j < p.nout && q < p.npub[j]) *p.pub[j][q] = p.out_buf[j];
  if (p.red) {
#pragma unroll
    for (int q = 0; q < kChainPub; ++q)
      if (q < p.red_npub) *p.red_pub[q] = p.red_buf;
  }
}

// One chain over blocks [b, b + nb) of the launch (k_chain: the whole grid; k_chain_multi:
// this chain's share of a grid that runs several independent chains).
template <typename T>
__device__ __forceinline__ void chain_run(const ChainParams& p, ChainSmem<T>& S, long long b, long long nb) {
  chain_load(p, S);
  if (p.late == nullptr && b == 0 && threadIdx.x == 0) chain_publish(p);
  const int nops = p.nops, nout = p.nout;
  const long long stride = nb * blockDim.x;
  if (sizeof(T) == 4 && S.axpy) {
    // the SGD update without the interpreter: 16-byte loads / stores, the same two roundings
    // (product, then difference) as the op-by-op program
    const float4* w4 = (const float4*)S.ip[S.ax_w];
    const float4* g4 = (const float4*)S.ip[S.ax_g];
    float4* o4 = (float4*)S.out_buf[0];
    const float sc = (float)S.sv[S.ax_s];
    for (long long i = b * blockDim.x + threadIdx.x; i < p.n / 4; i += stride) {
      const float4 w = w4[i], g = g4[i];
      o4[i] = make_float4(__fsub_rn(w.x, __fmul_rn(g.x, sc)), __fsub_rn(w.y, __fmul_rn(g.y, sc)),
                          __fsub_rn(w.z, __fmul_rn(g.z, sc)), __fsub_rn(w.w, __fmul_rn(g.w, sc)));
    }
  } else {
    for (long long i = b * blockDim.x + threadIdx.x; i < p.n; i += stride) {
      chain_eval(S, nops, i);
      for (int j = 0; j < nout; ++j) S.out_buf[j][i] = S.r[S.out_reg[j]][threadIdx.x];
    }
  }
  if (p.late != nullptr) {
    __syncthreads();
    if (threadIdx.x == 0) {
      __threadfence();
      if (atomicAdd(p.late, 1u) == (unsigned)(nb - 1)) {
        chain_publish(p);
        *p.late = 0u;
      }
    }
  }
}

template <typename T>
__global__ void __launch_bounds__(256) k_chain(ChainParams p) {
  COEX_PDL_ENTER();
  stamp(p.ds, SK_FUSED);
  __shared__ ChainSmem<T> S;
  count_op(p.ds);
  chain_run(p, S, blockIdx.x, gridDim.x);
}

// Several independent elementwise chains in one launch (e.g. every parameter's SGD update
// of a step): block ranges [off[j], off[j+1]) run chain j.  The planner groups only chains
// that neither read what another publishes nor publish late.
constexpr int kMaxMultiChain = 8;
struct MultiChainParams {
  DevState* ds;
  int count;
  int off[kMaxMultiChain + 1];
  ChainParams c[kMaxMultiChain];
};
template <typename T>
__global__ void __launch_bounds__(256) k_chain_multi(const __grid_constant__ MultiChainParams mp) {
  COEX_PDL_ENTER();
  stamp(mp.ds, SK_FUSED);
  __shared__ ChainSmem<T> S;
  count_op(mp.ds);
  int j = 0;
  while (j + 1 < mp.count && (int)blockIdx.x >= mp.off[j + 1]) ++j;
  chain_run(mp.c[j], S, (long long)blockIdx.x - mp.off[j], (long long)(mp.off[j + 1] - mp.off[j]));
}

// Chain closed by SUM / MEAN: one block evaluates the chain in 2048-element
// chunks into shared memory; the parity path (EXACT) adds in row-major order on
// one thread, the tolerance path reduces with warp shuffles in double.
template <typename T, bool EXACT>
__global__ void __launch_bounds__(256) k_chain_reduce(ChainParams p) {
  COEX_PDL_ENTER();
  stamp(p.ds, SK_FUSED);
  constexpr int CH = 1024;
  __shared__ T vals[CH];
  __shared__ double part[8];
  __shared__ ChainSmem<T> S;
  chain_load(p, S);
  count_op(p.ds);
  const int nops = p.nops, nout = p.nout, red_reg = p.red_reg;
  double acc = 0.0;
  for (long long base = 0; base < p.n; base += CH) {
    const int cnt = (int)min((long long)CH, p.n - base);
    for (int t = threadIdx.x; t < cnt; t += blockDim.x) {
      const long long i = base + t;
      chain_eval(S, nops, i);
      for (int j = 0; j < nout; ++j) S.out_buf[j][i] = S.r[S.out_reg[j]][threadIdx.x];
      vals[t] = chain_src(S, red_reg, i);
    }
    __syncthreads();
    if constexpr (EXACT) {
      if (threadIdx.x == 0) {
        int t = 0;
        for (; t + 8 <= cnt; t += 8) {
          double v0 = vals[t], v1 = vals[t + 1], v2 = vals[t + 2], v3 = vals[t + 3];
          double v4 = vals[t + 4], v5 = vals[t + 5], v6 = vals[t + 6], v7 = vals[t + 7];
          acc = __dadd_rn(acc, v0); acc = __dadd_rn(acc, v1); acc = __dadd_rn(acc, v2); acc = __dadd_rn(acc, v3);
          acc = __dadd_rn(acc, v4); acc = __dadd_rn(acc, v5); acc = __dadd_rn(acc, v6); acc = __dadd_rn(acc, v7);
        }
        for (; t < cnt; ++t) acc = __dadd_rn(acc, (double)vals[t]);
      }
    } else {
      double s = 0.0;
      for (int t = threadIdx.x; t < cnt; t += blockDim.x) s += (double)vals[t];
      for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
      if ((threadIdx.x & 31) == 0) part[threadIdx.x >> 5] = s;
      __syncthreads();
      if (threadIdx.x == 0)
        for (int w = 0; w < (int)(blockDim.x >> 5); ++w) acc += part[w];
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    ((T*)p.red_buf)[0] = (T)(p.red == 2 ? __ddiv_rn(acc, (double)p.n) : acc);
    chain_publish(p);     // single block: every input has been read
  }
}

// ------------------------------------------------------------------ fill / copy / pointer ops
struct FillParams {
  DevState* ds;
  double value;
  long long n;
  Out out;
};
template <typename T>
__global__ void __launch_bounds__(256) k_fill(FillParams p) {
  COEX_PDL_ENTER();
  T* o = (T*)p.out.buf[0];
  publish_early(p.out, o);
  const long long stride = (long long)gridDim.x * blockDim.x;
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < p.n; i += stride) o[i] = (T)p.value;
}

// Convert float64 host payload (mapped) into the context precision.
// TO_INDEX(u, V) evaluated in f64 on the fed value itself (oracle: clip(floor((u+1)*0.5*V),
// 0, V-1)).  Index feeds apply it while converting the f64 host / generator value to the
// compute precision: an fp32-rounded u would move floor() across an integer for ~V * 2^-24
// of the draws (C4: a dozen token ids per step).
__device__ __forceinline__ double index_of(double u, double V) {
  const double v = floor(__dmul_rn(__dmul_rn(__dadd_rn(u, 1.0), 0.5), V));
  if (v != v) return v;
  return v < 0.0 ? 0.0 : (v > V - 1.0 ? V - 1.0 : v);
}
__device__ __forceinline__ double feed_value(double u, double iv) { return iv > 0.0 ? index_of(u, iv) : u; }

template <typename T>
__global__ void __launch_bounds__(256) k_from_f64(const double* src, T* dst, long long n, double iv) {
  COEX_PDL_ENTER();
  const long long stride = (long long)gridDim.x * blockDim.x;
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride)
    dst[i] = (T)feed_value(src[i], iv);
}
template <typename T>
__global__ void __launch_bounds__(256) k_to_f64(const T* src, double* dst, long long n) {
  COEX_PDL_ENTER();
  const long long stride = (long long)gridDim.x * blockDim.x;
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) dst[i] = (double)src[i];
}

// Pointer-only ops (RESHAPE view, READ_VAR, ASSIGN_VAR): no data movement.
enum PtrOp { PTR_ALIAS = 0, PTR_READ_VAR = 1, PTR_ASSIGN_VAR = 2 };
struct PtrParams {
  DevState* ds;
  int op;
  In a;
  void** var_cur;      // committed pointer table entry of the variable
  void** var_ovl;      // overlay table entry (null = not assigned this pass)
  int* var_ovl_shape;
  int shape_id;
  Out out;
};
__global__ void k_ptr(PtrParams p) {
  COEX_PDL_ENTER();
  stamp(p.ds, SK_PTR);
  if (skip(p.ds)) return;
  void* v;
  if (p.op == PTR_READ_VAR) {
    v = *p.var_ovl;                            // overlay first, then committed
    if (v == nullptr) v = *p.var_cur;
  } else {
    v = (void*)res<char>(p.a);
    if (p.op == PTR_ASSIGN_VAR) {              // AssignVar writes the overlay
      *p.var_ovl = v;
      *p.var_ovl_shape = p.shape_id;
    }
  }
  for (int i = 0; i < p.out.npub; ++i) *p.out.pub[i] = v;
}

// ------------------------------------------------------------------ synthetic data
// SyntheticDataset.next (dataset.py:44-51): element e = (e-th xorshift64* draw) * 2 - 1.
// Each thread owns a run of kSynthRun consecutive elements; it jumps to the
// run's first state with GF(2) matrices J_j = T^(kSynthRun * 2^j), walks the
// run, and the block stores through shared memory so global writes coalesce.
constexpr int kSynthRun = 32;
constexpr int kSynthThreads = 128;
constexpr int kJumpBits = 40;
// Jump matrices are stored as 4-bit lookup tables: tab[j][nibble][value] =
// J_j applied to (value << 4*nibble); one application = 16 independent loads.
constexpr int kJumpTabWords = 16 * 16;

__device__ __forceinline__ unsigned long long xs_next(unsigned long long x) {
  x ^= x >> 12;
  x ^= x << 25;
  x ^= x >> 27;
  return x;
}
__device__ __forceinline__ double xs_unit_pm1(unsigned long long x) {
  unsigned long long r = (x * 0x2545F4914F6CDD1Dull) >> 11;
  return __dsub_rn(__dmul_rn(__dmul_rn((double)r, 0x1p-53), 2.0), 1.0);
}
__device__ __forceinline__ unsigned long long gf2_apply(const unsigned long long* tab, unsigned long long v) {
  unsigned long long r = 0;
#pragma unroll
  for (int nib = 0; nib < 16; ++nib) r ^= __ldg(tab + nib * 16 + ((v >> (4 * nib)) & 15ull));
  return r;
}
// State at the start of run `run` (each run = kSynthRun draws) from s0.
__device__ __forceinline__ unsigned long long jump_to_run(const unsigned long long* tabs, unsigned long long s,
                                                          long long run) {
  for (int j = 0; j < kJumpBits && (run >> j) != 0; ++j)
    if ((run >> j) & 1) s = gf2_apply(tabs + kJumpTabWords * j, s);
  return s;
}

struct SynthParams {
  DevState* ds;
  const unsigned long long* jump;   // kJumpBits nibble tables (kJumpTabWords each)
  const unsigned long long* state_ptr;  // graph mode: state from the feed record (null = use state)
  unsigned long long state;
  long long n;
  Out out;
  double iv;                        // > 0: index feed, TO_INDEX(u, iv) applied in f64
};

template <typename T>
__global__ void __launch_bounds__(kSynthThreads) k_synth(SynthParams p) {
  COEX_PDL_ENTER();
  if (skip(p.ds)) return;
  T* o = (T*)p.out.buf[0];
  publish_early(p.out, o);
  __shared__ T stage[kSynthThreads * kSynthRun];
  const unsigned long long s0 = p.state_ptr ? *p.state_ptr : p.state;
  const long long per_block = (long long)kSynthThreads * kSynthRun;
  for (long long base = (long long)blockIdx.x * per_block; base < p.n; base += (long long)gridDim.x * per_block) {
    unsigned long long s = jump_to_run(p.jump, s0, base / kSynthRun + threadIdx.x);
#pragma unroll
    for (int i = 0; i < kSynthRun; ++i) {
      s = xs_next(s);
      stage[threadIdx.x * kSynthRun + i] = (T)feed_value(xs_unit_pm1(s), p.iv);
    }
    __syncthreads();
    long long lim = min(per_block, p.n - base);
    for (long long i = threadIdx.x; i < lim; i += kSynthThreads) o[base + i] = stage[i];
    __syncthreads();
  }
}

// ------------------------------------------------------------------ handshake
// Device side of ChannelSet over pinned mapped host rings.

// Spin until the next ring entry is published, the pass is cancelled, or (never) forever.
// Returns false on cancel.  Accumulates spin time as graph stall.
__device__ __forceinline__ bool wait_seq(DevState* ds, const Mailbox* mb, const volatile unsigned long long* seqp,
                                         unsigned long long want) {
  unsigned long long t0 = 0;
  int polls = 0;
  while (ld_acquire_sys(seqp) != want) {
    if (t0 == 0) t0 = globaltimer();
    if (mb->cancel == ds->pass_id) {
      ds->cancelled = 1;
      ds->stall_ns += globaltimer() - t0;
      return false;
    }
    if (++polls > 64) __nanosleep(200);
  }
  if (t0 != 0) ds->stall_ns += globaltimer() - t0;
  return true;
}

struct DecideParams {
  DevState* ds;
  Mailbox* mb;
  cudaGraphConditionalHandle handle;
  long long id;        // expected branch node id / loop id
  int kind;            // 0 = case (SWITCH), 1 = loop (WHILE)
  int skip_value;      // value that runs no body: ncases for SWITCH, 0 for WHILE
};

__global__ void k_decide(DecideParams p) {
  COEX_PDL_ENTER();
  DevState* ds = p.ds;
  stamp(ds, SK_DECIDE);
  if (ds->cancelled) {
    cudaGraphSetConditional(p.handle, (unsigned)p.skip_value);
    return;
  }
  long long idx = ds->dec_head;
  const DecEntry* e = &p.mb->dec[idx % kDecCap];
  if (!wait_seq(ds, p.mb, &e->seq, seq_of(ds->pass_id, idx))) {
    cudaGraphSetConditional(p.handle, (unsigned)p.skip_value);
    return;
  }
  if (e->kind != p.kind || e->id != p.id) {      // DecisionMismatch, fatal
    ds->status = 3;
    ds->cancelled = 1;
    cudaGraphSetConditional(p.handle, (unsigned)p.skip_value);
    return;
  }
  stamp(ds, SK_AFTER_WAIT | SK_DECIDE);
  int v = e->value;
  ds->dec_head = idx + 1;
  p.mb->dec_consumed = idx + 1;
  cudaGraphSetConditional(p.handle, (unsigned)v);
}

// Segment guard: runs the next straight-line segment (an IF body) unless the pass is cancelled.
struct GuardParams {
  DevState* ds;
  Mailbox* mb;
  cudaGraphConditionalHandle handle;
};
__global__ void k_guard(GuardParams p) {
  COEX_PDL_ENTER();
  DevState* ds = p.ds;
  stamp(ds, SK_GUARD);
  if (!ds->cancelled && p.mb->cancel == ds->pass_id) ds->cancelled = 1;
  cudaGraphSetConditional(p.handle, ds->cancelled ? 0u : 1u);
}

// Commit gate: the overlay may only be committed once the skeleton has
// reached StepEnd without diverging.  The host publishes a
// commit token (decision kind 2) from coex_pass_wait; a cancel instead leaves
// the pass uncommitted even when the device already finished every op.
struct GateParams {
  DevState* ds;
  Mailbox* mb;
};
__global__ void k_commit_gate(GateParams p) {
  COEX_PDL_ENTER();
  DevState* ds = p.ds;
  stamp(ds, SK_GATE);
  if (ds->cancelled) return;
  long long idx = ds->dec_head;
  const DecEntry* e = &p.mb->dec[idx % kDecCap];
  if (!wait_seq(ds, p.mb, &e->seq, seq_of(ds->pass_id, idx))) return;
  if (e->kind != 2) {
    ds->status = 3;
    ds->cancelled = 1;
    return;
  }
  stamp(ds, SK_AFTER_WAIT | SK_GATE);
  ds->dec_head = idx + 1;
  p.mb->dec_consumed = idx + 1;
}

// Feed: wait for the slot's next entry; scalar / device-pointer feeds complete here,
// host-payload and synthetic feeds are expanded by the following k_feed_fill.
struct FeedRecord {
  int type;
  unsigned long long state;
  unsigned long long off;
  const void* dptr;
};
struct FeedWaitParams {
  DevState* ds;
  Mailbox* mb;
  long long slot;
  long long numel;       // static element count of the specialisation
  int ndim;
  long long shape[kMaxRank];
  FeedRecord* rec;       // device scratch for k_feed_fill
  void* buf;             // slot buffer
  void** cell;           // slot cell (re-pointed for device-resident feeds)
  int is_f64;
  double iv;             // > 0: index feed (TO_INDEX fused into the feed, see index_of)
};

__global__ void k_feed_wait(FeedWaitParams p) {
  COEX_PDL_ENTER();
  DevState* ds = p.ds;
  stamp(ds, SK_FEED_WAIT);
  if (ds->cancelled) return;
  long long idx = ds->feed_head;
  const FeedEntry* e = &p.mb->feed[idx % kFeedCap];
  if (!wait_seq(ds, p.mb, &e->seq, seq_of(ds->pass_id, idx))) return;
  bool ok = (e->slot == p.slot) && (e->ndim == p.ndim);
  for (int d = 0; ok && d < p.ndim; ++d) ok = (e->shape[d] == p.shape[d]);
  if (!ok) {                      // orchestrator bug or shape miss: cancel (host reports it)
    ds->status = (e->slot == p.slot) ? 9 : 3;
    ds->cancelled = 1;
    return;
  }
  stamp(ds, SK_AFTER_WAIT | SK_FEED_WAIT);
  ds->feed_head = idx + 1;
  p.mb->feed_consumed = idx + 1;
  p.rec->type = e->type;
  p.rec->state = e->state;
  p.rec->off = e->off;
  p.rec->dptr = e->dptr;
  if (e->type == FEED_SCALAR) {
    const double v = feed_value(e->scalar, p.iv);
    if (p.is_f64) *(double*)p.buf = v; else *(float*)p.buf = (float)v;
    *p.cell = p.buf;
  } else if (e->type == FEED_DEVICE && p.iv > 0.0) {
    *p.cell = p.buf;               // k_feed_fill converts the device tensor into indices
  } else if (e->type == FEED_DEVICE) {
    *p.cell = (void*)e->dptr;      // bind by pointer, no copy
  } else {
    *p.cell = p.buf;
  }
}

struct FeedFillParams {
  DevState* ds;
  const FeedRecord* rec;
  const double* arena;   // mapped host feed payload arena
  const unsigned long long* jump;
  long long n;
  void* buf;
  double iv;             // > 0: index feed
};

template <typename T>
__global__ void __launch_bounds__(kSynthThreads) k_feed_fill(FeedFillParams p) {
  COEX_PDL_ENTER();
  stamp(p.ds, SK_FEED_FILL);
  if (skip(p.ds)) return;
  const int type = p.rec->type;
  T* o = (T*)p.buf;
  if (type == FEED_HOST || type == FEED_MAPPED) {
    // FEED_HOST: the staged payload in the mapped feed arena; FEED_MAPPED: the caller's own
    // registered host buffer, read in place (one bus crossing, no host staging copy)
    const double* src = type == FEED_HOST ? p.arena + p.rec->off : (const double*)p.rec->dptr;
    const long long stride = (long long)gridDim.x * blockDim.x;
    if ((((uintptr_t)src) & 15) == 0) {
      const long long n2 = p.n / 2;
      for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n2; i += stride) {
        const double2 v = ((const double2*)src)[i];
        o[2 * i] = (T)feed_value(v.x, p.iv);
        o[2 * i + 1] = (T)feed_value(v.y, p.iv);
      }
      if (blockIdx.x == 0 && threadIdx.x == 0 && (p.n & 1)) o[p.n - 1] = (T)feed_value(src[p.n - 1], p.iv);
    } else {
      for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < p.n; i += stride)
        o[i] = (T)feed_value(src[i], p.iv);
    }
  } else if (type == FEED_DEVICE && p.iv > 0.0) {
    // a device-resident tensor fed into an index slot: its values are already in the compute
    // precision, the transform runs on them (what the unfused TO_INDEX kernel would do)
    const T* src = (const T*)p.rec->dptr;
    const long long stride = (long long)gridDim.x * blockDim.x;
    for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < p.n; i += stride)
      o[i] = (T)ew_apply(EW_TO_INDEX, src[i], (T)p.iv);
  } else if (type == FEED_SYNTH) {
    __shared__ T stage[kSynthThreads * kSynthRun];
    const unsigned long long s0 = p.rec->state;
    const long long per_block = (long long)kSynthThreads * kSynthRun;
    for (long long base = (long long)blockIdx.x * per_block; base < p.n; base += (long long)gridDim.x * per_block) {
      unsigned long long s = jump_to_run(p.jump, s0, base / kSynthRun + threadIdx.x);
#pragma unroll
      for (int i = 0; i < kSynthRun; ++i) {
        s = xs_next(s);
        stage[threadIdx.x * kSynthRun + i] = (T)feed_value(xs_unit_pm1(s), p.iv);
      }
      __syncthreads();
      long long lim = min(per_block, p.n - base);
      for (long long i = threadIdx.x; i < lim; i += kSynthThreads) o[base + i] = stage[i];
      __syncthreads();
    }
  }
}

// Fetch: copy the node's latest output into the mapped fetch arena, then publish.
struct FetchParams {
  DevState* ds;
  Mailbox* mb;
  In a;
  long long node;
  long long numel;
  int ndim;
  long long shape[kMaxRank];
  char* arena;                 // mapped host fetch payload arena (device view)
  unsigned long long arena_cap;
  int elsize;
};

__global__ void __launch_bounds__(256) k_fetch(FetchParams p) {
  COEX_PDL_ENTER();
  DevState* ds = p.ds;
  stamp(ds, SK_FETCH);
  if (ds->cancelled) return;
  __shared__ unsigned long long off;
  __shared__ long long idx;
  const char* src = res<char>(p.a);
  const unsigned long long bytes = (unsigned long long)p.numel * p.elsize;
  if (threadIdx.x == 0) {
    idx = ds->fetch_head;
    off = (ds->fetch_bytes + 15ull) & ~15ull;
    if (off + bytes > p.arena_cap) off = 0;     // ring wrap (host copies payloads out promptly)
    ds->fetch_bytes = off + bytes;
    ds->fetch_head = idx + 1;
  }
  __syncthreads();
  // 16-byte vector copy when possible
  if ((bytes & 15ull) == 0 && (((uintptr_t)src) & 15) == 0) {
    const uint4* s4 = (const uint4*)src;
    uint4* d4 = (uint4*)(p.arena + off);
    for (unsigned long long i = threadIdx.x; i < bytes / 16; i += blockDim.x) d4[i] = s4[i];
  } else {
    for (unsigned long long i = threadIdx.x; i < bytes; i += blockDim.x) p.arena[off + i] = src[i];
  }
  __threadfence_system();
  __syncthreads();
  if (threadIdx.x == 0) {
    FetchEntry* e = &p.mb->fetch[idx % kFetchCap];
    e->node = p.node;
    e->off = off;
    e->numel = p.numel;
    e->ndim = p.ndim;
    for (int d = 0; d < p.ndim; ++d) e->shape[d] = p.shape[d];
    __threadfence_system();
    st_release_sys(&e->seq, seq_of(ds->pass_id, idx));
  }
}

// Pass begin / end (+ commit of the overlay into the variable store).
struct BeginParams {
  DevState* ds;
  Mailbox* mb;
  void** var_ovl;
  int nvars;
  void** cells;              // the program's pointer cells, reset to their build-time
  void* const* cells_init;   // values (every one a valid buffer) at the start of each pass
  long long ncells;
};
__global__ void k_pass_begin(BeginParams p) {
  COEX_PDL_ENTER();
  DevState* ds = p.ds;
  for (int i = threadIdx.x; i < p.nvars; i += blockDim.x) p.var_ovl[i] = nullptr;
  for (long long i = threadIdx.x; i < p.ncells; i += blockDim.x) p.cells[i] = p.cells_init[i];
  if (threadIdx.x == 0) {
    ds->cancelled = 0;
    ds->status = 0;
    ds->pass_id = p.mb->pass_id;
    ds->dec_head = ds->feed_head = ds->fetch_head = 0;
    ds->fetch_bytes = 0;
    ds->stall_ns = 0;
    ds->ops = 0;
    ds->trace_n = 0;
    ds->t_begin = globaltimer();
  }
  __syncthreads();
  stamp(ds, SK_BEGIN);
}

constexpr int kMaxCommit = 64;
struct CommitParams {
  DevState* ds;
  int n;
  int var_index[kMaxCommit];
  void** var_cur;             // committed pointer table
  void** var_ovl;             // overlay table
  void** var_spare;           // per-pass spare buffers provided by the host
  long long bytes[kMaxCommit];
};
// Grid (x: chunks, y: assigned variable): copy the overlay value into the
// variable's spare buffer with 16-byte vector stores; block (0, v) flips the
// committed pointer (nothing reads var_cur until the next pass).
__global__ void __launch_bounds__(256) k_commit(CommitParams p) {
  COEX_PDL_ENTER();
  stamp(p.ds, SK_COMMIT);
  if (p.ds->cancelled) return;
  const int j = blockIdx.y;
  if (j >= p.n) return;
  const int v = p.var_index[j];
  const char* src = (const char*)p.var_ovl[v];
  if (src == nullptr) return;
  char* dst = (char*)p.var_spare[v];
  const long long bytes = p.bytes[j];
  const long long tid = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  const long long nth = (long long)gridDim.x * blockDim.x;
  if ((bytes & 15) == 0 && ((uintptr_t)src & 15) == 0 && ((uintptr_t)dst & 15) == 0) {
    const uint4* s4 = (const uint4*)src;
    uint4* d4 = (uint4*)dst;
    for (long long i = tid; i < bytes / 16; i += nth) d4[i] = s4[i];
  } else {
    for (long long i = tid; i < bytes; i += nth) dst[i] = src[i];
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) p.var_cur[v] = dst;
}

struct EndParams {
  DevState* ds;
  Mailbox* mb;
  void** var_ovl;
  int* var_ovl_shape;
  int nvars;
};
__global__ void k_pass_end(EndParams p) {
  COEX_PDL_ENTER();
  DevState* ds = p.ds;
  if (threadIdx.x == 0) stamp(ds, SK_END);
  // one lane per 64-variable word of the dirty bitmap (only the context's defined variables)
  const int nwords = (p.nvars + 63) / 64;
  for (int w = threadIdx.x; w < kMaxDevVars / 64; w += blockDim.x) {
    unsigned long long mask = 0;
    if (w < nwords && !ds->cancelled) {
      for (int b = 0; b < 64; ++b) {
        const int i = w * 64 + b;
        if (i < p.nvars && p.var_ovl[i] != nullptr) {
          mask |= 1ull << b;
          p.mb->var_shape_id[i] = p.var_ovl_shape[i];
        }
      }
    }
    p.mb->dirty[w] = mask;
    if (w == 0) p.mb->dirty_mask = mask;
  }
  __syncwarp();
  if (threadIdx.x != 0) return;
  p.mb->committed = ds->cancelled ? 0 : 1;
  p.mb->status = ds->status;
  p.mb->exec_ns = globaltimer() - ds->t_begin;
  p.mb->stall_ns = ds->stall_ns;
  p.mb->ops = ds->ops;
  p.mb->fetches = ds->fetch_head;
  __threadfence_system();
  st_release_sys(&p.mb->done, ds->pass_id);
}

}  // namespace coex
