// runtime.cu -- host side of libcoexb200.so (C-ABI in include/coex_b200.h).
//
// * Context: device, one execution stream, stream-ordered allocator, the
//   device pass state, and the pinned+mapped mailbox (decision / feed / fetch
//   rings, cancel word, done word) shared with the device.
// * Eager side: refcounted device tensors; coex_exec_op launches one kernel
//   from kernels.cuh (execute_kernel, pkg/src/coex/tensor.py:246-291).
// * Symbolic side: coex_prog_build turns the host planner's plan (a SymProgram
//   specialised to one shape signature) into ONE CUDA graph: compute kernels
//   become kernel nodes, SwitchCase / While become SWITCH / WHILE conditional
//   nodes driven by k_decide kernels that spin on the mapped decision ring,
//   InputFeed / OutputFetch become feed / fetch kernels on the mapped rings.
//   A co-execution step is one cudaGraphLaunch; the host only publishes
//   decisions and fed values.
#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>
#include <cstddef>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <stdexcept>
#include <string>
#include <thread>
#include <unordered_map>
#include <vector>

#include "../../include/coex_b200.h"
#include "kernels.cuh"
#include "nvls.cuh"
#include "gemm_tc.cuh"
#include "gemm_tf32.cuh"
#include "ext_ops.cuh"
#include "xformer_ops.cuh"
#include "attn_tc.cuh"

#include <cudaTypedefs.h>
#include <dlfcn.h>
#include <cerrno>
#include <sys/syscall.h>
#include <unistd.h>

using namespace coex;

namespace {

thread_local std::string g_err;

int fail(int code, const std::string& msg) {
  g_err = msg;
  return code;
}

#define CK(call)                                                                                  \
  do {                                                                                            \
    cudaError_t e_ = (call);                                                                      \
    if (e_ != cudaSuccess)                                                                        \
      return fail(COEX_CUDA_ERROR, std::string(#call) + ": " + cudaGetErrorString(e_) + " @" +    \
                                       std::to_string(__LINE__));                                 \
  } while (0)

constexpr int kMaxVars = 1024;
static_assert(kMaxVars == kMaxDevVars, "variable table sizes");
constexpr int kNumSMs = 148;

struct Buf {
  void* ptr = nullptr;
  size_t bytes = 0;
  int refs = 0;
};

struct TRec {
  Buf* buf = nullptr;
  int ndim = 0;
  int64_t shape[COEX_MAX_RANK] = {0};
  int64_t numel = 1;
};

struct Var {
  std::string name;
  TRec t;
  Buf* spare = nullptr;   // var-owned buffer the next commit writes into
};

int64_t numel_of(int ndim, const int64_t* shape) {
  int64_t n = 1;
  for (int i = 0; i < ndim; ++i) n *= shape[i];
  return n;
}

// A kernel launch, usable both eagerly and as a graph kernel node.
struct Launch {
  void* fn = nullptr;
  dim3 grid{1}, block{1};
  size_t smem = 0;
  alignas(64) unsigned char params[8192];     // k_chain_multi carries up to 8 chain programs
  size_t psize = 0;
  void* args[1];
  // collective instead of a kernel (fn == nullptr): in-place sum all-reduce of ar_count
  // elements at ar_buf over the context's communicator (synchronised batch norm)
  void* ar_buf = nullptr;
  int64_t ar_count = 0;
  int ar_f64 = 1;
  // tcgen05 GEMM whose result lands in the op's Out (1: the GEMM itself, 2: its split-K
  // reduction) -- the NVLS fusion retargets these (Builder::nvls_fuse)
  int tc_dest = 0;
  void* fn_red = nullptr;      // the GEMM's epilogue-reduction instantiation (nullptr: none)
  unsigned red_grid = 0;       // its grid / dynamic shared memory (single-CTA-per-SM variant)
  size_t red_smem = 0;
  void allreduce(void* b, int64_t n, bool f64) {
    fn = nullptr;
    ar_buf = b;
    ar_count = n;
    ar_f64 = f64 ? 1 : 0;
  }
  template <typename P>
  void set(void* f, dim3 g, dim3 b, const P& p) {
    static_assert(sizeof(P) <= sizeof(params), "kernel params too large");
    fn = f;
    grid = g;
    block = b;
    memcpy(params, &p, sizeof(P));
    psize = sizeof(P);
  }
  void** argv() {
    args[0] = params;
    return args;
  }
};

// Blocks that each own a contiguous range of `rows` rows of `units` 16-byte units: enough
// for ~8 rows of work per thread, at most 8 blocks per SM.
dim3 blocks_for_rows(int64_t rows, int64_t units) {
  const int64_t rpi = units >= 256 ? 1 : 256 / (units > 0 ? units : 1);
  int64_t b = rows / (rpi * 8);
  if (b > (int64_t)148 * 8) b = 148 * 8;
  if (b < 1) b = 1;
  return dim3((unsigned)b);
}

dim3 grid_for(int64_t n, int threads = 256, int max_per_sm = 8) {
  int64_t b = (n + threads - 1) / threads;
  if (b < 1) b = 1;
  int64_t cap = (int64_t)kNumSMs * max_per_sm;
  return dim3((unsigned)(b < cap ? b : cap));
}

}  // namespace

struct coex_ctx {
  std::vector<std::pair<char*, size_t>> pinned;   // coex_host_register ranges
  int device = 0;
  int prec = COEX_F64;
  size_t esize = 8;
  cudaStream_t stream = nullptr;
  std::unordered_map<int64_t, TRec> tensors;
  int64_t next_id = 1;
  std::vector<Var> vars;
  std::unordered_map<std::string, int> var_index;
  void** d_var_cur = nullptr;
  void** d_var_ovl = nullptr;
  int* d_var_ovl_shape = nullptr;
  void** d_var_spare = nullptr;
  void** h_var_cur = nullptr;     // pinned mirror
  void** h_var_spare = nullptr;   // pinned mirror
  DevState* d_state = nullptr;
  Mailbox* mb = nullptr;
  Mailbox* d_mb = nullptr;
  double* feed_arena = nullptr;
  double* d_feed_arena = nullptr;
  size_t feed_cap = 0;            // doubles
  char* fetch_arena = nullptr;
  char* d_fetch_arena = nullptr;
  size_t fetch_cap = 0;           // bytes
  unsigned long long* d_jump = nullptr;
  double* h_stage = nullptr;      // pinned staging for put/get
  size_t stage_cap = 0;
  double timeout_s = 120.0;
  int64_t kernel_count = 0;
  coex_prog* active = nullptr;
  unsigned long long pass_counter = 0;
  cudaEvent_t events[64] = {nullptr};
  unsigned long long* d_trace = nullptr;
  int trace_cap = 0;
  void* comm = nullptr;                  // ncclComm_t
  int rank = 0, world = 1;
  cudaStream_t cap_stream = nullptr;     // side stream used to capture collectives into graphs
  // NVLS gradient region (nvls.cuh): this rank's copy and the team's multicast alias of the
  // same bytes; the first kNvlsFlagBytes hold the barrier flags
  char* nv_local = nullptr;
  char* nv_mc = nullptr;
  size_t nv_bytes = 0;
  unsigned long long nv_mc_handle = 0, nv_mem_handle = 0;
  int nv_world = 0, nv_creator = 0, nv_attached = 0;
  unsigned int* nv_gen = nullptr;        // barrier generations (ordinary device memory)
  int nv_next_slot = 0;
  int nv_mode = 0;                       // RedMode: RED_MC (multicast) / RED_P2P (IPC-opened peers)
  double* d_red_part = nullptr;          // k_reduce_multi partials / counter (context scratch)
  unsigned int* d_red_counter = nullptr;
  char* nv_peer[kMaxPeers] = {nullptr};  // RED_P2P: every rank's region (own = nv_local)
  bool nv_p2p_own = false;               // RED_P2P: nv_local from cudaMalloc (freed here)
};

namespace {

bool is_f64(const coex_ctx* c) { return c->prec == COEX_F64; }
// COEX_TF32=1: fp32-mode MatMuls as 3xTF32 on tcgen05 (csrc/gemm_tf32.cuh) instead of the
// SIMT FFMA kernel.  Off by default: the tensor core's fp32 accumulation carries ~2^-19
// relative error per MMA (measured, tools/tf32_err.py: 2.1e-6 per op at K <= 3072 vs 5e-7
// for FFMA), which the north_star's 1e-5 end-to-end gradient bar does not absorb
// (tests/test_gpu_contract.py fp32 cases).  Read per call: the planner reads the same variable.
bool tf32_on() {
  const char* e = getenv("COEX_TF32");
  return e && e[0] == '1';
}
bool tf32_path(const coex_ctx* c) { return c->prec == COEX_F32 && tf32_on(); }


int alloc_buf(coex_ctx* c, size_t bytes, Buf** out) {
  Buf* b = new Buf();
  b->bytes = bytes;
  b->refs = 1;
  if (bytes > 0) {
    cudaError_t e = cudaMallocAsync(&b->ptr, bytes < 16 ? 16 : bytes, c->stream);
    if (e != cudaSuccess) {
      delete b;
      return fail(COEX_CUDA_ERROR, std::string("cudaMallocAsync: ") + cudaGetErrorString(e));
    }
  }
  *out = b;
  return COEX_OK;
}

void release(coex_ctx* c, Buf* b) {
  if (b == nullptr) return;
  if (--b->refs == 0) {
    if (b->ptr) cudaFreeAsync(b->ptr, c->stream);
    delete b;
  }
}

int64_t new_handle(coex_ctx* c, const TRec& t) {
  int64_t id = c->next_id++;
  c->tensors[id] = t;
  return id;
}

int ensure_stage(coex_ctx* c, size_t doubles) {
  if (doubles <= c->stage_cap) return COEX_OK;
  if (c->h_stage) {
    CK(cudaStreamSynchronize(c->stream));
    cudaFreeHost(c->h_stage);
  }
  size_t cap = doubles < 4096 ? 4096 : doubles;
  CK(cudaHostAlloc((void**)&c->h_stage, cap * sizeof(double), cudaHostAllocDefault));
  c->stage_cap = cap;
  return COEX_OK;
}

// ---- GF(2) jump matrices for the synthetic-data generator ----
unsigned long long xs_step_host(unsigned long long x) {
  x ^= x >> 12;
  x ^= x << 25;
  x ^= x >> 27;
  return x;
}
void mat_apply(const unsigned long long* cols, unsigned long long v, unsigned long long* r) {
  unsigned long long acc = 0;
  for (int b = 0; b < 64; ++b)
    if ((v >> b) & 1ull) acc ^= cols[b];
  *r = acc;
}
void mat_square(const unsigned long long* in, unsigned long long* out) {
  for (int b = 0; b < 64; ++b) mat_apply(in, in[b], &out[b]);
}

// ---- shape inference (tensor.py:131-187) ----
int infer_ext(int kind, const coex_attrs* at, const TRec* in, int* ndim, int64_t* shape);

int infer(int kind, const coex_attrs* at, int nin, const TRec* in, int* ndim, int64_t* shape) {
  static const int arity[] = {2, 2, 2, 2, 1, 1, 1, 1, 1, 1, 1, 0, 0, 1,
                              2, 2, 2, 3, 3, 2, 1, 1, 1, 2, 2, 2,
                              2, 2, 2, 3, 3, 2, 2, 1, 2, 2, 2, 2, 1, 2, 2, 2,
                              1, 1, 3, 1, 2, 1, 2, 1, 2,
                              1, 2, 1, 2, 1};
  static_assert(sizeof(arity) / sizeof(arity[0]) == COEX_NUM_KINDS, "arity table");
  if (kind < 0 || kind >= COEX_NUM_KINDS) return fail(COEX_BAD_ATTRS, "unknown op kind");
  if (nin != arity[kind]) return fail(COEX_BAD_ATTRS, "wrong number of tensor inputs");
  if (kind >= COEX_CONV2D) return infer_ext(kind, at, in, ndim, shape);
  switch (kind) {
    case COEX_ADD: case COEX_SUB: case COEX_MUL: {
      const TRec &a = in[0], &b = in[1];
      bool same = a.ndim == b.ndim;
      for (int i = 0; same && i < a.ndim; ++i) same = a.shape[i] == b.shape[i];
      const TRec& r = (same || b.ndim == 0) ? a : (a.ndim == 0 ? b : a);
      if (!(same || a.ndim == 0 || b.ndim == 0)) return fail(COEX_SHAPE_MISMATCH, "elementwise: incompatible shapes");
      *ndim = r.ndim;
      memcpy(shape, r.shape, sizeof(int64_t) * r.ndim);
      return COEX_OK;
    }
    case COEX_NEG: case COEX_RELU: case COEX_SIGMOID: case COEX_ASSIGN_VAR:
      *ndim = in[0].ndim;
      memcpy(shape, in[0].shape, sizeof(int64_t) * in[0].ndim);
      return COEX_OK;
    case COEX_SUM: case COEX_MEAN:
      if (kind == COEX_MEAN && in[0].numel == 0) return fail(COEX_SHAPE_MISMATCH, "mean of an empty tensor");
      *ndim = 0;
      return COEX_OK;
    case COEX_MATMUL:
      if (in[0].ndim != 2 || in[1].ndim != 2) return fail(COEX_SHAPE_MISMATCH, "matmul: rank-2 operands required");
      if (in[0].shape[1] != in[1].shape[0]) return fail(COEX_SHAPE_MISMATCH, "matmul: inner dimensions differ");
      *ndim = 2;
      shape[0] = in[0].shape[0];
      shape[1] = in[1].shape[1];
      return COEX_OK;
    case COEX_TRANSPOSE: {
      if (at == nullptr || at->n != in[0].ndim) return fail(COEX_BAD_ATTRS, "transpose: perm is not a permutation");
      bool seen[COEX_MAX_RANK] = {false};
      for (int i = 0; i < at->n; ++i) {
        int64_t p = at->dims[i];
        if (p < 0 || p >= at->n || seen[p]) return fail(COEX_BAD_ATTRS, "transpose: perm is not a permutation");
        seen[p] = true;
        shape[i] = in[0].shape[p];
      }
      *ndim = at->n;
      return COEX_OK;
    }
    case COEX_RESHAPE: {
      if (at == nullptr || at->n < 0 || at->n > COEX_MAX_RANK) return fail(COEX_BAD_ATTRS, "reshape: bad target shape");
      if (numel_of(at->n, at->dims) != in[0].numel) return fail(COEX_BAD_ATTRS, "reshape: size mismatch");
      *ndim = at->n;
      memcpy(shape, at->dims, sizeof(int64_t) * at->n);
      return COEX_OK;
    }
    case COEX_FILL:
      if (at == nullptr || at->n < 0 || at->n > COEX_MAX_RANK) return fail(COEX_BAD_ATTRS, "fill: bad shape");
      for (int i = 0; i < at->n; ++i)
        if (at->dims[i] < 0) return fail(COEX_BAD_ATTRS, "fill: bad shape");
      *ndim = at->n;
      memcpy(shape, at->dims, sizeof(int64_t) * at->n);
      return COEX_OK;
    default:
      return fail(COEX_BAD_ATTRS, "read_var is executed against the variable store");
  }
}

// Extension op shapes (paper_2201_09210_b200/tensor.py _conv_shape / infer_shape).
int infer_ext(int kind, const coex_attrs* at, const TRec* in, int* ndim, int64_t* shape) {
  auto same = [](const TRec& a, const TRec& b) {
    if (a.ndim != b.ndim) return false;
    for (int i = 0; i < a.ndim; ++i)
      if (a.shape[i] != b.shape[i]) return false;
    return true;
  };
  switch (kind) {
    case COEX_TANH: case COEX_LEAKY_RELU: case COEX_GELU: case COEX_SQRT:
      *ndim = in[0].ndim;
      memcpy(shape, in[0].shape, sizeof(int64_t) * in[0].ndim);
      return COEX_OK;
    case COEX_RELU_GRAD: case COEX_LEAKY_RELU_GRAD: case COEX_BCE_TERM: case COEX_TO_INDEX: case COEX_GELU_GRAD:
    case COEX_DIV: {
      const TRec &a = in[0], &b = in[1];
      if (!(same(a, b) || a.ndim == 0 || b.ndim == 0)) return fail(COEX_SHAPE_MISMATCH, "elementwise: incompatible shapes");
      const TRec& r = (same(a, b) || b.ndim == 0) ? a : b;
      *ndim = r.ndim;
      memcpy(shape, r.shape, sizeof(int64_t) * r.ndim);
      return COEX_OK;
    }
    case COEX_BATCHNORM: case COEX_BATCHNORM_DX: case COEX_BN_DGAMMA: case COEX_SUM_ROWS: {
      const TRec& x = in[0];
      if (x.ndim < 1 || x.numel == 0) return fail(COEX_SHAPE_MISMATCH, "column op: non-empty operand of rank >= 1 required");
      const int64_t C = x.shape[x.ndim - 1];
      if (kind != COEX_SUM_ROWS && C > (int64_t)kColMaxSlots * 256)
        return fail(COEX_SHAPE_MISMATCH, "column op: more than 2048 channels");
      if (kind == COEX_SUM_ROWS || kind == COEX_BN_DGAMMA) {
        if (kind == COEX_BN_DGAMMA && !same(x, in[1])) return fail(COEX_SHAPE_MISMATCH, "bn_dgamma: dy differs from x");
        *ndim = 1;
        shape[0] = C;
        return COEX_OK;
      }
      if (in[1].ndim != 1 || in[1].shape[0] != C) return fail(COEX_SHAPE_MISMATCH, "batchnorm: gamma must be [C]");
      if (kind == COEX_BATCHNORM && (in[2].ndim != 1 || in[2].shape[0] != C))
        return fail(COEX_SHAPE_MISMATCH, "batchnorm: beta must be [C]");
      if (kind == COEX_BATCHNORM_DX && !same(x, in[2])) return fail(COEX_SHAPE_MISMATCH, "batchnorm_dx: dy differs from x");
      *ndim = x.ndim;
      memcpy(shape, x.shape, sizeof(int64_t) * x.ndim);
      return COEX_OK;
    }
    case COEX_EMBEDDING: {
      if (in[0].ndim != 2 || in[1].ndim + 1 > COEX_MAX_RANK) return fail(COEX_SHAPE_MISMATCH, "embedding: table [V, d] required");
      *ndim = in[1].ndim + 1;
      memcpy(shape, in[1].shape, sizeof(int64_t) * in[1].ndim);
      shape[in[1].ndim] = in[0].shape[1];
      return COEX_OK;
    }
    case COEX_EMBEDDING_DW: {
      const TRec &ids = in[0], &dy = in[1];
      if (at == nullptr || at->n != 1 || at->dims[0] < 1) return fail(COEX_BAD_ATTRS, "embedding_dw: attribute [vocab] expected");
      bool ok = dy.ndim == ids.ndim + 1;
      for (int i = 0; ok && i < ids.ndim; ++i) ok = dy.shape[i] == ids.shape[i];
      if (!ok) return fail(COEX_SHAPE_MISMATCH, "embedding_dw: gradient does not match ids + [d]");
      *ndim = 2;
      shape[0] = at->dims[0];
      shape[1] = dy.shape[dy.ndim - 1];
      return COEX_OK;
    }
    case COEX_LAYERNORM: case COEX_LAYERNORM_DX: case COEX_LN_DGAMMA: {
      const TRec& x = in[0];
      if (x.ndim < 1 || x.numel == 0) return fail(COEX_SHAPE_MISMATCH, "layernorm: non-empty operand required");
      const int64_t d = x.shape[x.ndim - 1];
      if (kind == COEX_LN_DGAMMA) {
        if (!same(x, in[1])) return fail(COEX_SHAPE_MISMATCH, "ln_dgamma: dy differs from x");
        if (d > 1024) return fail(COEX_SHAPE_MISMATCH, "ln_dgamma: rows longer than 1024");
        *ndim = 1;
        shape[0] = d;
        return COEX_OK;
      }
      if (in[1].ndim != 1 || in[1].shape[0] != d) return fail(COEX_SHAPE_MISMATCH, "layernorm: gamma must be [d]");
      if (kind == COEX_LAYERNORM && (in[2].ndim != 1 || in[2].shape[0] != d))
        return fail(COEX_SHAPE_MISMATCH, "layernorm: beta must be [d]");
      if (kind == COEX_LAYERNORM_DX && !same(x, in[2])) return fail(COEX_SHAPE_MISMATCH, "layernorm_dx: dy differs from x");
      *ndim = x.ndim;
      memcpy(shape, x.shape, sizeof(int64_t) * x.ndim);
      return COEX_OK;
    }
    case COEX_BIAS_ADD: {
      const TRec &x = in[0], &b = in[1];
      if (x.ndim < 1 || b.ndim != 1 || b.shape[0] != x.shape[x.ndim - 1])
        return fail(COEX_SHAPE_MISMATCH, "bias_add: bias does not match the last dim");
      *ndim = x.ndim;
      memcpy(shape, x.shape, sizeof(int64_t) * x.ndim);
      return COEX_OK;
    }
    case COEX_BMM: case COEX_BMM_NT: case COEX_BMM_TN: {
      const TRec &a = in[0], &b = in[1];
      if (a.ndim != 3 || b.ndim != 3 || a.shape[0] != b.shape[0])
        return fail(COEX_SHAPE_MISMATCH, "bmm: rank-3 operands with equal batch required");
      const int64_t m = kind == COEX_BMM_TN ? a.shape[2] : a.shape[1], ka = kind == COEX_BMM_TN ? a.shape[1] : a.shape[2];
      const int64_t n = kind == COEX_BMM_NT ? b.shape[1] : b.shape[2], kb = kind == COEX_BMM_NT ? b.shape[2] : b.shape[1];
      if (ka != kb) return fail(COEX_SHAPE_MISMATCH, "bmm: inner dimensions differ");
      *ndim = 3;
      shape[0] = a.shape[0]; shape[1] = m; shape[2] = n;
      return COEX_OK;
    }
    case COEX_CAUSAL_SOFTMAX: case COEX_SOFTMAX_GRAD: case COEX_REL_SKEW: case COEX_REL_UNSKEW: {
      const TRec& x = in[0];
      if (x.ndim < 2 || x.shape[x.ndim - 1] != x.shape[x.ndim - 2])
        return fail(COEX_SHAPE_MISMATCH, "softmax: square trailing [T, T] block required");
      if (kind == COEX_SOFTMAX_GRAD && !same(x, in[1])) return fail(COEX_SHAPE_MISMATCH, "softmax_grad: dy differs from y");
      *ndim = x.ndim;
      memcpy(shape, x.shape, sizeof(int64_t) * x.ndim);
      return COEX_OK;
    }
    case COEX_CROSS_ENTROPY: case COEX_CROSS_ENTROPY_GRAD: {
      const TRec &lg = in[0], &ids = in[1];
      if (lg.ndim != 2 || ids.ndim != 1 || ids.shape[0] != lg.shape[0] || lg.shape[0] == 0)
        return fail(COEX_SHAPE_MISMATCH, "cross_entropy: logits [R, V] and ids [R] required");
      if (kind == COEX_CROSS_ENTROPY) {
        *ndim = 0;
      } else {
        *ndim = 2;
        shape[0] = lg.shape[0];
        shape[1] = lg.shape[1];
      }
      return COEX_OK;
    }
    case COEX_SLICE: case COEX_CONCAT: case COEX_SUM_AXIS: {
      const int want = kind == COEX_SLICE ? 3 : 1;
      if (at == nullptr || at->n != want) return fail(COEX_BAD_ATTRS, "axis op: [axis(, start, length)] expected");
      const TRec& x = in[0];
      const int64_t ax = at->dims[0];
      if (ax < 0 || ax >= x.ndim) return fail(COEX_SHAPE_MISMATCH, "axis op: axis out of range");
      *ndim = x.ndim;
      memcpy(shape, x.shape, sizeof(int64_t) * x.ndim);
      if (kind == COEX_SLICE) {
        if (at->dims[1] < 0 || at->dims[2] < 0 || at->dims[1] + at->dims[2] > x.shape[ax])
          return fail(COEX_SHAPE_MISMATCH, "slice: range exceeds the axis");
        shape[ax] = at->dims[2];
      } else if (kind == COEX_SUM_AXIS) {
        for (int i = (int)ax; i + 1 < x.ndim; ++i) shape[i] = x.shape[i + 1];
        *ndim = x.ndim - 1;
      } else {
        const TRec& y = in[1];
        if (y.ndim != x.ndim) return fail(COEX_SHAPE_MISMATCH, "concat: ranks differ");
        for (int i = 0; i < x.ndim; ++i)
          if (i != ax && y.shape[i] != x.shape[i]) return fail(COEX_SHAPE_MISMATCH, "concat: shapes differ off the axis");
        shape[ax] = x.shape[ax] + y.shape[ax];
      }
      return COEX_OK;
    }
    case COEX_GLOBAL_AVGPOOL: case COEX_GLOBAL_AVGPOOL_GRAD: {
      const TRec& x = in[0];
      if (x.ndim != 4 || numel_of(x.ndim, x.shape) == 0) return fail(COEX_SHAPE_MISMATCH, "global_avgpool: rank-4 NHWC input required");
      if (kind == COEX_GLOBAL_AVGPOOL) {
        *ndim = 2; shape[0] = x.shape[0]; shape[1] = x.shape[3];
        return COEX_OK;
      }
      if (in[1].ndim != 2 || in[1].shape[0] != x.shape[0] || in[1].shape[1] != x.shape[3])
        return fail(COEX_SHAPE_MISMATCH, "global_avgpool_grad: gradient does not match [N, C]");
      *ndim = 4; memcpy(shape, x.shape, sizeof(int64_t) * 4);
      return COEX_OK;
    }
    default: break;
  }
  if (kind == COEX_CONV2D_DX) {          // (dy, w, x): x's shape; dy must be conv2d(x, w)'s output
    int nd; int64_t sh[COEX_MAX_RANK];
    const TRec xw[2] = {in[2], in[1]};
    int rc = infer_ext(COEX_CONV2D, at, xw, &nd, sh);
    if (rc) return rc;
    if (!(in[0].ndim == 4 && sh[0] == in[0].shape[0] && sh[1] == in[0].shape[1] && sh[2] == in[0].shape[2] &&
          sh[3] == in[0].shape[3]))
      return fail(COEX_SHAPE_MISMATCH, "conv2d_dx: gradient is not conv2d(x, w)'s output");
    *ndim = 4; memcpy(shape, in[2].shape, sizeof(int64_t) * 4);
    return COEX_OK;
  }
  if (kind >= COEX_MAXPOOL && kind <= COEX_AVGPOOL_GRAD) {
    if (at == nullptr || at->n != 3 || at->dims[0] < 1 || at->dims[1] < 1 || at->dims[2] < 0)
      return fail(COEX_BAD_ATTRS, "pool: attribute [kernel, stride, pad] expected");
    const int64_t k = at->dims[0], st = at->dims[1], pd = at->dims[2];
    const TRec& x = in[0];
    if (x.ndim != 4 || numel_of(x.ndim, x.shape) == 0) return fail(COEX_SHAPE_MISMATCH, "pool: rank-4 NHWC input required");
    if (pd >= k || x.shape[1] + 2 * pd < k || x.shape[2] + 2 * pd < k)
      return fail(COEX_SHAPE_MISMATCH, "pool: window does not fit the input");
    const int64_t o[4] = {x.shape[0], (x.shape[1] + 2 * pd - k) / st + 1, (x.shape[2] + 2 * pd - k) / st + 1, x.shape[3]};
    *ndim = 4;
    if (kind == COEX_MAXPOOL || kind == COEX_AVGPOOL) {
      memcpy(shape, o, sizeof(o));
      return COEX_OK;
    }
    const TRec& g = in[1];
    if (g.ndim != 4 || g.shape[0] != o[0] || g.shape[1] != o[1] || g.shape[2] != o[2] || g.shape[3] != o[3])
      return fail(COEX_SHAPE_MISMATCH, "pool grad: gradient does not match the pooled geometry");
    memcpy(shape, x.shape, sizeof(int64_t) * 4);
    return COEX_OK;
  }
  // convolutions
  if (at == nullptr || at->n != 3 || at->dims[0] < 1 || at->dims[1] < 1 || at->dims[2] < 0)
    return fail(COEX_BAD_ATTRS, "conv: attribute [kernel, stride, pad] expected");
  const int64_t k = at->dims[0], st = at->dims[1], pd = at->dims[2];
  const TRec &x = in[0], &w = in[1];
  if (x.ndim != 4) return fail(COEX_SHAPE_MISMATCH, "conv: rank-4 NHWC input required");
  const int64_t N = x.shape[0], H = x.shape[1], W = x.shape[2], C = x.shape[3];
  *ndim = 4;
  if (kind == COEX_CONV2D_T) {
    if (w.ndim != 2 || w.shape[1] != C || w.shape[0] % (k * k)) return fail(COEX_SHAPE_MISMATCH, "conv2d_t: weight mismatch");
    const int64_t Ho = (H - 1) * st - 2 * pd + k, Wo = (W - 1) * st - 2 * pd + k;
    if (H < 1 || W < 1 || Ho < 1 || Wo < 1) return fail(COEX_SHAPE_MISMATCH, "conv2d_t: empty output");
    shape[0] = N; shape[1] = Ho; shape[2] = Wo; shape[3] = w.shape[0] / (k * k);
    return COEX_OK;
  }
  if (H + 2 * pd < k || W + 2 * pd < k) return fail(COEX_SHAPE_MISMATCH, "conv: kernel larger than padded input");
  const int64_t Ho = (H + 2 * pd - k) / st + 1, Wo = (W + 2 * pd - k) / st + 1;
  if (kind == COEX_CONV2D) {
    if (w.ndim != 2 || w.shape[0] != k * k * C) return fail(COEX_SHAPE_MISMATCH, "conv2d: weight mismatch");
    shape[0] = N; shape[1] = Ho; shape[2] = Wo; shape[3] = w.shape[1];
    return COEX_OK;
  }
  if (w.ndim != 4 || w.shape[0] != N || w.shape[1] != Ho || w.shape[2] != Wo)
    return fail(COEX_SHAPE_MISMATCH, "conv2d_dw: gradient does not match the output geometry");
  *ndim = 2;
  shape[0] = k * k * C;
  shape[1] = w.shape[3];
  return COEX_OK;
}

// ---- kernel selection, shared by eager launches and graph nodes ----
constexpr int kMaxIn = 3;
struct OpSpec {
  int kind = 0;
  int nin = 0;
  In in[kMaxIn] = {{nullptr, nullptr, nullptr}, {nullptr, nullptr, nullptr}, {nullptr, nullptr, nullptr}};
  int in_ndim[kMaxIn] = {0, 0, 0};
  int64_t in_shape[kMaxIn][COEX_MAX_RANK] = {{0}};
  int out_ndim = 0;
  int64_t out_shape[COEX_MAX_RANK] = {0};
  int attr_n = 0;
  int64_t attr_dims[COEX_MAX_RANK] = {0};
  double value = 0.0;
  int trans_a = 0, trans_b = 0;
  void* scratch[2] = {nullptr, nullptr};   // bf16 K-major operand copies (tcgen05 path)
  char* ws = nullptr;                      // extension ops: scratch workspace base (nullptr = size query)
  char* pz = nullptr;                      // extension ops: the op's persistent zeroed state
  Out out{};
  Out out2{}, out3{};                      // fused batch-norm backward: dgamma, dbeta
  void* shadow = nullptr;                  // bf16 copy of the output to write (softmax-type producers)
  void* in_shadow[kMaxIn] = {nullptr, nullptr, nullptr};   // shared bf16 copies of GEMM operands
  int in_conv[kMaxIn] = {1, 1, 1};         // 1: this op converts into in_shadow / scratch first
  int bias = 0;                            // MatMul: in[2] is a [N] bias added by the epilogue
  int skip_f32 = 0;                        // elementwise with a shadow: the fp32 output has no reader
  DevState* ds = nullptr;
};

// Plan-only kind: batchnorm_dx + bn_dgamma + sum_rows over the same (x, dy) fused into one
// column-statistics pass (planner.py _bn_bwd_groups); three outputs dx, dgamma, dbeta.
constexpr int kBnBwdFused = 100;
// Plan-only kind: layernorm_dx + ln_dgamma + sum_rows over the same (x, dy) in one pass
// (planner.py _bn_bwd_groups; outputs dx, dgamma, dbeta; fp32 / bf16 modes, 4 | d <= 1024).
constexpr int kLnBwdFused = 103;
constexpr int kSkewAdd = 104;      // add(a, rel_skew(x)) in one pass (planner _skew_pairs)
// Plan-only kind: batchnorm whose apply pass also writes relu / leaky_relu of its output
// (planner.py _bn_act_pairs; attr dims[0] = the activation's EW code; second output out2).
constexpr int kBnAct = 101;
// Plan-only kind: cross_entropy + cross_entropy_grad of the same logits / ids in one pass
// (planner.py _ce_pairs; out = the gradient, out2 = the loss; value = global rows or 0).
constexpr int kCeFused = 102;
bool is_ext_compute(int kind) {
  return (kind >= COEX_CONV2D && kind <= COEX_SUM_ROWS) || kind == kBnBwdFused || kind == kBnAct || kind == kCeFused ||
         kind == kLnBwdFused || kind == kSkewAdd ||
         (kind >= COEX_EMBEDDING && kind <= COEX_GLOBAL_AVGPOOL_GRAD && kind != COEX_GELU && kind != COEX_GELU_GRAD) ||
         (kind >= COEX_SLICE && kind <= COEX_SUM_AXIS);
}
int ew_code(int kind) {
  switch (kind) {
    case COEX_ADD: return EW_ADD;
    case COEX_SUB: return EW_SUB;
    case COEX_MUL: return EW_MUL;
    case COEX_NEG: return EW_NEG;
    case COEX_RELU: return EW_RELU;
    case COEX_SIGMOID: return EW_SIGMOID;
    case COEX_TANH: return EW_TANH;
    case COEX_LEAKY_RELU: return EW_LRELU;
    case COEX_RELU_GRAD: return EW_RELU_GRAD;
    case COEX_LEAKY_RELU_GRAD: return EW_LRELU_GRAD;
    case COEX_TO_INDEX: return EW_TO_INDEX;
    case COEX_GELU: return EW_GELU;
    case COEX_GELU_GRAD: return EW_GELU_GRAD;
    case COEX_SQRT: return EW_SQRT;
    case COEX_DIV: return EW_DIV;
    default: return EW_BCE;
  }
}

// ---- TMA tensor maps (driver entry point; no -lcuda link dependency) ----
PFN_cuTensorMapEncodeTiled_v12000 tmap_encoder() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  if (fn == nullptr) {
    cudaDriverEntryPointQueryResult q;
    void* p = nullptr;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = (PFN_cuTensorMapEncodeTiled_v12000)p;
  }
  return fn;
}

int64_t bf16_pitch(int64_t K) { return (K + 7) / 8 * 8; }

// ---- NCCL, bound at run time (single-GPU use needs no NCCL at all) ----
typedef struct { char internal[128]; } nccl_uid_t;
typedef void* nccl_comm_t;
enum { kNcclFloat = 7, kNcclDouble = 8, kNcclSum = 0, kNcclAvg = 4 };   // nccl.h ncclDataType_t / ncclRedOp_t
struct NcclApi {
  int (*get_unique_id)(nccl_uid_t*) = nullptr;
  int (*comm_init_rank)(nccl_comm_t*, int, nccl_uid_t, int) = nullptr;
  int (*all_reduce)(const void*, void*, size_t, int, int, nccl_comm_t, cudaStream_t) = nullptr;
  int (*comm_destroy)(nccl_comm_t) = nullptr;
  const char* (*error_string)(int) = nullptr;
  bool ok = false;
};
NcclApi& nccl() {
  static NcclApi api;
  static bool tried = false;
  if (!tried) {
    tried = true;
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);     // reuse torch's copy if loaded
    if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
    if (h) {
      api.get_unique_id = (int (*)(nccl_uid_t*))dlsym(h, "ncclGetUniqueId");
      api.comm_init_rank = (int (*)(nccl_comm_t*, int, nccl_uid_t, int))dlsym(h, "ncclCommInitRank");
      api.all_reduce = (int (*)(const void*, void*, size_t, int, int, nccl_comm_t, cudaStream_t))dlsym(h, "ncclAllReduce");
      api.comm_destroy = (int (*)(nccl_comm_t))dlsym(h, "ncclCommDestroy");
      api.error_string = (const char* (*)(int))dlsym(h, "ncclGetErrorString");
      api.ok = api.get_unique_id && api.comm_init_rank && api.all_reduce && api.comm_destroy;
    }
  }
  return api;
}

// bf16 [rows][pitch] K-major tile source: box {64, box_rows}, 128-byte swizzle, OOB -> 0.
int make_tmap(CUtensorMap* m, void* base, int64_t rows, int64_t K, int box_rows) {
  auto enc = tmap_encoder();
  if (!enc) return fail(COEX_CUDA_ERROR, "cuTensorMapEncodeTiled unavailable");
  cuuint64_t dims[2] = {(cuuint64_t)(K > 0 ? K : 1), (cuuint64_t)(rows > 0 ? rows : 1)};
  cuuint64_t strides[1] = {(cuuint64_t)bf16_pitch(K > 0 ? K : 1) * 2};
  cuuint32_t box[2] = {(cuuint32_t)TC_BK, (cuuint32_t)box_rows};
  cuuint32_t es[2] = {1, 1};
  CUresult r = enc(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, base, dims, strides, box, es,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return fail(COEX_CUDA_ERROR, "cuTensorMapEncodeTiled failed: " + std::to_string((int)r));
  return COEX_OK;
}

// SIMT MatMul kernel choice (parity / fp32 paths): 64x64 tiles when they fill the SMs.
template <typename T>
void simt_matmul_launch(coex_ctx* c, const MatmulParams& p, Launch* L) {
  const int64_t tiles_big = ((p.M + 63) / 64) * ((p.N + 63) / 64);
  const bool exact = is_f64(c);
  if (tiles_big >= kNumSMs) {
    dim3 g((unsigned)(tiles_big < kNumSMs * 4 ? tiles_big : kNumSMs * 4));
    if (exact) L->set((void*)k_matmul_pipe<T, 64, 64, 16, 4, 4, true, sizeof(T) == 8 ? 2 : 3>, g, dim3(256), p);
    else L->set((void*)k_matmul_pipe<T, 64, 64, 16, 4, 4, false, sizeof(T) == 8 ? 2 : 3>, g, dim3(256), p);
  } else {
    int64_t tiles = ((p.M + 15) / 16) * ((p.N + 15) / 16);
    dim3 g((unsigned)(tiles < kNumSMs * 8 ? (tiles < 1 ? 1 : tiles) : kNumSMs * 8));
    if (exact) L->set((void*)k_matmul_pipe<T, 16, 16, 32, 1, 1, true, 4>, g, dim3(256), p);
    else L->set((void*)k_matmul_pipe<T, 16, 16, 32, 1, 1, false, 4>, g, dim3(256), p);
  }
}

// bf16 [K rows][pitch(MN)] MN-major operand: box {64 MN, 64 K}, 128-byte swizzle, OOB -> 0.
int make_tmap_mn(CUtensorMap* m, void* base, int64_t mn, int64_t K) {
  auto enc = tmap_encoder();
  if (!enc) return fail(COEX_CUDA_ERROR, "cuTensorMapEncodeTiled unavailable");
  cuuint64_t dims[2] = {(cuuint64_t)(mn > 0 ? mn : 1), (cuuint64_t)(K > 0 ? K : 1)};
  cuuint64_t strides[1] = {(cuuint64_t)bf16_pitch(mn > 0 ? mn : 1) * 2};
  cuuint32_t box[2] = {64, (cuuint32_t)TC_BK};
  cuuint32_t es[2] = {1, 1};
  CUresult r = enc(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, base, dims, strides, box, es,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return fail(COEX_CUDA_ERROR, "cuTensorMapEncodeTiled (MN) failed: " + std::to_string((int)r));
  return COEX_OK;
}

template <typename T>
int build_launch_t(coex_ctx* c, const OpSpec& s, Launch* L) {
  const int64_t n = numel_of(s.out_ndim, s.out_shape);
  switch (s.kind) {
    case COEX_ADD: case COEX_SUB: case COEX_MUL: case COEX_NEG: case COEX_RELU: case COEX_SIGMOID:
    case COEX_TANH: case COEX_LEAKY_RELU: case COEX_RELU_GRAD: case COEX_LEAKY_RELU_GRAD: case COEX_BCE_TERM:
    case COEX_TO_INDEX: case COEX_GELU: case COEX_GELU_GRAD: case COEX_SQRT: case COEX_DIV: {
      EwParams p{};
      p.ds = s.ds;
      p.a = s.in[0];
      p.b = s.in[1];
      p.op = ew_code(s.kind);
      int binary = ew_binary(p.op);
      p.a_scalar = binary && s.in_ndim[0] == 0 && n != 1;
      p.b_scalar = binary && s.in_ndim[1] == 0 && n != 1;
      p.n = n;
      p.out = s.out;
      p.shadow = (__nv_bfloat16*)s.shadow;
      p.skip_f32 = s.shadow ? s.skip_f32 : 0;
      L->set((void*)k_elementwise<T>, grid_for(sizeof(T) == 4 && n % 4 == 0 ? n / 4 : n), dim3(256), p);
      return COEX_OK;
    }
    case COEX_SUM: case COEX_MEAN: {
      ReduceParams p{};
      p.ds = s.ds;
      p.a = s.in[0];
      p.n = numel_of(s.in_ndim[0], s.in_shape[0]);
      p.mean = s.kind == COEX_MEAN;
      p.out = s.out;
      if (is_f64(c)) {
        L->set((void*)k_reduce_seq_smem<T>, dim3(1), dim3(256), p);
      } else if (p.n >= (1 << 20) && c->d_red_part != nullptr) {
        // large tolerance-mode sums: every SM (was one block of 1024 threads)
        int64_t g = p.n / 16384;
        g = g < 2 * kNumSMs ? g : 2 * kNumSMs;
        p.part = c->d_red_part;
        p.counter = c->d_red_counter;
        L->set((void*)k_reduce_multi<T>, dim3((unsigned)(g < 2 ? 2 : g)), dim3(256), p);
      } else {
        L->set((void*)k_reduce_tree<T>, dim3(1), dim3(1024), p);
      }
      return COEX_OK;
    }
    case COEX_TRANSPOSE: {
      TransposeParams p{};
      p.ds = s.ds;
      p.a = s.in[0];
      p.rank = s.out_ndim;
      p.n = n;
      int64_t istr[COEX_MAX_RANK];
      int64_t acc = 1;
      for (int d = s.in_ndim[0] - 1; d >= 0; --d) {
        istr[d] = acc;
        acc *= s.in_shape[0][d];
      }
      for (int d = 0; d < s.out_ndim; ++d) {
        p.out_shape[d] = s.out_shape[d];
        p.src_stride[d] = istr[s.attr_dims[d]];
      }
      p.out = s.out;
      if (s.out_ndim == 2 && s.attr_dims[0] == 1) {
        int64_t tiles = ((s.out_shape[1] + 31) / 32) * ((s.out_shape[0] + 31) / 32);
        L->set((void*)k_transpose2d<T>, dim3((unsigned)(tiles < kNumSMs * 8 ? (tiles < 1 ? 1 : tiles) : kNumSMs * 8)),
               dim3(32, 8), p);
      } else {
        const int64_t inner = s.out_shape[s.out_ndim - 1];
        if (s.out_ndim >= 2 && s.attr_dims[s.out_ndim - 1] == s.out_ndim - 1 && inner % (16 / (int64_t)sizeof(T)) == 0)
          L->set((void*)k_transpose_rows<T>, grid_for(n / (16 / sizeof(T))), dim3(256), p);
        else
          L->set((void*)k_transpose<T>, grid_for(n), dim3(256), p);
      }
      return COEX_OK;
    }
    case COEX_MATMUL: {
      if (c->prec == COEX_BF16) return fail(COEX_INVALID, "bf16 matmul is lowered by build_launches");
      MatmulParams p{};
      p.ds = s.ds;
      p.a = s.in[0];
      p.b = s.in[1];
      p.trans_a = s.trans_a;
      p.trans_b = s.trans_b;
      // logical shapes: A [M,K], B [K,N]; stored transposed when trans_*
      p.M = s.trans_a ? s.in_shape[0][1] : s.in_shape[0][0];
      p.K = s.trans_a ? s.in_shape[0][0] : s.in_shape[0][1];
      p.N = s.trans_b ? s.in_shape[1][0] : s.in_shape[1][1];
      p.lda = s.in_shape[0][1];
      p.ldb = s.in_shape[1][1];
      p.out = s.out;
      simt_matmul_launch<T>(c, p, L);
      return COEX_OK;
    }
    case COEX_FILL: {
      FillParams p{};
      p.ds = s.ds;
      p.value = s.value;
      p.n = n;
      p.out = s.out;
      L->set((void*)k_fill<T>, grid_for(n), dim3(256), p);
      return COEX_OK;
    }
    default:
      return fail(COEX_BAD_ATTRS, "op kind has no kernel");
  }
}

int build_launch(coex_ctx* c, const OpSpec& s, Launch* L) {
  return is_f64(c) ? build_launch_t<double>(c, s, L) : build_launch_t<float>(c, s, L);
}

// ---- tcgen05 GEMM launch: C[M,N] = A[M,K] . B^T where A / B are bf16 K-major [rows][pitch(K)] ----
// BN = 64 / 128 / 256 by N; split-K (deterministic slice reduction) when the tile grid cannot
// fill the SMs.  Output: the node's Out (publishes) or `raw` scratch.
struct TcPlan {
  int bn = 256, splits = 1;
  int64_t tiles = 1;
};
// Tile width and split-K count from a small cost model of one launch: waves of CTAs, each
// bounded by its MMA time or its L2->SMEM operand stream, plus the fp32 epilogue store and a
// fixed prologue; split-K adds the slice reduction.  (Per-SM figures: 1/148 of the measured
// bf16 peak, ~135 GB/s of L2 operand bandwidth, ~44 GB/s of concurrent store bandwidth.)
int duo_kmax() {
  static int kmax = -1;
  if (kmax < 0) {
    const char* e = getenv("COEX_DUO_KMAX");
    kmax = e ? atoi(e) : 32;
  }
  return kmax;
}
// COEX_DUO_MODEL=0: the cost model ignores the two-CTA slots (A/B)
bool duo_model() {
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("COEX_DUO_MODEL");
    v = (e && e[0] == '0') ? 0 : 1;
  }
  return v == 1;
}
int duo_mode();
double bn256_bias() {
  static double v = -1;
  if (v < 0) {
    const char* e = getenv("COEX_BN256_BIAS");
    v = e ? atof(e) : 0.9;
  }
  return v;
}
double duo_penalty() {
  static double v = -1;
  if (v < 0) {
    const char* e = getenv("COEX_DUO_PENALTY");
    v = e ? atof(e) : 1.7;
  }
  return v;
}
// The DUO (two CTAs per SM) decision for a launch of tile width bn whose split holds
// `kblocks` K-blocks (= ceil(K / BK) / splits, integer division as the launch computes it);
// tc_plan prices tiles with the same rule the launch applies.
bool tc_use_duo(int bn, int64_t kblocks) {
  const int dm = duo_mode();
  return bn <= 128 && (dm == 1 || (dm < 0 && kblocks <= duo_kmax()));
}

TcPlan tc_plan(int64_t M, int64_t N, int64_t K, bool allow_split) {
  TcPlan best;
  double best_t = 1e30;
  const int64_t nk = (K + TC_BK - 1) / TC_BK;
  static int force_bn = -1;
  if (force_bn < 0) {
    const char* e = getenv("COEX_FORCE_BN");     // tuning experiments only
    force_bn = e ? atoi(e) : 0;
  }
  static int max_split = -1;
  if (max_split < 0) {
    const char* e = getenv("COEX_MAX_SPLIT");     // tuning experiments only
    max_split = e ? atoi(e) : 32;
  }
  const int bns[3] = {64, 128, 256};
  for (int bn : bns) {
    if (force_bn && bn != force_bn) continue;
    if (bn > 64 && N <= bn / 2) continue;
    const int64_t tiles = ((M + TC_BM - 1) / TC_BM) * ((N + bn - 1) / bn);
    int64_t smax = allow_split ? (nk / 2 < 32 ? (nk / 2 > 1 ? nk / 2 : 1) : 32) : 1;
    if (smax > max_split) smax = max_split < 1 ? 1 : max_split;
    for (int64_t sp = 1; sp <= smax; ++sp) {
      // persistent CTAs: items per CTA run back to back, the epilogue of one item overlapping
      // the MMAs of the next (two TMEM accumulators)
      const int64_t items = (tiles < 1 ? 1 : tiles) * sp;
      const double kper = (double)((nk + sp - 1) / sp);
      // launches the DUO variant takes (tc_gemm_launches) hold two CTAs per SM
      const int64_t slots = duo_model() && tc_use_duo(bn, nk / sp) ? 2 * kNumSMs : kNumSMs;
      const int64_t rounds = (items + slots - 1) / slots;
      // per-SM figures fitted to measured launches (tools/ncu_ops.py qkt / gemm_8192 with
      // COEX_FORCE_BN): ~115 GB/s of TMA operand feed, ~23.5 GB/s of epilogue stores and
      // ~0.9 us of fixed cost per work item (barrier round trips, TMEM hand-off)
      const double mma = kper * 2.0 * TC_BM * bn * TC_BK / 10.7e12;
      const double feed = kper * (double)(TC_BM + bn) * TC_BK * 2 / 115e9;
      const double epi = (double)TC_BM * bn * 4 / 23.5e9;
      double body = mma > feed ? mma : feed;
      if (epi > body) body = epi;
      // the DUO variant's two-stage ring leaves TMA latency exposed: measured per-item cost
      // (tools/ncu_ops.py c4_* with COEX_DUO / COEX_FORCE_BN) ~1.7x the single-CTA model
      if (slots > kNumSMs) body *= duo_penalty();
      double t = rounds * (body + 0.9e-6) + epi + 2e-6;
      if (sp > 1) t += (double)(sp + 1) * M * N * 4 / 5.5e12 + 3e-6;
      if (bn == 256) t *= bn256_bias();           // measured: the wide tile beats the model
      if (t < best_t * 0.98) {
        best_t = t;
        best.bn = bn;
        best.splits = (int)sp;
        best.tiles = tiles < 1 ? 1 : tiles;
      }
    }
  }
  return best;
}

size_t matmul_split_ws(int64_t M, int64_t N, int64_t K) {
  const TcPlan t = tc_plan(M, N, K, true);
  return t.splits > 1 ? (size_t)t.splits * M * N * 4 : 0;
}

// 3xTF32 launch shape: BN 64 for narrow outputs, else 128; split-K when the tile grid covers
// under half of the SMs and each slice keeps >= 8 K blocks of 32
TcPlan tf32_plan(int64_t M, int64_t N, int64_t K, bool allow_split) {
  TcPlan t;
  t.bn = N <= 64 ? 64 : 128;
  t.tiles = ((M + TC_BM - 1) / TC_BM) * ((N + t.bn - 1) / t.bn);
  if (t.tiles < 1) t.tiles = 1;
  const int64_t nk = (K + TF_BK - 1) / TF_BK;
  t.splits = 1;
  if (allow_split && t.tiles * 2 <= kNumSMs) {
    int64_t sp = kNumSMs / t.tiles;
    if (sp > nk / 8) sp = nk / 8;
    if (sp > 16) sp = 16;
    t.splits = sp > 1 ? (int)sp : 1;
  }
  // accuracy: one TMEM accumulation chain covers at most COEX_TF32_MAXK K elements (slices are
  // summed in IEEE fp32 by k_splitk_reduce)
  static int64_t maxk = -1;
  if (maxk < 0) {
    const char* e = getenv("COEX_TF32_MAXK");
    maxk = e ? atoll(e) : 1024;
  }
  if (allow_split && maxk > 0) {
    const int64_t need = (K + maxk - 1) / maxk;
    if (need > t.splits) t.splits = (int)(need < 64 ? need : 64);
  }
  return t;
}
size_t matmul_split_ws_c(const coex_ctx* c, int64_t M, int64_t N, int64_t K) {
  if (!tf32_path(c)) return matmul_split_ws(M, N, K);
  const TcPlan t = tf32_plan(M, N, K, true);
  return t.splits > 1 ? (size_t)t.splits * M * N * 4 : 0;
}

// fp32 hi / lo planes [2][rows][ld]: 3-D map {ld, rows, 2}, box {32, box_rows, 1}, 128-byte swizzle
int make_tmap_tf32(CUtensorMap* m, void* base, int64_t rows, int64_t ld, int box_rows) {
  auto enc = tmap_encoder();
  if (!enc) return fail(COEX_CUDA_ERROR, "cuTensorMapEncodeTiled unavailable");
  cuuint64_t dims[3] = {(cuuint64_t)ld, (cuuint64_t)(rows > 0 ? rows : 1), 2};
  cuuint64_t strides[2] = {(cuuint64_t)ld * 4, (cuuint64_t)ld * 4 * (rows > 0 ? rows : 1)};
  cuuint32_t box[3] = {(cuuint32_t)TF_BK, (cuuint32_t)box_rows, 1};
  cuuint32_t es[3] = {1, 1, 1};
  CUresult r = enc(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, base, dims, strides, box, es,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return fail(COEX_CUDA_ERROR, "cuTensorMapEncodeTiled (tf32) failed: " + std::to_string((int)r));
  return COEX_OK;
}

// fp32-mode MatMul: operand split (k_cvt_tf32, one launch for both operands) + k_gemm_tf32
// (+ split-K reduction)
int tf32_gemm_launches(coex_ctx* c, const OpSpec& s, int64_t M, int64_t N, int64_t K, Launch* L, int* nL) {
  const int64_t ld = tf32_pitch(K > 0 ? K : 1);
  TfCvtParams q{};
  q.ds = s.ds;
  q.src[0] = s.in[0];
  q.src[1] = s.in[1];
  q.rows[0] = M;
  q.rows[1] = N;
  q.K = K;
  q.ld = ld;
  q.trans[0] = s.trans_a ? 1 : 0;                  // A stored [K][M] when folded from a transpose
  q.trans[1] = s.trans_b ? 0 : 1;                  // B^T rows: B stored [K][N] unless folded
  q.dst[0] = (float*)s.scratch[0];
  q.dst[1] = (float*)s.scratch[1];
  const int64_t units = (M > N ? M : N) * ld / 4;
  int64_t gx = (units + 255) / 256;
  if (q.trans[0] || q.trans[1]) {
    const int64_t tiles = (((M > N ? M : N) + 31) / 32) * ((ld + 31) / 32);
    if (tiles > gx) gx = tiles;
  }
  if (gx > kNumSMs * 16) gx = kNumSMs * 16;
  *nL = 0;
  L[(*nL)++].set((void*)k_cvt_tf32, dim3((unsigned)(gx < 1 ? 1 : gx), 2), dim3(256), q);
  const TcPlan t = tf32_plan(M, N, K, s.ws != nullptr);
  TcGemmParams gp;
  memset(&gp, 0, sizeof(gp));
  int rc = make_tmap_tf32(&gp.tmA, s.scratch[0], M, ld, TC_BM);
  if (!rc) rc = make_tmap_tf32(&gp.tmB, s.scratch[1], N, ld, t.bn);
  if (rc) return rc;
  gp.ds = s.ds;
  gp.a = s.in[0];
  gp.b = s.in[1];
  gp.M = M;
  gp.N = N;
  gp.K = K;
  gp.out = s.out;
  gp.splits = t.splits;
  gp.raw = t.splits > 1 ? (float*)s.ws : nullptr;
  gp.cv.phases = 1;
  gp.batch = 1;
  const int64_t items = t.tiles * t.splits;
  Launch& G = L[(*nL)++];
  G.set(t.bn == 64 ? (void*)k_gemm_tf32<64> : (void*)k_gemm_tf32<128>,
        dim3((unsigned)(items < kNumSMs ? items : kNumSMs)), dim3(TC_THREADS), gp);
  G.smem = t.bn == 64 ? TfCfg<64>::SMEM : TfCfg<128>::SMEM;
  static bool attr = false;
  if (!attr) {
    CK(cudaFuncSetAttribute((const void*)k_gemm_tf32<64>, cudaFuncAttributeMaxDynamicSharedMemorySize, TfCfg<64>::SMEM));
    CK(cudaFuncSetAttribute((const void*)k_gemm_tf32<128>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                            TfCfg<128>::SMEM));
    attr = true;
  }
  if (t.splits > 1) {
    SplitReduceParams r{};
    r.ds = s.ds;
    r.ws = (float*)s.ws;
    r.n = M * N;
    r.splits = t.splits;
    r.a = s.in[0];
    r.b = s.in[1];
    r.out = s.out;
    L[(*nL)++].set((void*)k_splitk_reduce, grid_for(M * N / 4 + 1), dim3(256), r);
  }
  return COEX_OK;
}

// Appends the GEMM (and its split-K reduction) to L.  `ws` = fp32 split slices (splits > 1).
// Kernel variants: AMODE 0/1 (2-D A, K- or MN-major) x B_MN, AMODE 2/3 (implicit conv) x B_MN.
template <int BN, bool DUO = false>
void* tc_fn(int amode, bool bmn) {
  switch (amode) {
    case 0: return bmn ? (void*)k_gemm_tc<BN, 0, true, DUO> : (void*)k_gemm_tc<BN, 0, false, DUO>;
    case 1: return bmn ? (void*)k_gemm_tc<BN, 1, true, DUO> : (void*)k_gemm_tc<BN, 1, false, DUO>;
    case 2: return (void*)k_gemm_tc<BN, 2, true, DUO>;
    default: return (void*)k_gemm_tc<BN, 3, true, DUO>;
  }
}
// epilogue-reduction variants (nvls.cuh) of the single-CTA kernels; nullptr: none (amode 2)
template <int BN>
void* tc_fn_red(int amode, bool bmn) {
  switch (amode) {
    case 0: return bmn ? (void*)k_gemm_tc<BN, 0, true, false, true> : (void*)k_gemm_tc<BN, 0, false, false, true>;
    case 1: return bmn ? (void*)k_gemm_tc<BN, 1, true, false, true> : (void*)k_gemm_tc<BN, 1, false, false, true>;
    case 3: return (void*)k_gemm_tc<BN, 3, true, false, true>;
    default: return nullptr;
  }
}
template <int BN>
int tc_attr_red(int amode, bool bmn) {
  static bool done[8] = {false};
  const int i = amode * 2 + (bmn ? 1 : 0);
  void* f = tc_fn_red<BN>(amode, bmn);
  if (f && !done[i]) {
    CK(cudaFuncSetAttribute((const void*)f, cudaFuncAttributeMaxDynamicSharedMemorySize, TcCfg<BN>::SMEM));
    done[i] = true;
  }
  return COEX_OK;
}
template <int BN, bool DUO = false>
int tc_attr(int amode, bool bmn) {
  static bool done[8] = {false};
  const int i = amode * 2 + (bmn ? 1 : 0);
  if (!done[i]) {
    CK(cudaFuncSetAttribute((const void*)tc_fn<BN, DUO>(amode, bmn), cudaFuncAttributeMaxDynamicSharedMemorySize,
                            TcCfg<BN, DUO>::SMEM));
    done[i] = true;
  }
  return COEX_OK;
}
// COEX_DUO: 0 never / 1 always (BN <= 128) / unset: the cost-model policy in tc_gemm_launches
int duo_mode() {
  static int m = -2;
  if (m == -2) {
    const char* e = getenv("COEX_DUO");
    m = e ? atoi(e) : -1;
  }
  return m;
}

// Batched operands (bmm): 3-D maps {inner, rows, batch} over [batch][rows][pitch(inner)] bf16.
int make_tmap3(CUtensorMap* m, void* base, int64_t rows, int64_t inner, int64_t batch, int box_inner, int box_rows) {
  auto enc = tmap_encoder();
  if (!enc) return fail(COEX_CUDA_ERROR, "cuTensorMapEncodeTiled unavailable");
  const int64_t pitch = bf16_pitch(inner > 0 ? inner : 1);
  cuuint64_t dims[3] = {(cuuint64_t)(inner > 0 ? inner : 1), (cuuint64_t)(rows > 0 ? rows : 1), (cuuint64_t)batch};
  cuuint64_t strides[2] = {(cuuint64_t)pitch * 2, (cuuint64_t)pitch * 2 * (rows > 0 ? rows : 1)};
  cuuint32_t box[3] = {(cuuint32_t)box_inner, (cuuint32_t)box_rows, 1};
  cuuint32_t es[3] = {1, 1, 1};
  CUresult r = enc(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, base, dims, strides, box, es,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return fail(COEX_CUDA_ERROR, "cuTensorMapEncodeTiled (3-D) failed: " + std::to_string((int)r));
  return COEX_OK;
}

// 4-D NHWC bf16 gather map for the implicit-GEMM convolutions: box {64 channels, bw*s, bh*s, bn},
// element strides {1, s, s, 1}, 128-byte swizzle, out-of-bounds (padding) -> 0.
int make_tmap_conv(CUtensorMap* m, void* base, int64_t N, int64_t H, int64_t W, int64_t C, int s, int bw, int bh,
                   int bn) {
  auto enc = tmap_encoder();
  if (!enc) return fail(COEX_CUDA_ERROR, "cuTensorMapEncodeTiled unavailable");
  cuuint64_t dims[4] = {(cuuint64_t)C, (cuuint64_t)W, (cuuint64_t)H, (cuuint64_t)N};
  cuuint64_t strides[3] = {(cuuint64_t)C * 2, (cuuint64_t)W * C * 2, (cuuint64_t)H * W * C * 2};
  cuuint32_t box[4] = {64, (cuuint32_t)(bw * s), (cuuint32_t)(bh * s), (cuuint32_t)bn};
  cuuint32_t es[4] = {1, (cuuint32_t)s, (cuuint32_t)s, 1};
  CUresult r = enc(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 4, base, dims, strides, box, es,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return fail(COEX_CUDA_ERROR, "cuTensorMapEncodeTiled (conv) failed: " + std::to_string((int)r));
  return COEX_OK;
}

// Pixel block {bw, bh, bn} of `pix` consecutive pixels of an Hg x Wg grid that tiles it exactly
// (so every M tile / K block of pixels is one TMA box).
bool conv_blocks(int64_t Hg, int64_t Wg, int pix, int* bw, int* bh, int* bn) {
  if (Wg >= pix) {
    if (Wg % pix) return false;
    *bw = pix; *bh = 1; *bn = 1;
  } else if (Hg * Wg >= pix) {
    if (pix % Wg || Hg % (pix / Wg)) return false;
    *bw = (int)Wg; *bh = pix / (int)Wg; *bn = 1;
  } else {
    if (pix % (Hg * Wg)) return false;
    *bw = (int)Wg; *bh = (int)Hg; *bn = pix / (int)(Hg * Wg);
  }
  return *bw * 2 <= 256 && *bh * 2 <= 256;
}

// amode: 0 A K-major [M][pitch(K)], 1 A MN-major [K][pitch(M)], 2 / 3 implicit convolution
// (A gathered by `conv_map` with geometry `cv`); b_mn: B stored [K][pitch(N)] instead of [N][pitch(K)].
int tc_gemm_launches(coex_ctx* c, DevState* ds, void* a16, void* b16, int64_t M, int64_t N, int64_t K,
                     const TcPlan& t, In na, In nb, const Out& out, float* raw, float* ws, Launch* L, int* nL,
                     int amode = 0, bool b_mn = false, const TcConv* cv = nullptr,
                     const CUtensorMap* conv_map = nullptr, int64_t batch = 1, const In* bias = nullptr) {
  TcGemmParams gp;
  memset(&gp, 0, sizeof(gp));
  if (bias) {
    if (amode >= 2 || batch > 1) return fail(COEX_INVALID, "GEMM bias epilogue: plain 2-D MatMul only");
    gp.bias = *bias;
    gp.has_bias = t.splits > 1 ? 0 : 1;          // split-K: the slice reduction adds it
  }
  int rc = COEX_OK;
  if (amode >= 2) gp.tmA = *conv_map;
  else if (batch > 1) rc = amode == 1 ? make_tmap3(&gp.tmA, a16, K, M, batch, 64, TC_BK) : make_tmap3(&gp.tmA, a16, M, K, batch, TC_BK, TC_BM);
  else rc = amode == 1 ? make_tmap_mn(&gp.tmA, a16, M, K) : make_tmap(&gp.tmA, a16, M, K, TC_BM);
  if (rc) return rc;
  if (cv) gp.cv = *cv;
  else gp.cv.phases = 1;
  gp.batch = (int)batch;
  gp.c_bstride = M * N;
  const int64_t brows = K * ((amode == 2 && cv) ? cv->phases : 1);    // sub-pixel phases stack their B
  if (batch > 1) rc = b_mn ? make_tmap3(&gp.tmB, b16, K, N, batch, 64, TC_BK) : make_tmap3(&gp.tmB, b16, N, K, batch, TC_BK, t.bn);
  else rc = b_mn ? make_tmap_mn(&gp.tmB, b16, N, brows) : make_tmap(&gp.tmB, b16, N, K, t.bn);
  if (rc) return rc;
  gp.ds = ds;
  gp.a = na;
  gp.b = nb;
  gp.M = M;
  gp.N = N;
  gp.K = K;
  gp.out = out;
  gp.splits = t.splits;
  gp.raw = t.splits > 1 ? ws : raw;
  Launch& G = L[(*nL)++];
  G.tc_dest = raw == nullptr ? 1 : 0;
  const int64_t items = ((M + TC_BM - 1) / TC_BM) * ((N + t.bn - 1) / t.bn) * t.splits *
                        (amode == 2 ? gp.cv.phases : 1) * (batch > 1 ? batch : 1);
  // two CTAs per SM for short-K launches that do not fill two waves of single CTAs
  const int64_t kblocks = (K + TC_BK - 1) / TC_BK / (t.splits > 0 ? t.splits : 1);
  const bool duo = tc_use_duo(t.bn, kblocks);
  void* fn;
  if (duo) {
    fn = t.bn == 64 ? tc_fn<64, true>(amode, b_mn) : tc_fn<128, true>(amode, b_mn);
    G.set(fn, dim3((unsigned)(items < 2 * kNumSMs ? items : 2 * kNumSMs)), dim3(TC_THREADS), gp);
    G.smem = t.bn == 64 ? TcCfg<64, true>::SMEM : TcCfg<128, true>::SMEM;
    rc = t.bn == 64 ? tc_attr<64, true>(amode, b_mn) : tc_attr<128, true>(amode, b_mn);
  } else {
    fn = t.bn == 64 ? tc_fn<64>(amode, b_mn) : t.bn == 128 ? tc_fn<128>(amode, b_mn) : tc_fn<256>(amode, b_mn);

    G.set(fn, dim3((unsigned)(items < kNumSMs ? items : kNumSMs)), dim3(TC_THREADS), gp);
    G.smem = t.bn == 64 ? TcCfg<64>::SMEM : t.bn == 128 ? TcCfg<128>::SMEM : TcCfg<256>::SMEM;
    rc = t.bn == 64 ? tc_attr<64>(amode, b_mn) : t.bn == 128 ? tc_attr<128>(amode, b_mn) : tc_attr<256>(amode, b_mn);
  }
  if (rc) return rc;
  // a possible gradient-region output (Builder::nvls_fuse): the single-CTA epilogue-reduction
  // instantiation of the same tile width (a DUO launch is retargeted to it)
  if (raw == nullptr && c->nv_local != nullptr) {
    G.fn_red = t.bn == 64 ? tc_fn_red<64>(amode, b_mn) : t.bn == 128 ? tc_fn_red<128>(amode, b_mn)
                                                         : tc_fn_red<256>(amode, b_mn);
    rc = t.bn == 64 ? tc_attr_red<64>(amode, b_mn) : t.bn == 128 ? tc_attr_red<128>(amode, b_mn)
                                                   : tc_attr_red<256>(amode, b_mn);
    if (rc) return rc;
    G.red_grid = (unsigned)(items < kNumSMs ? items : kNumSMs);
    G.red_smem = t.bn == 64 ? TcCfg<64>::SMEM : t.bn == 128 ? TcCfg<128>::SMEM : TcCfg<256>::SMEM;
  }
  if (t.splits > 1) {
    SplitReduceParams r{};
    r.ds = ds;
    r.ws = ws;
    r.n = M * N;
    r.splits = t.splits;
    r.a = na;
    r.b = nb;
    if (bias) {
      r.bias = *bias;
      r.has_bias = 1;
      r.ncols = N;
    }

    if (raw != nullptr) {            // reduce into scratch: a private, never-published Out
      r.out = Out{};
      r.out.buf[0] = raw;
    } else {
      r.out = out;
    }
    L[*nL].tc_dest = raw == nullptr ? 2 : 0;
    L[(*nL)++].set((void*)k_splitk_reduce, grid_for(M * N / 4 + 1), dim3(256), r);
  }
  return COEX_OK;
}

// fp32 [rows][K] -> bf16 [rows][pitch(K)] (flattened k_cvt_bf16, one operand)
void cvt_rows_launch(DevState* ds, In src, void* dst, int64_t rows, int64_t K, Launch* L) {
  CvtParams q{};
  q.ds = ds; q.src[0] = src; q.rows[0] = rows; q.K = K; q.ld = bf16_pitch(K); q.trans[0] = 0;
  q.dst[0] = (__nv_bfloat16*)dst;
  const int64_t gx = (rows * q.ld / 8 + 255) / 256;
  L->set((void*)k_cvt_bf16, dim3((unsigned)(gx < kNumSMs * 16 ? (gx < 1 ? 1 : gx) : kNumSMs * 16), 1), dim3(256), q);
}

// fp32 NHWC x -> zero-bordered bf16 copy (implicit-GEMM gather source)
void cvt_pad_launch(DevState* ds, In src, void* dst, int64_t N, int64_t H, int64_t W, int64_t C, int P, Launch* L) {
  PadCvtParams q{};
  q.ds = ds; q.x = src; q.dst = (__nv_bfloat16*)dst; q.N = N; q.H = (int)H; q.W = (int)W; q.C = (int)C; q.P = P;
  L->set((void*)k_cvt_pad_bf16, grid_for(N * H * W * C / 8), dim3(256), q);
}

// COEX_IMPLICIT: bitmask of implicit-GEMM convolution paths (1 conv2d, 2 conv2d_dw, 4 conv2d_t);
// default all on.
int implicit_mask() {
  static int m = -1;
  if (m < 0) {
    const char* e = getenv("COEX_IMPLICIT");
    m = e ? atoi(e) : 7;
  }
  return m;
}

// smallest output pixel grid (per image) that takes the implicit-GEMM convolution paths
// (COEX_IMPLICIT_MINPIX; conv2d_t uses a quarter of it on its input grid)
int64_t implicit_minpix() {
  static int64_t m = -1;
  if (m < 0) {
    const char* e = getenv("COEX_IMPLICIT_MINPIX");
    m = e ? atoll(e) : 256;
  }
  return m;
}

// smallest conv2d_t input grid (per image) on the sub-pixel implicit path (COEX_CONVT_MINPIX)
int64_t convt_minpix() {
  static int64_t m = -1;
  if (m < 0) {
    const char* e = getenv("COEX_CONVT_MINPIX");
    m = e ? atoll(e) : implicit_minpix() / 4;
  }
  return m;
}

// narrowest conv2d_t output (channels) that takes the sub-pixel implicit path (COEX_CONVT_MINF)
int64_t convt_min_f() {
  static int64_t m = -1;
  if (m < 0) {
    const char* e = getenv("COEX_CONVT_MINF");
    m = e ? atoll(e) : 32;
  }
  return m;
}

// few-channel im2col specialisations (image layers)
void* im2col_small_fn(int64_t C, int64_t k) {
  if (C == 3 && k == 4) return (void*)k_im2col_small<3, 4>;
  if (C == 3 && k == 7) return (void*)k_im2col_small<3, 7>;
  if (C == 3 && k == 3) return (void*)k_im2col_small<3, 3>;
  return nullptr;
}

// COEX_CE_STREAM=1: the streaming two-pass cross-entropy for wide rows instead of the
// shared-memory-staged one (measured slower on C4: 2.34 vs 1.32 ms per step -- the second pass
// re-reads rows that no longer fit in L2 with ~600 rows in flight; kept for A/B)
bool ce_stream() {
  const char* e = getenv("COEX_CE_STREAM");
  return e && e[0] == '1';
}

// COEX_COL_BULK=0 keeps the register-pipelined column statistics (A/B measurement)
bool col_bulk() {
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("COEX_COL_BULK");
    v = (e && e[0] == '0') ? 0 : 1;
  }
  return v == 1;
}

struct Carve {
  char* base;
  size_t off = 0;
  explicit Carve(char* b) : base(b) {}
  void* take(size_t bytes) {
    off = (off + 255) & ~(size_t)255;
    void* r = base ? base + off : nullptr;
    off += bytes < 16 ? 16 : bytes;
    return r;
  }
};

Out private_out(void* buf) {
  Out o{};
  o.buf[0] = buf;
  return o;
}

// Extension ops (conv family, batch-norm family): up to 5 launches per op.  Two workspaces:
// s.ws = scratch, fully rewritten by the op before it is read (im2col / bf16 operand copies,
// split-K partials, cols) -- shared by every op of a program (ops run in stream order); s.pz =
// the op's own persistent state (fp64 atomic accumulators, block counters: zero at rest, reset
// by the op itself).  With s.ws == nullptr only the sizes are computed (*ws_bytes, *pz_bytes).
template <typename T>
int build_xop_t(coex_ctx* c, const OpSpec& s, Launch* L, int* nL, size_t* ws_bytes, size_t* pz_bytes) {
  Carve cv(s.ws);
  Carve pv(s.pz);
  const bool build = s.ws != nullptr;
  const bool bf16 = c->prec == COEX_BF16;
  const size_t es = sizeof(T);
  *nL = 0;
  const int64_t k = s.attr_dims[0], st = s.attr_dims[1], pd = s.attr_dims[2];
  switch (s.kind) {
    case COEX_CONV2D: {
      const int64_t N = s.in_shape[0][0], H = s.in_shape[0][1], W = s.in_shape[0][2], C = s.in_shape[0][3];
      const int64_t Ho = s.out_shape[1], Wo = s.out_shape[2], F = s.out_shape[3];
      const int64_t M = N * Ho * Wo, Kc = k * k * C;
      Im2colParams ip{};
      ip.ds = s.ds; ip.x = s.in[0];
      ip.N = N; ip.H = H; ip.W = W; ip.C = C; ip.Ho = Ho; ip.Wo = Wo;
      ip.k = (int)k; ip.s = (int)st; ip.p = (int)pd;
      int bw, bh, bnn;
      // implicit GEMM pays off on the larger pixel grids (measured per op on the C2 shapes:
      // tools/cmp_implicit.py); small grids keep the materialised im2col operand
      if (bf16 && (implicit_mask() & 1) && C % 64 == 0 && st <= 2 && Ho * Wo >= implicit_minpix() &&
          conv_blocks(Ho, Wo, 128, &bw, &bh, &bnn)) {
        // implicit GEMM: A gathered from bf16 NHWC x by 4-D TMA boxes (no im2col matrix)
        const TcPlan t = tc_plan(M, F, Kc, true);
        const int P = (int)pd;
        void* X = cv.take((size_t)N * (H + 2 * P) * (W + 2 * P) * C * 2);
        void* B = cv.take((size_t)Kc * bf16_pitch(F) * 2);
        float* ws = t.splits > 1 ? (float*)cv.take((size_t)t.splits * M * F * 4) : nullptr;
        if (!build) break;
        cvt_pad_launch(s.ds, s.in[0], X, N, H, W, C, P, &L[(*nL)++]);
        cvt_rows_launch(s.ds, s.in[1], B, Kc, F, &L[(*nL)++]);
        TcConv g{};
        g.C = (int)C; g.taps_x = (int)k; g.s = (int)st; g.Hg = (int)Ho; g.Wg = (int)Wo;
        g.bw = bw; g.bh = bh; g.bn = bnn; g.phases = 1; g.off_y[0] = g.off_x[0] = 0;   // padding is in the copy
        CUtensorMap map;
        int rc = make_tmap_conv(&map, X, N, H + 2 * P, W + 2 * P, C, (int)st, bw, bh, bnn);
        if (rc) return rc;
        return tc_gemm_launches(c, s.ds, nullptr, B, M, F, Kc, t, s.in[0], s.in[1], s.out, nullptr, ws, L, nL, 2, true,
                                &g, &map);
      }
      if (bf16) {
        const TcPlan t = tc_plan(M, F, Kc, true);
        void* A = cv.take((size_t)M * bf16_pitch(Kc) * 2);
        void* B = cv.take((size_t)Kc * bf16_pitch(F) * 2);       // w as stored: [Kc][F], MN-major B
        float* ws = t.splits > 1 ? (float*)cv.take((size_t)t.splits * M * F * 4) : nullptr;
        if (!build) break;
        ip.dst = A; ip.ld = bf16_pitch(Kc); ip.trans = 0;
        if (C % 8 == 0 && M < (1ll << 31))
          L[(*nL)++].set((void*)k_im2col_bf16v, blocks_for_rows(M, Kc / 8), dim3(256), ip);
        else if (M < (1ll << 31))
          L[(*nL)++].set(im2col_small_fn(C, k) ? im2col_small_fn(C, k) : (void*)k_im2col_bf16s,
                         im2col_small_fn(C, k) ? grid_for(M) : grid_for(M * ip.ld / 8), dim3(256), ip);
        else
          L[(*nL)++].set((void*)k_im2col<float, __nv_bfloat16>, grid_for(M * ip.ld / 8), dim3(256), ip);
        CvtParams q{};
        q.ds = s.ds; q.src[0] = s.in[1]; q.rows[0] = Kc; q.K = F; q.ld = bf16_pitch(F); q.trans[0] = 0;
        q.dst[0] = (__nv_bfloat16*)B;
        const int64_t gx = (Kc * q.ld / 8 + 255) / 256;
        L[(*nL)++].set((void*)k_cvt_bf16, dim3((unsigned)(gx < kNumSMs * 16 ? (gx < 1 ? 1 : gx) : kNumSMs * 16), 1),
                       dim3(256), q);
        return tc_gemm_launches(c, s.ds, A, B, M, F, Kc, t, s.in[0], s.in[1], s.out, nullptr, ws, L, nL, 0, true);
      }
      void* A = cv.take((size_t)M * Kc * es);
      if (!build) break;
      ip.dst = A; ip.ld = Kc; ip.trans = 0;
      L[(*nL)++].set((void*)k_im2col<T, T>, grid_for(M * Kc), dim3(256), ip);
      MatmulParams mp{};
      mp.ds = s.ds; mp.a = In{A, nullptr, nullptr}; mp.b = s.in[1];
      mp.M = M; mp.K = Kc; mp.N = F; mp.lda = Kc; mp.ldb = F; mp.out = s.out;
      simt_matmul_launch<T>(c, mp, &L[(*nL)++]);
      return COEX_OK;
    }
    case COEX_CONV2D_T: case COEX_CONV2D_DX: {
      // conv2d_dx(dy, w, x) is conv2d_t(dy, w) onto x's geometry (out_shape): the output may
      // exceed the transposed-convolution size by up to s-1 rows / columns (no window
      // reached them in the forward pass) -- those stay zero; only the exact geometry takes
      // the sub-pixel implicit path
      const int64_t N = s.in_shape[0][0], H = s.in_shape[0][1], W = s.in_shape[0][2], C = s.in_shape[0][3];
      const int64_t Ho = s.out_shape[1], Wo = s.out_shape[2], F = s.out_shape[3];
      const int64_t M = N * H * W, Nc = k * k * F;
      int bw, bh, bnn;
      if (bf16 && (implicit_mask() & 4) && C % 64 == 0 && st >= 1 && k % st == 0 && k - 2 * pd == st &&
          Ho == (H - 1) * st - 2 * pd + k && Wo == (W - 1) * st - 2 * pd + k &&
          H * W >= convt_minpix() && F >= convt_min_f() && conv_blocks(H, W, 128, &bw, &bh, &bnn)) {
        // sub-pixel decomposition: st*st stride-1 implicit GEMMs (one per output phase) over the
        // bf16 NHWC input, epilogue scattering straight into the output -- no cols / col2im
        const int Tp = (int)(k / st), phases = (int)(st * st);
        const int64_t Kr = (int64_t)Tp * Tp * C;
        const TcPlan t = tc_plan(M * phases, F, Kr, false);
        int lo = 0, hi = 0;                          // offset range over the phases
        for (int ph = 0; ph < phases; ++ph) {
          const int py = ph / (int)st, ky0 = (py + (int)pd) % (int)st;
          const int o = (py + (int)pd - ky0) / (int)st - (Tp - 1);
          lo = o < lo ? o : lo;
          hi = o + Tp - 1 > hi ? o + Tp - 1 : hi;
        }
        const int Pp = -lo > hi ? -lo : hi;          // zero border of the bf16 copy
        void* X = cv.take((size_t)N * (H + 2 * Pp) * (W + 2 * Pp) * C * 2);
        void* B = cv.take((size_t)phases * Kr * bf16_pitch(F) * 2);
        if (!build) break;
        cvt_pad_launch(s.ds, s.in[0], X, N, H, W, C, Pp, &L[(*nL)++]);
        WPhaseParams wp{};
        wp.ds = s.ds; wp.w = s.in[1]; wp.dst = (__nv_bfloat16*)B; wp.ld = bf16_pitch(F);
        wp.k = (int)k; wp.so = (int)st; wp.pad = (int)pd; wp.T = Tp; wp.C = (int)C; wp.F = (int)F;
        L[(*nL)++].set((void*)k_convt_wphase, grid_for(phases * Kr * wp.ld), dim3(256), wp);
        TcConv g{};
        g.C = (int)C; g.taps_x = Tp; g.s = 1; g.Hg = (int)H; g.Wg = (int)W; g.bw = bw; g.bh = bh; g.bn = bnn;
        g.phases = phases; g.so = (int)st; g.Ho = (int)Ho; g.Wo = (int)Wo; g.b_rows = Kr; g.pad = (int)pd;
        g.bord = Pp;
        for (int ph = 0; ph < phases; ++ph) {
          const int py = ph / (int)st, px = ph % (int)st;
          const int ky0 = (py + (int)pd) % (int)st, kx0 = (px + (int)pd) % (int)st;
          g.off_y[ph] = (py + (int)pd - ky0) / (int)st - (Tp - 1) + Pp;
          g.off_x[ph] = (px + (int)pd - kx0) / (int)st - (Tp - 1) + Pp;
        }
        CUtensorMap map;
        int rc = make_tmap_conv(&map, X, N, H + 2 * Pp, W + 2 * Pp, C, 1, bw, bh, bnn);
        if (rc) return rc;
        return tc_gemm_launches(c, s.ds, nullptr, B, M, F, Kr, t, s.in[0], s.in[1], s.out, nullptr, nullptr, L, nL, 2,
                                true, &g, &map);
      }
      Col2imParams cp{};
      cp.ds = s.ds; cp.N = N; cp.H = H; cp.W = W; cp.F = F; cp.Ho = Ho; cp.Wo = Wo;
      cp.k = (int)k; cp.s = (int)st; cp.p = (int)pd; cp.a = s.in[0]; cp.b = s.in[1]; cp.out = s.out;
      if (bf16) {
        const TcPlan t = tc_plan(M, Nc, C, true);
        void* A = cv.take((size_t)M * bf16_pitch(C) * 2);
        void* B = cv.take((size_t)Nc * bf16_pitch(C) * 2);
        float* cols = (float*)cv.take((size_t)M * Nc * 4);
        float* ws = t.splits > 1 ? (float*)cv.take((size_t)t.splits * M * Nc * 4) : nullptr;
        if (!build) break;
        CvtParams q{};
        q.ds = s.ds; q.src[0] = s.in[0]; q.src[1] = s.in[1]; q.rows[0] = M; q.rows[1] = Nc; q.K = C;
        q.ld = bf16_pitch(C); q.trans[0] = 0; q.trans[1] = 0;
        q.dst[0] = (__nv_bfloat16*)A; q.dst[1] = (__nv_bfloat16*)B;
        const int64_t rows_max = M > Nc ? M : Nc;
        L[(*nL)++].set((void*)k_cvt_bf16, dim3((unsigned)(rows_max < kNumSMs * 16 ? rows_max : kNumSMs * 16), 2),
                       dim3(256), q);
        int rc = tc_gemm_launches(c, s.ds, A, B, M, Nc, C, t, s.in[0], s.in[1], s.out, cols, ws, L, nL);
        if (rc) return rc;
        cp.cols = cols;
        if (F % 4 == 0 && N * Ho * Wo < (1ll << 31))
          L[(*nL)++].set((void*)k_col2im_v<4>, blocks_for_rows(N * Ho * Wo, F / 4), dim3(256), cp);
        else if (N * Ho * Wo < (1ll << 31))
          L[(*nL)++].set(F == 3 ? (void*)k_col2im_px<3> : (void*)k_col2im_v<1>,
                         F == 3 ? grid_for(N * Ho * Wo) : blocks_for_rows(N * Ho * Wo, F), dim3(256), cp);
        else
          L[(*nL)++].set((void*)k_col2im<float, float>, grid_for(N * Ho * Wo * F), dim3(256), cp);
        return COEX_OK;
      }
      void* cols = cv.take((size_t)M * Nc * es);
      if (!build) break;
      MatmulParams mp{};
      mp.ds = s.ds; mp.a = s.in[0]; mp.b = s.in[1]; mp.trans_b = 1;
      mp.M = M; mp.K = C; mp.N = Nc; mp.lda = C; mp.ldb = C; mp.out = private_out(cols);
      simt_matmul_launch<T>(c, mp, &L[(*nL)++]);
      cp.cols = cols;
      L[(*nL)++].set((void*)k_col2im<T, T>, grid_for(N * Ho * Wo * F), dim3(256), cp);
      return COEX_OK;
    }
    case COEX_SLICE: case COEX_CONCAT: case COEX_SUM_AXIS: {
      if (!build) break;
      AxisParams ap{};
      ap.ds = s.ds; ap.a = s.in[0]; ap.b = s.nin > 1 ? s.in[1] : In{nullptr, nullptr, nullptr}; ap.out = s.out;
      const int ax = (int)s.attr_dims[0];
      ap.outer = 1; ap.inner = 1;
      for (int i = 0; i < ax; ++i) ap.outer *= s.in_shape[0][i];
      for (int i = ax + 1; i < s.in_ndim[0]; ++i) ap.inner *= s.in_shape[0][i];
      ap.A = s.in_shape[0][ax];
      ap.A2 = s.nin > 1 ? s.in_shape[1][ax] : 0;
      ap.start = s.attr_dims[1]; ap.length = s.attr_dims[2];
      ap.mode = s.kind == COEX_SLICE ? 0 : s.kind == COEX_CONCAT ? 1 : 2;
      const int64_t work = ap.mode == 2 ? ap.outer * ap.inner : numel_of(s.out_ndim, s.out_shape);
      L[(*nL)++].set(is_f64(c) ? (void*)k_axis<double> : (void*)k_axis<float>, grid_for(work < 1 ? 1 : work), dim3(256), ap);
      return COEX_OK;
    }
    case COEX_MAXPOOL: case COEX_MAXPOOL_GRAD: case COEX_AVGPOOL: case COEX_AVGPOOL_GRAD: case COEX_GLOBAL_AVGPOOL:
    case COEX_GLOBAL_AVGPOOL_GRAD: {
      // maxpool_grad: pass 1 stores every window's argmax tap (1 byte) in scratch, pass 2
      // gathers -- instead of recomputing up to ceil(k/s)^2 window maxima per input element
      unsigned char* idx = nullptr;
      if (s.kind == COEX_MAXPOOL_GRAD) idx = (unsigned char*)cv.take((size_t)numel_of(s.in_ndim[1], s.in_shape[1]));
      if (!build) break;
      PoolParams pp{};
      pp.ds = s.ds; pp.x = s.in[0]; pp.dy = s.nin > 1 ? s.in[1] : In{nullptr, nullptr, nullptr}; pp.out = s.out;
      pp.N = s.in_shape[0][0]; pp.H = s.in_shape[0][1]; pp.W = s.in_shape[0][2]; pp.C = s.in_shape[0][3];
      pp.k = (int)k; pp.s = (int)st; pp.p = (int)pd;
      const bool f64 = is_f64(c);
      void* fn = nullptr;
      int64_t work = pp.N * pp.H * pp.W * pp.C;
      switch (s.kind) {
        case COEX_MAXPOOL: case COEX_AVGPOOL:
          pp.Ho = s.out_shape[1]; pp.Wo = s.out_shape[2];
          work = pp.N * pp.Ho * pp.Wo * pp.C;
          fn = s.kind == COEX_MAXPOOL ? (f64 ? (void*)k_pool<double, 0> : (void*)k_pool<float, 0>)
                                      : (f64 ? (void*)k_pool<double, 2> : (void*)k_pool<float, 2>);
          break;
        case COEX_MAXPOOL_GRAD: case COEX_AVGPOOL_GRAD:
          pp.Ho = s.in_shape[1][1]; pp.Wo = s.in_shape[1][2];
          if (s.kind == COEX_MAXPOOL_GRAD) {
            pp.idx = idx;
            PoolParams p1 = pp;
            p1.out = Out{};
            L[(*nL)++].set(f64 ? (void*)k_pool<double, 6> : (void*)k_pool<float, 6>,
                           grid_for(pp.N * pp.Ho * pp.Wo * pp.C), dim3(256), p1);
          }
          fn = s.kind == COEX_MAXPOOL_GRAD ? (f64 ? (void*)k_pool<double, 1> : (void*)k_pool<float, 1>)
                                           : (f64 ? (void*)k_pool<double, 3> : (void*)k_pool<float, 3>);
          break;
        case COEX_GLOBAL_AVGPOOL:
          work = pp.N * pp.C;
          fn = f64 ? (void*)k_pool<double, 4> : (void*)k_pool<float, 4>;
          break;
        default:
          fn = f64 ? (void*)k_pool<double, 5> : (void*)k_pool<float, 5>;
      }
      L[(*nL)++].set(fn, grid_for(work), dim3(256), pp);
      return COEX_OK;
    }
    case COEX_CONV2D_DW: {
      const int64_t N = s.in_shape[0][0], H = s.in_shape[0][1], W = s.in_shape[0][2], C = s.in_shape[0][3];
      const int64_t Ho = s.in_shape[1][1], Wo = s.in_shape[1][2], F = s.in_shape[1][3];
      const int64_t P = N * Ho * Wo, Kc = k * k * C;
      Im2colParams ip{};
      ip.ds = s.ds; ip.x = s.in[0];
      ip.N = N; ip.H = H; ip.W = W; ip.C = C; ip.Ho = Ho; ip.Wo = Wo;
      ip.k = (int)k; ip.s = (int)st; ip.p = (int)pd;
      int bw, bh, bnn;
      if (bf16 && (implicit_mask() & 2) && C % 64 == 0 && st <= 2 && Ho * Wo >= implicit_minpix() &&
          conv_blocks(Ho, Wo, 64, &bw, &bh, &bnn)) {
        // implicit GEMM: A = im2col(x)^T gathered from bf16 NHWC x (64-pixel K blocks,
        // (tap, 64-channel) M halves, MN-major), B = dy [P][pitch(F)] MN-major
        const TcPlan t = tc_plan(Kc, F, P, true);
        const int Pd = (int)pd;
        void* X = cv.take((size_t)N * (H + 2 * Pd) * (W + 2 * Pd) * C * 2);
        void* B = cv.take((size_t)P * bf16_pitch(F) * 2);
        float* ws = t.splits > 1 ? (float*)cv.take((size_t)t.splits * Kc * F * 4) : nullptr;
        if (!build) break;
        cvt_pad_launch(s.ds, s.in[0], X, N, H, W, C, Pd, &L[(*nL)++]);
        cvt_rows_launch(s.ds, s.in[1], B, P, F, &L[(*nL)++]);
        TcConv g{};
        g.C = (int)C; g.taps_x = (int)k; g.s = (int)st; g.Hg = (int)Ho; g.Wg = (int)Wo;
        g.bw = bw; g.bh = bh; g.bn = bnn; g.phases = 1; g.off_y[0] = g.off_x[0] = 0;   // padding is in the copy
        CUtensorMap map;
        int rc = make_tmap_conv(&map, X, N, H + 2 * Pd, W + 2 * Pd, C, (int)st, bw, bh, bnn);
        if (rc) return rc;
        return tc_gemm_launches(c, s.ds, nullptr, B, Kc, F, P, t, s.in[0], s.in[1], s.out, nullptr, ws, L, nL, 3, true,
                                &g, &map);
      }
      if (bf16) {
        // dW = im2col(x)^T . dy with both operands MN-major: A = im2col(x) [P][pitch(Kc)],
        // B = dy [P][pitch(F)] in bf16 -- no transposition pass
        const TcPlan t = tc_plan(Kc, F, P, true);
        void* A = cv.take((size_t)P * bf16_pitch(Kc) * 2);
        void* B = cv.take((size_t)P * bf16_pitch(F) * 2);
        float* ws = t.splits > 1 ? (float*)cv.take((size_t)t.splits * Kc * F * 4) : nullptr;
        if (!build) break;
        ip.dst = A; ip.ld = bf16_pitch(Kc); ip.trans = 0;
        if (C % 8 == 0 && P < (1ll << 31))
          L[(*nL)++].set((void*)k_im2col_bf16v, blocks_for_rows(P, Kc / 8), dim3(256), ip);
        else if (P < (1ll << 31))
          L[(*nL)++].set(im2col_small_fn(C, k) ? im2col_small_fn(C, k) : (void*)k_im2col_bf16s,
                         im2col_small_fn(C, k) ? grid_for(P) : grid_for(P * ip.ld / 8), dim3(256), ip);
        else
          L[(*nL)++].set((void*)k_im2col<float, __nv_bfloat16>, grid_for(P * ip.ld / 8), dim3(256), ip);
        CvtParams q{};
        q.ds = s.ds; q.src[0] = s.in[1]; q.rows[0] = P; q.K = F; q.ld = bf16_pitch(F); q.trans[0] = 0;
        q.dst[0] = (__nv_bfloat16*)B;
        const int64_t units = P * q.ld / 8;
        const int64_t gx = (units + 255) / 256;
        L[(*nL)++].set((void*)k_cvt_bf16, dim3((unsigned)(gx < kNumSMs * 16 ? (gx < 1 ? 1 : gx) : kNumSMs * 16), 1),
                       dim3(256), q);
        return tc_gemm_launches(c, s.ds, A, B, Kc, F, P, t, s.in[0], s.in[1], s.out, nullptr, ws, L, nL, 1, true);
      }
      void* A = cv.take((size_t)P * Kc * es);
      if (!build) break;
      ip.dst = A; ip.ld = Kc; ip.trans = 0;
      L[(*nL)++].set((void*)k_im2col<T, T>, grid_for(P * Kc), dim3(256), ip);
      MatmulParams mp{};
      mp.ds = s.ds; mp.a = In{A, nullptr, nullptr}; mp.b = s.in[1]; mp.trans_a = 1;
      mp.M = Kc; mp.K = P; mp.N = F; mp.lda = Kc; mp.ldb = F; mp.out = s.out;
      simt_matmul_launch<T>(c, mp, &L[(*nL)++]);
      return COEX_OK;
    }
    case COEX_BATCHNORM: case COEX_BATCHNORM_DX: case COEX_BN_DGAMMA: case COEX_SUM_ROWS: case kBnBwdFused:
    case kBnAct: {
      const int64_t C = s.in_shape[0][s.in_ndim[0] - 1];
      const int64_t Rw = numel_of(s.in_ndim[0], s.in_shape[0]) / C;
      if (s.kind == COEX_SUM_ROWS && !is_f64(c) && C % 4 == 0 && (C > 1024 || (Rw >= 4096 && C >= 256))) {
        // tolerance modes, 4 | C: 16-byte column groups, row chunks sized to fill the SMs
        const int64_t gx = (C + 255) / 256;
        int64_t gy = 1;
        while (gy < 256 && gx * gy < kNumSMs * 4 && Rw / (gy * 2) >= 64) gy *= 2;
        RowParams rp{};
        rp.ds = s.ds; rp.x = s.in[0]; rp.rows = Rw; rp.d = C; rp.out = s.out;
        if (gy > 1) {
          rp.acc = (double*)pv.take((size_t)C * 8);
          rp.counter = (unsigned int*)pv.take(16);
        }
        if (!build) break;
        L[(*nL)++].set((void*)k_colsum_v4, dim3((unsigned)gx, (unsigned)gy), dim3(256), rp);
        return COEX_OK;
      }
      if (s.kind == COEX_SUM_ROWS && (C > 1024 || (!is_f64(c) && Rw >= 4096 && C >= 256))) {
        // wide rows / tall tolerance-mode sums: column-parallel sum over row chunks
        const int64_t gx = (C + 255) / 256;
        int64_t gy = 1;
        while (gy < 64 && gx * gy < kNumSMs * 4 && Rw / (gy * 2) >= 64) gy *= 2;
        RowParams rp{};
        rp.ds = s.ds; rp.x = s.in[0]; rp.rows = Rw; rp.d = C; rp.out = s.out;
        if (gy > 1) rp.acc = (double*)pv.take((size_t)C * 8);
        if (!build) break;
        L[(*nL)++].set(is_f64(c) ? (void*)k_colsum_wide<double> : (void*)k_colsum_wide<float>,
                       dim3((unsigned)gx, (unsigned)gy), dim3(256), rp);
        if (gy > 1) L[(*nL)++].set(is_f64(c) ? (void*)k_acc_out<double> : (void*)k_acc_out<float>, grid_for(C), dim3(256), rp);
        return COEX_OK;
      }
      const int64_t n = numel_of(s.in_ndim[0], s.in_shape[0]);
      const int64_t R = n / C;
      // partial blocks: enough to stream x at full bandwidth, few enough that the last block's
      // merge of G x C partials stays small
      // tolerance modes accumulate with fp64 atomics (no merge of per-block partials)
      const bool atomic = !is_f64(c);
      int64_t G = n / 16384;
      static int64_t gmin = -1;                      // COEX_COL_MINBLOCKS (tuning experiments)
      if (gmin < 0) {
        const char* e = getenv("COEX_COL_MINBLOCKS");
        gmin = e ? atoll(e) : 0;
      }
      if (atomic && G < gmin) G = gmin;
      if (!atomic && G > 32768 / C) G = 32768 / C;
      if (G > kNumSMs * 2) G = kNumSMs * 2;
      if (G > R) G = R;
      if (G < 1) G = 1;
      const bool v4 = !is_f64(c) && C % 4 == 0;
      const bool dy = s.kind == COEX_BATCHNORM_DX || s.kind == COEX_BN_DGAMMA || s.kind == kBnBwdFused;
      void* colfn;
      if (v4 && C <= 1024) colfn = dy ? (void*)k_colstats<float, 4, 1, true> : (void*)k_colstats<float, 4, 1, false>;
      else if (v4) colfn = dy ? (void*)k_colstats<float, 4, 2, true> : (void*)k_colstats<float, 4, 2, false>;
      else colfn = dy ? (void*)k_colstats<T, 1, kColMaxSlots, true> : (void*)k_colstats<T, 1, kColMaxSlots, false>;
      // bulk-streamed statistics (tolerance modes, C <= 1024): rows of 16 KB chunks
      size_t bulk_smem = 0;
      if (atomic && v4 && C <= 1024 && col_bulk()) {
        const int64_t rpi = 256 / (C / 4 < 256 ? C / 4 : 256);
        const int64_t cr = (4096 / C > rpi ? 4096 / C : rpi) / rpi * rpi;
        bulk_smem = (size_t)kColStages * cr * C * 4 * (dy ? 2 : 1);
        colfn = dy ? (void*)k_colstats<float, 4, 1, true, true> : (void*)k_colstats<float, 4, 1, false, true>;
        static int occ[2] = {0, 0};
        int& oc = occ[dy ? 1 : 0];
        if (oc == 0) {
          CK(cudaFuncSetAttribute(colfn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bulk_smem));
          if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&oc, colfn, 256, bulk_smem) != cudaSuccess || oc < 1) {
            cudaGetLastError();
            oc = 1;
          }
        }
        if (G > (int64_t)oc * kNumSMs) G = (int64_t)oc * kNumSMs;
      }
      ColStatsParams cp{};
      cp.ds = s.ds; cp.x = s.in[0]; cp.R = R; cp.C = C;
      if (bulk_smem) cp.chunk_rows = (int64_t)(bulk_smem / ((size_t)kColStages * C * 4 * (dy ? 2 : 1)));
      cp.atomic = atomic ? 1 : 0;
      cp.part = (double*)pv.take((size_t)(atomic ? kColReplicas : G) * C * 4 * 8);
      cp.stats = (double*)pv.take((size_t)C * 4 * 8);
      cp.counter = (unsigned int*)pv.take(16);
      cp.a = s.in[0];
      cp.b = s.nin > 1 ? s.in[1] : In{nullptr, nullptr, nullptr};
      // synchronised batch norm (data parallel: dp.py marks a row-sharded batchnorm /
      // batchnorm_dx / bn_dgamma with the GLOBAL row count): rank-local raw sums, an in-place
      // all-reduce of the [C][4] doubles over the context's communicator, finalisation over
      // the global batch, then the usual apply pass
      const bool sync = s.value > 0.0 && s.kind != COEX_SUM_ROWS && s.kind != kBnBwdFused;
      if (!build) break;
      if (sync) {
        if (c->comm == nullptr) return fail(COEX_BAD_ATTRS, "synchronised batch norm without a communicator");
        cp.raw = 1;
        cp.mode = s.kind == COEX_BATCHNORM || s.kind == kBnAct ? COL_BN
                  : s.kind == COEX_BN_DGAMMA ? COL_BN_DGAMMA : COL_BN_DX;
        if (s.kind == COEX_BN_DGAMMA) cp.dy = s.in[1];
        else if (s.kind == COEX_BATCHNORM_DX) cp.dy = s.in[2];
        cp.out = Out{};
        L[*nL].set(colfn, dim3((unsigned)G), dim3(256), cp);
        L[(*nL)++].smem = bulk_smem;
        L[(*nL)++].allreduce(cp.stats, 4 * C, true);
        BnFinalizeParams fp{};
        fp.ds = s.ds; fp.stats = cp.stats; fp.C = C; fp.R = s.value; fp.mode = cp.mode;
        fp.a = cp.a; fp.b = cp.b;
        if (s.kind == COEX_BN_DGAMMA) fp.out = s.out;
        L[(*nL)++].set(is_f64(c) ? (void*)k_bn_finalize<double> : (void*)k_bn_finalize<float>, dim3(1), dim3(256), fp);
        if (s.kind == COEX_BN_DGAMMA) return COEX_OK;
      }
      if (!sync && (s.kind == COEX_SUM_ROWS || s.kind == COEX_BN_DGAMMA)) {
        cp.mode = s.kind == COEX_SUM_ROWS ? COL_SUM_ROWS : COL_BN_DGAMMA;
        if (s.kind == COEX_BN_DGAMMA) cp.dy = s.in[1];
        cp.out = s.out;
        L[*nL].set(colfn, dim3((unsigned)G), dim3(256), cp);
        L[(*nL)++].smem = bulk_smem;
        return COEX_OK;
      }
      if (!sync) {
        cp.mode = (s.kind == COEX_BATCHNORM || s.kind == kBnAct) ? COL_BN : COL_BN_DX;
        if (s.kind == COEX_BATCHNORM_DX || s.kind == kBnBwdFused) cp.dy = s.in[2];
        cp.out = Out{};
        if (s.kind == kBnBwdFused) {
          cp.extra = 1;
          cp.out_g = s.out2;
          cp.out_b = s.out3;
        }
        L[*nL].set(colfn, dim3((unsigned)G), dim3(256), cp);
        L[(*nL)++].smem = bulk_smem;
      }
      BnApplyParams ap{};
      ap.ds = s.ds; ap.x = s.in[0]; ap.g = s.in[1]; ap.third = s.in[2]; ap.stats = cp.stats;
      ap.n = n; ap.C = C; ap.dx = s.kind != COEX_BATCHNORM && s.kind != kBnAct; ap.out = s.out;
      ap.act = s.kind == kBnAct ? (int)s.attr_dims[0] : -1;
      if (s.kind == kBnAct) ap.out2 = s.out2;
      if (v4) {
        L[*nL].set((void*)k_bn_apply_v4, grid_for(n / 4), dim3(256), ap);
        L[(*nL)++].smem = (size_t)3 * C * sizeof(float);
      } else {
        L[(*nL)++].set((void*)k_bn_apply<T>, grid_for(n), dim3(256), ap);
      }
      return COEX_OK;
    }
    case COEX_BMM: case COEX_BMM_NT: case COEX_BMM_TN: {
      const int64_t Bt = s.in_shape[0][0];
      const bool tn = s.kind == COEX_BMM_TN, nt = s.kind == COEX_BMM_NT;
      const int64_t M = s.out_shape[1], N = s.out_shape[2];
      const int64_t K = tn ? s.in_shape[0][1] : s.in_shape[0][2];
      if (bf16) {
        // operands converted as stored: A [B][M][K] (K-major) or [B][K][M] (tn: MN-major);
        // B [B][K][N] (MN-major) or [B][N][K] (nt: K-major); 3-D TMA maps, batch = grid items
        const TcPlan t = tc_plan(M * Bt, N, K, false);
        const int64_t arow = tn ? K : M, acol = tn ? M : K, brow = nt ? N : K, bcol = nt ? K : N;
        // shared bf16 copies from the plan (or a bf16 shadow written by the producer); eager:
        // private copies in the workspace
        void* A = s.in_shadow[0] ? s.in_shadow[0] : cv.take((size_t)Bt * arow * bf16_pitch(acol) * 2);
        void* B = s.in_shadow[1] ? s.in_shadow[1] : cv.take((size_t)Bt * brow * bf16_pitch(bcol) * 2);
        if (!build) break;
        if (!s.in_shadow[0] || s.in_conv[0]) cvt_rows_launch(s.ds, s.in[0], A, Bt * arow, acol, &L[(*nL)++]);
        if (!s.in_shadow[1] || s.in_conv[1]) cvt_rows_launch(s.ds, s.in[1], B, Bt * brow, bcol, &L[(*nL)++]);
        const int rc = tc_gemm_launches(c, s.ds, A, B, M, N, K, t, s.in[0], s.in[1], s.out, nullptr, nullptr, L, nL,
                                        tn ? 1 : 0, !nt, nullptr, nullptr, Bt);
        // planner-proven causal structure (attr dims[0]: 1 = only C's lower triangle is read,
        // 2 = A lower-triangular, 3 = A upper-triangular)
        if (rc == COEX_OK && s.attr_n >= 1 && s.attr_dims[0] > 0) {
          TcGemmParams* gp = (TcGemmParams*)L[*nL - 1].params;
          if (s.attr_dims[0] == 1) gp->tri_out = 1;
          else gp->tri_a = (int)s.attr_dims[0] - 1;
        }
        return rc;
      }
      if (!build) break;
      MatmulParams mp{};
      mp.ds = s.ds; mp.a = s.in[0]; mp.b = s.in[1]; mp.trans_a = tn; mp.trans_b = nt;
      mp.M = M; mp.N = N; mp.K = K;
      mp.lda = s.in_shape[0][2]; mp.ldb = s.in_shape[1][2];
      mp.sa = s.in_shape[0][1] * s.in_shape[0][2]; mp.sb = s.in_shape[1][1] * s.in_shape[1][2]; mp.sc = M * N;
      mp.out = s.out;
      simt_matmul_launch<T>(c, mp, &L[*nL]);
      L[(*nL)++].grid.y = (unsigned)Bt;
      return COEX_OK;
    }
    case COEX_EMBEDDING: case COEX_EMBEDDING_DW: case COEX_LAYERNORM: case COEX_LAYERNORM_DX: case COEX_LN_DGAMMA:
    case COEX_BIAS_ADD: case COEX_CAUSAL_SOFTMAX: case COEX_SOFTMAX_GRAD: case COEX_CROSS_ENTROPY:
    case COEX_CROSS_ENTROPY_GRAD: case COEX_REL_SKEW: case COEX_REL_UNSKEW: case kCeFused: case kLnBwdFused:
    case kSkewAdd: {
      RowParams rp{};
      rp.ds = s.ds; rp.x = s.in[0]; rp.y = s.in[1];
      rp.z = s.nin > 2 ? s.in[2] : In{nullptr, nullptr, nullptr};
      rp.out = s.out;
      rp.scale = s.value;
      rp.shadow = (__nv_bfloat16*)s.shadow;
      const int64_t xn = numel_of(s.in_ndim[0], s.in_shape[0]);
      const int64_t d = s.in_shape[0][s.in_ndim[0] - 1];
      auto warp_rows = [&](int64_t rows) {
        int64_t b = (rows + 7) / 8;
        return dim3((unsigned)(b < kNumSMs * 8 ? (b < 1 ? 1 : b) : kNumSMs * 8));
      };
      switch (s.kind) {
        case COEX_EMBEDDING: {
          if (!build) break;
          rp.d = s.in_shape[0][1]; rp.vocab = s.in_shape[0][0];
          rp.rows = numel_of(s.in_ndim[1], s.in_shape[1]);
          L[(*nL)++].set(is_f64(c) ? (void*)k_embed<double> : (void*)k_embed<float>, grid_for(rp.rows * rp.d), dim3(256), rp);
          return COEX_OK;
        }
        case COEX_EMBEDDING_DW: {
          if (!build) break;
          rp.d = s.out_shape[1]; rp.vocab = s.out_shape[0];
          rp.rows = numel_of(s.in_ndim[0], s.in_shape[0]);
          ZeroParams zp{};
          zp.ds = s.ds; zp.out = s.out; zp.out.npub = 0; zp.out.late = nullptr;
          zp.bytes = rp.vocab * rp.d * (int64_t)es; zp.a = s.in[0]; zp.b = s.in[1];
          L[(*nL)++].set((void*)k_zero, grid_for(zp.bytes / 16 + 1), dim3(256), zp);
          L[(*nL)++].set(is_f64(c) ? (void*)k_embed_dw<double> : (void*)k_embed_dw<float>, grid_for(rp.rows * rp.d),
                         dim3(256), rp);
          return COEX_OK;
        }
        case COEX_LAYERNORM: case COEX_LAYERNORM_DX: {
          if (!build) break;
          rp.d = d; rp.rows = xn / d;
          void* fn = s.kind == COEX_LAYERNORM ? (is_f64(c) ? (void*)k_layernorm<double, 0> : (void*)k_layernorm<float, 0>)
                                              : (is_f64(c) ? (void*)k_layernorm<double, 1> : (void*)k_layernorm<float, 1>);
          if (!is_f64(c) && d % 4 == 0 && d <= 1024) {   // 16-byte rows: PER float4 groups per lane
            const bool fw = s.kind == COEX_LAYERNORM;
            const int per = (int)((d / 4 + 31) / 32);
            fn = per <= 2 ? (fw ? (void*)k_layernorm_v4<0, 2> : (void*)k_layernorm_v4<1, 2>)
                 : per <= 4 ? (fw ? (void*)k_layernorm_v4<0, 4> : (void*)k_layernorm_v4<1, 4>)
                 : per <= 6 ? (fw ? (void*)k_layernorm_v4<0, 6> : (void*)k_layernorm_v4<1, 6>)
                            : (fw ? (void*)k_layernorm_v4<0, 8> : (void*)k_layernorm_v4<1, 8>);
            // 128-thread blocks (4 rows each): 7 resident per SM at 72 registers instead of 3 of
            // 256 threads -- fewer partial waves (ncu: 2.31 waves, 33 % warps active before)
            const int64_t b = (rp.rows + 3) / 4;
            L[(*nL)++].set(fn, dim3((unsigned)(b < kNumSMs * 16 ? (b < 1 ? 1 : b) : kNumSMs * 16)), dim3(128), rp);
            return COEX_OK;
          }
          L[(*nL)++].set(fn, warp_rows(rp.rows), dim3(256), rp);
          return COEX_OK;
        }
        case kLnBwdFused: {
          rp.acc = (double*)pv.take((size_t)2 * kColReplicas * d * 8);
          rp.counter = (unsigned int*)pv.take(16);
          if (!build) break;
          if (is_f64(c) || d % 4 || d > 1024) return fail(COEX_INVALID, "fused layernorm backward: fp32 rows, 4 | d <= 1024");
          rp.d = d; rp.rows = xn / d;
          LnBwdParams lp{};
          lp.p = rp;
          lp.out_g = s.out2;
          lp.out_b = s.out3;
          const int per = (int)((d / 4 + 31) / 32);
          void* fn = per <= 2 ? (void*)k_ln_bwd_v4<2> : per <= 4 ? (void*)k_ln_bwd_v4<4>
                   : per <= 6 ? (void*)k_ln_bwd_v4<6> : (void*)k_ln_bwd_v4<8>;
          // 128-thread blocks: at ~135 registers three are resident per SM (one of 256 threads
          // before), one wave of blocks
          int64_t blocks = (rp.rows + 3) / 4;
          if (blocks > kNumSMs * 3) blocks = kNumSMs * 3;
          L[(*nL)++].set(fn, dim3((unsigned)(blocks < 1 ? 1 : blocks)), dim3(128), lp);
          return COEX_OK;
        }
        case COEX_LN_DGAMMA: {
          rp.acc = (double*)pv.take((size_t)kColReplicas * d * 8);
          rp.counter = (unsigned int*)pv.take(16);
          if (!build) break;
          rp.d = d; rp.rows = xn / d;
          L[(*nL)++].set(is_f64(c) ? (void*)k_ln_dgamma<double> : (void*)k_ln_dgamma<float>, warp_rows(rp.rows / 4),
                         dim3(256), rp);
          return COEX_OK;
        }
        case COEX_BIAS_ADD: {
          if (!build) break;
          rp.d = d; rp.rows = xn / d;
          L[(*nL)++].set(is_f64(c) ? (void*)k_bias_add<double> : (void*)k_bias_add<float>,
                         grid_for(sizeof(T) == 4 && d % 4 == 0 ? xn / 4 : xn), dim3(256), rp);
          return COEX_OK;
        }
        case COEX_CAUSAL_SOFTMAX: case COEX_SOFTMAX_GRAD: {
          if (!build) break;
          rp.d = d; rp.rows = xn / d; rp.T = (int)d;
          void* fn = s.kind == COEX_CAUSAL_SOFTMAX ? (is_f64(c) ? (void*)k_causal_softmax<double> : (void*)k_causal_softmax<float>)
                                                   : (is_f64(c) ? (void*)k_softmax_grad<double> : (void*)k_softmax_grad<float>);
          L[(*nL)++].set(fn, warp_rows(rp.rows), dim3(256), rp);
          return COEX_OK;
        }
        case kSkewAdd: {
          if (!build) break;
          if (is_f64(c) || d % 4) return fail(COEX_INVALID, "fused rel_skew + add: fp32 rows, 4 | T");
          rp.d = d; rp.rows = xn / d;
          L[(*nL)++].set((void*)k_rel_skew_v4<0, true>, warp_rows(rp.rows), dim3(256), rp);
          return COEX_OK;
        }
        case COEX_REL_SKEW: case COEX_REL_UNSKEW: {
          if (!build) break;
          if (!is_f64(c) && d % 4 == 0) {           // 16-byte row stores
            rp.d = d; rp.rows = xn / d;
            L[(*nL)++].set(s.kind == COEX_REL_SKEW ? (void*)k_rel_skew_v4<0, false> : (void*)k_rel_skew_v4<1, false>,
                           warp_rows(rp.rows), dim3(256), rp);
            return COEX_OK;
          }
          rp.d = d; rp.rows = xn / d;
          void* fn = s.kind == COEX_REL_SKEW ? (is_f64(c) ? (void*)k_rel_skew<double, 0> : (void*)k_rel_skew<float, 0>)
                                             : (is_f64(c) ? (void*)k_rel_skew<double, 1> : (void*)k_rel_skew<float, 1>);
          L[(*nL)++].set(fn, warp_rows(rp.rows), dim3(256), rp);
          return COEX_OK;
        }
        case kCeFused: {   // loss + gradient (+ bf16 shadow) in one pass over the logits
          const int64_t R = s.in_shape[0][0], V = s.in_shape[0][1];
          rp.acc = (double*)pv.take((size_t)R * 8);
          rp.counter = (unsigned int*)pv.take(16);
          if (!build) break;
          rp.d = V; rp.rows = R; rp.vocab = V;
          rp.spitch = (V + 7) / 8 * 8;
          rp.skip_f32 = (int)s.attr_dims[0];
          rp.out2 = s.out2;
          const size_t smem = (size_t)V * 4;
          if (is_f64(c) || smem > 220 * 1024) {      // f64 parity / very wide rows: two passes
            rp.shadow = nullptr;
            rp.skip_f32 = 0;
            RowParams lp = rp;
            lp.out = s.out2;
            L[(*nL)++].set(is_f64(c) ? (void*)k_cross_entropy<double, 0> : (void*)k_cross_entropy<float, 0>,
                           dim3((unsigned)(R < kNumSMs * 8 ? R : kNumSMs * 8)), dim3(256), lp);
            L[(*nL)++].set(is_f64(c) ? (void*)k_cross_entropy<double, 1> : (void*)k_cross_entropy<float, 1>,
                           dim3((unsigned)(R < kNumSMs * 8 ? R : kNumSMs * 8)), dim3(256), rp);
            return COEX_OK;
          }
          if (V >= 8192 && ce_stream()) {             // wide vocabulary: streaming two-pass kernel
            L[(*nL)++].set((void*)k_ce_stream, dim3((unsigned)(R < kNumSMs * 4 ? R : kNumSMs * 4)), dim3(256), rp);
            return COEX_OK;
          }
          const bool wide = V >= 8192;
          // wide rows whose halves fit 110 KB: a CTA pair per row, two pairs' CTAs per SM
          // (COEX_CE_PAIR=0: one 1024-thread CTA per row)
          const char* cpe = getenv("COEX_CE_PAIR");
          if (wide && (size_t)((V + 1) / 2 + 8) * 4 <= 110 * 1024 && !(cpe && cpe[0] == '0')) {
            static bool pair_attr = false;
            if (!pair_attr) {
              CK(cudaFuncSetAttribute((void*)k_ce_pair<512>, cudaFuncAttributeMaxDynamicSharedMemorySize, 110 * 1024));
              pair_attr = true;
            }
            const int64_t pairs = R < kNumSMs ? R : kNumSMs;
            L[*nL].set((void*)k_ce_pair<512>, dim3((unsigned)(2 * pairs)), dim3(512), rp);
            L[(*nL)++].smem = (size_t)((V + 1) / 2 + 8) * 4;
            return COEX_OK;
          }
          void* fn = wide ? (void*)k_ce_fused<1024> : (void*)k_ce_fused<128>;
          static bool attr_set = false;
          if (!attr_set) {
            CK(cudaFuncSetAttribute((void*)k_ce_fused<1024>, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024));
            CK(cudaFuncSetAttribute((void*)k_ce_fused<128>, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024));
            attr_set = true;
          }
          const int64_t per_sm = wide ? 1 : 8;
          L[*nL].set(fn, dim3((unsigned)(R < kNumSMs * per_sm ? R : kNumSMs * per_sm)), dim3(wide ? 1024 : 128), rp);
          L[(*nL)++].smem = smem;
          return COEX_OK;
        }
        default: {   // cross-entropy (loss / gradient)
          const int64_t R = s.in_shape[0][0];
          if (s.kind == COEX_CROSS_ENTROPY) {
            rp.acc = (double*)pv.take((size_t)R * 8);
            rp.counter = (unsigned int*)pv.take(16);
          }
          if (!build) break;
          rp.d = s.in_shape[0][1]; rp.rows = R; rp.vocab = rp.d;
          void* fn = s.kind == COEX_CROSS_ENTROPY ? (is_f64(c) ? (void*)k_cross_entropy<double, 0> : (void*)k_cross_entropy<float, 0>)
                                                  : (is_f64(c) ? (void*)k_cross_entropy<double, 1> : (void*)k_cross_entropy<float, 1>);
          L[(*nL)++].set(fn, dim3((unsigned)(R < kNumSMs * 8 ? R : kNumSMs * 8)), dim3(256), rp);
          return COEX_OK;
        }
      }
      break;
    }
    default:
      return fail(COEX_BAD_ATTRS, "op kind has no extension kernel");
  }
  *ws_bytes = cv.off;
  if (pz_bytes) *pz_bytes = pv.off;
  return COEX_OK;
}

int build_xop(coex_ctx* c, const OpSpec& s, Launch* L, int* nL, size_t* ws_bytes, size_t* pz_bytes = nullptr) {
  return is_f64(c) ? build_xop_t<double>(c, s, L, nL, ws_bytes, pz_bytes)
                   : build_xop_t<float>(c, s, L, nL, ws_bytes, pz_bytes);
}
constexpr int kMaxLaunches = 6;

bool needs_scratch(const coex_ctx* c, int kind) {
  return (c->prec == COEX_BF16 || tf32_path(c)) && kind == COEX_MATMUL;
}

// bf16 copies of the MatMul operands as stored ([rows][pitch(cols)]; K- or MN-major use);
// 3xTF32: hi / lo fp32 planes of the K-major operands (A [M][K], B^T [N][K])
void scratch_bytes(const coex_ctx* c, const OpSpec& s, size_t* a, size_t* b) {
  const int64_t ra = s.in_shape[0][0], ca = s.in_shape[0][1], rb = s.in_shape[1][0], cb = s.in_shape[1][1];
  if (tf32_path(c)) {
    const int64_t M = s.trans_a ? ca : ra, K = s.trans_a ? ra : ca, N = s.trans_b ? rb : cb;
    *a = (size_t)2 * (M > 0 ? M : 1) * tf32_pitch(K > 0 ? K : 1) * 4;
    *b = (size_t)2 * (N > 0 ? N : 1) * tf32_pitch(K > 0 ? K : 1) * 4;
    return;
  }
  const size_t a1 = (size_t)(ra > 0 ? ra : 1) * bf16_pitch(ca > 0 ? ca : 1) * 2;   // as stored
  const size_t a2 = (size_t)(ca > 0 ? ca : 1) * bf16_pitch(ra > 0 ? ra : 1) * 2;   // transposed
  const size_t b1 = (size_t)(rb > 0 ? rb : 1) * bf16_pitch(cb > 0 ? cb : 1) * 2;
  const size_t b2 = (size_t)(cb > 0 ? cb : 1) * bf16_pitch(rb > 0 ? rb : 1) * 2;
  *a = a1 > a2 ? a1 : a2;
  *b = b1 > b2 ? b1 : b2;
}

// One op -> its launches (bf16 MatMul = operand conversion + tcgen05 GEMM; extension ops
// up to kMaxLaunches, see build_xop).
int build_launches(coex_ctx* c, const OpSpec& s, Launch* L, int* nL) {
  if (is_ext_compute(s.kind)) {
    size_t wb = 0;
    return build_xop(c, s, L, nL, &wb);
  }
  if (!needs_scratch(c, s.kind)) {
    *nL = 1;
    return build_launch(c, s, L);
  }
  const int64_t M = s.trans_a ? s.in_shape[0][1] : s.in_shape[0][0];
  const int64_t K = s.trans_a ? s.in_shape[0][0] : s.in_shape[0][1];
  const int64_t N = s.trans_b ? s.in_shape[1][0] : s.in_shape[1][1];
  if (tf32_path(c)) return tf32_gemm_launches(c, s, M, N, K, L, nL);
  // operands are converted as stored (no transposition): A [M][K] -> K-major, A folded from a
  // transpose ([K][M]) -> MN-major; B [K][N] -> MN-major, B folded ([N][K]) -> K-major.  A
  // conversion is skipped when an earlier GEMM of the pass already made this copy.
  // conversion flag 2 (planner: narrow operand): transposed conversion into a K-major copy.
  // Eager calls use the same narrow rule.
  int ca = s.in_conv[0], cb = s.in_conv[1];
  if (s.ws == nullptr && ca == 1 && cb == 1) {     // eager: no plan flags
    if (s.trans_a && M < 64) ca = 2;
    if (!s.trans_b && N < 64) cb = 2;
  }
  const bool a_mn = s.trans_a && ca != 2, b_mn = !s.trans_b && cb != 2;
  *nL = 0;
  if (ca == 1 && cb == 1) {                         // both operands as stored: one launch
    CvtParams q{};
    q.ds = s.ds; q.src[0] = s.in[0]; q.src[1] = s.in[1];
    q.rows[0] = s.in_shape[0][0]; q.K = s.in_shape[0][1]; q.ld = bf16_pitch(q.K);
    q.rows[1] = s.in_shape[1][0]; q.Kb = s.in_shape[1][1]; q.ldb = bf16_pitch(q.Kb); q.own_b = 1;
    q.dst[0] = (__nv_bfloat16*)s.scratch[0]; q.dst[1] = (__nv_bfloat16*)s.scratch[1];
    const int64_t ga = (q.rows[0] * q.ld / 8 + 255) / 256, gb = (q.rows[1] * q.ldb / 8 + 255) / 256;
    int64_t gx = ga > gb ? ga : gb;
    if (gx > kNumSMs * 16) gx = kNumSMs * 16;
    L[(*nL)++].set((void*)k_cvt_bf16, dim3((unsigned)(gx < 1 ? 1 : gx), 2), dim3(256), q);
  } else {
    if (ca == 1) cvt_rows_launch(s.ds, s.in[0], s.scratch[0], s.in_shape[0][0], s.in_shape[0][1], &L[(*nL)++]);
    if (cb == 1) cvt_rows_launch(s.ds, s.in[1], s.scratch[1], s.in_shape[1][0], s.in_shape[1][1], &L[(*nL)++]);
  }
  for (int w = 0; w < 2; ++w) {
    if ((w == 0 ? ca : cb) != 2) continue;
    CvtParams q{};                                  // element (r, k) = src[k * R + r]
    q.ds = s.ds; q.src[0] = s.in[w]; q.rows[0] = w == 0 ? M : N; q.K = K; q.ld = bf16_pitch(K); q.trans[0] = 1;
    q.dst[0] = (__nv_bfloat16*)s.scratch[w];
    const int64_t tiles = ((q.rows[0] + 31) / 32) * ((q.ld + 31) / 32);
    L[(*nL)++].set((void*)k_cvt_bf16, dim3((unsigned)(tiles < kNumSMs * 16 ? (tiles < 1 ? 1 : tiles) : kNumSMs * 16), 1),
                   dim3(256), q);
  }
  return tc_gemm_launches(c, s.ds, s.scratch[0], s.scratch[1], M, N, K, tc_plan(M, N, K, s.ws != nullptr), s.in[0],
                          s.in[1], s.out, nullptr, (float*)s.ws, L, nL, a_mn ? 1 : 0, b_mn, nullptr, nullptr, 1,
                          s.bias ? &s.in[2] : nullptr);
}

int launch_now(coex_ctx* c, Launch& L) {
  if (L.fn == nullptr && L.ar_buf != nullptr) {
    NcclApi& n = nccl();
    if (!n.ok || c->comm == nullptr) return fail(COEX_CUDA_ERROR, "collective launch without a communicator");
    if (n.all_reduce(L.ar_buf, L.ar_buf, (size_t)L.ar_count, L.ar_f64 ? kNcclDouble : kNcclFloat, kNcclSum, c->comm,
                     c->stream))
      return fail(COEX_CUDA_ERROR, "ncclAllReduce failed");
    return COEX_OK;
  }
  CK(cudaLaunchKernel(L.fn, L.grid, L.block, L.argv(), L.smem, c->stream));
  c->kernel_count++;
  return COEX_OK;
}

int fa_set_attrs() {
  static bool done = false;
  if (done) return COEX_OK;
  CK(cudaFuncSetAttribute((void*)k_fa_fwd, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kFaFwdSmem));
  CK(cudaFuncSetAttribute((void*)k_fa_bwd_kv, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kFaKvSmem));
  CK(cudaFuncSetAttribute((void*)k_fa_bwd_q, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kFaQSmem));
  done = true;
  return COEX_OK;
}

TRec* get_t(coex_ctx* c, int64_t id) {
  auto it = c->tensors.find(id);
  return it == c->tensors.end() ? nullptr : &it->second;
}

int set_var_cur(coex_ctx* c, int idx) {
  c->h_var_cur[idx] = c->vars[idx].t.buf ? c->vars[idx].t.buf->ptr : nullptr;
  CK(cudaMemcpyAsync(c->d_var_cur + idx, c->h_var_cur + idx, sizeof(void*), cudaMemcpyHostToDevice, c->stream));
  return COEX_OK;
}

}  // namespace

// =============================================================== C-ABI: context
namespace {
void nvls_release(coex_ctx* c);
}  // namespace

extern "C" {

const char* coex_last_error(void) { return g_err.c_str(); }
const char* coex_version(void) { return "coexb200 0.1.0 sm_100a"; }

// The tcgen05 GEMM launch shape the runtime picks for an [M, K] x [K, N] bf16 MatMul (tile
// width, split-K count, two-CTA-per-SM variant) -- host-only, for tests and tuning tools.
int coex_gemm_plan(int64_t M, int64_t N, int64_t K, int allow_split, int* bn, int* splits, int* duo) {
  const TcPlan t = tc_plan(M, N, K, allow_split != 0);
  *bn = t.bn;
  *splits = t.splits;
  *duo = tc_use_duo(t.bn, (K + TC_BK - 1) / TC_BK / (t.splits > 0 ? t.splits : 1)) ? 1 : 0;
  return COEX_OK;
}

int coex_ctx_create(int device, int precision, coex_ctx** out) {
  if (precision < COEX_F64 || precision > COEX_BF16) return fail(COEX_INVALID, "bad precision");
  CK(cudaSetDevice(device));
  coex_ctx* c = new coex_ctx();
  c->device = device;
  c->prec = precision;
  c->esize = precision == COEX_F64 ? 8 : 4;
  CK(cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking));
  cudaMemPool_t pool;
  CK(cudaDeviceGetDefaultMemPool(&pool, device));
  uint64_t thresh = ~0ull;
  CK(cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thresh));
  CK(cudaMalloc(&c->d_var_cur, kMaxVars * sizeof(void*)));
  CK(cudaMalloc(&c->d_var_ovl, kMaxVars * sizeof(void*)));
  CK(cudaMalloc(&c->d_var_ovl_shape, kMaxVars * sizeof(int)));
  CK(cudaMalloc(&c->d_var_spare, kMaxVars * sizeof(void*)));
  CK(cudaMemset(c->d_var_cur, 0, kMaxVars * sizeof(void*)));
  CK(cudaMemset(c->d_var_ovl, 0, kMaxVars * sizeof(void*)));
  CK(cudaMemset(c->d_var_spare, 0, kMaxVars * sizeof(void*)));
  CK(cudaHostAlloc((void**)&c->h_var_cur, kMaxVars * sizeof(void*), cudaHostAllocDefault));
  CK(cudaHostAlloc((void**)&c->h_var_spare, kMaxVars * sizeof(void*), cudaHostAllocDefault));
  memset(c->h_var_cur, 0, kMaxVars * sizeof(void*));
  memset(c->h_var_spare, 0, kMaxVars * sizeof(void*));
  CK(cudaMalloc(&c->d_state, sizeof(DevState)));
  CK(cudaMemset(c->d_state, 0, sizeof(DevState)));
  CK(cudaHostAlloc((void**)&c->mb, sizeof(Mailbox), cudaHostAllocMapped));
  memset((void*)c->mb, 0, sizeof(Mailbox));
  CK(cudaHostGetDevicePointer((void**)&c->d_mb, c->mb, 0));
  c->feed_cap = (size_t)32 << 20;   // doubles (256 MiB)
  CK(cudaMalloc(&c->d_red_part, sizeof(double) * kReduceMaxBlocks + 64));
  c->d_red_counter = (unsigned int*)(c->d_red_part + kReduceMaxBlocks);
  CK(cudaMemset(c->d_red_part, 0, sizeof(double) * kReduceMaxBlocks + 64));
  CK(cudaHostAlloc((void**)&c->feed_arena, c->feed_cap * sizeof(double), cudaHostAllocMapped));
  CK(cudaHostGetDevicePointer((void**)&c->d_feed_arena, c->feed_arena, 0));
  c->fetch_cap = (size_t)64 << 20;  // bytes
  CK(cudaHostAlloc((void**)&c->fetch_arena, c->fetch_cap, cudaHostAllocMapped));
  CK(cudaHostGetDevicePointer((void**)&c->d_fetch_arena, c->fetch_arena, 0));
  // jump matrices J_j = T^(kSynthRun * 2^j), stored as 4-bit lookup tables
  std::vector<unsigned long long> jm(kJumpTabWords * kJumpBits), cur(64), tmp(64);
  for (int b = 0; b < 64; ++b) cur[b] = xs_step_host(1ull << b);
  for (int s = 1; s < kSynthRun; s <<= 1) {      // T^kSynthRun by repeated squaring
    mat_square(cur.data(), tmp.data());
    cur.swap(tmp);
  }
  for (int j = 0; j < kJumpBits; ++j) {
    for (int nib = 0; nib < 16; ++nib)
      for (int v = 0; v < 16; ++v) {
        unsigned long long r;
        mat_apply(cur.data(), (unsigned long long)v << (4 * nib), &r);
        jm[kJumpTabWords * j + nib * 16 + v] = r;
      }
    mat_square(cur.data(), tmp.data());
    cur.swap(tmp);
  }
  CK(cudaMalloc(&c->d_jump, jm.size() * sizeof(unsigned long long)));
  CK(cudaMemcpy(c->d_jump, jm.data(), jm.size() * sizeof(unsigned long long), cudaMemcpyHostToDevice));
  *out = c;
  return COEX_OK;
}

int coex_ctx_destroy(coex_ctx* c) {
  if (c == nullptr) return COEX_OK;
  cudaStreamSynchronize(c->stream);
  for (auto& r : c->pinned) cudaHostUnregister(r.first);
  c->pinned.clear();
  for (auto& kv : c->tensors) release(c, kv.second.buf);
  for (auto& v : c->vars) {
    release(c, v.t.buf);
    release(c, v.spare);
  }
  cudaStreamSynchronize(c->stream);
  cudaFree(c->d_var_cur);
  cudaFree(c->d_var_ovl);
  cudaFree(c->d_var_ovl_shape);
  cudaFree(c->d_var_spare);
  cudaFreeHost(c->h_var_cur);
  cudaFreeHost(c->h_var_spare);
  cudaFree(c->d_state);
  cudaFreeHost((void*)c->mb);
  cudaFreeHost(c->feed_arena);
  cudaFreeHost(c->fetch_arena);
  cudaFree(c->d_jump);
  if (c->d_red_part) cudaFree(c->d_red_part);
  if (c->h_stage) cudaFreeHost(c->h_stage);
  for (auto& ev : c->events)
    if (ev) cudaEventDestroy(ev);
  nvls_release(c);
  if (c->comm && nccl().ok) nccl().comm_destroy(c->comm);
  if (c->cap_stream) cudaStreamDestroy(c->cap_stream);
  cudaStreamDestroy(c->stream);
  delete c;
  return COEX_OK;
}

int coex_ctx_sync(coex_ctx* c) {
  CK(cudaStreamSynchronize(c->stream));
  return COEX_OK;
}

int coex_ctx_set_timeout(coex_ctx* c, double seconds) {
  c->timeout_s = seconds;
  return COEX_OK;
}

int64_t coex_ctx_kernel_count(coex_ctx* c) { return c ? c->kernel_count : 0; }

// ---- NVLS multicast region (nvls.cuh) through the driver API, resolved at run time ----
}  // extern "C"
namespace {
struct CuApi {
  bool ok = false;
  CUresult (*mc_create)(CUmemGenericAllocationHandle*, const CUmulticastObjectProp*) = nullptr;
  CUresult (*mc_add_device)(CUmemGenericAllocationHandle, CUdevice) = nullptr;
  CUresult (*mc_bind_mem)(CUmemGenericAllocationHandle, size_t, CUmemGenericAllocationHandle, size_t, size_t,
                          unsigned long long) = nullptr;
  CUresult (*mc_unbind)(CUmemGenericAllocationHandle, CUdevice, size_t, size_t) = nullptr;
  CUresult (*mc_granularity)(size_t*, const CUmulticastObjectProp*, CUmulticastGranularity_flags) = nullptr;
  CUresult (*mem_create)(CUmemGenericAllocationHandle*, size_t, const CUmemAllocationProp*, unsigned long long) = nullptr;
  CUresult (*mem_release)(CUmemGenericAllocationHandle) = nullptr;
  CUresult (*mem_granularity)(size_t*, const CUmemAllocationProp*, CUmemAllocationGranularity_flags) = nullptr;
  CUresult (*addr_reserve)(CUdeviceptr*, size_t, size_t, CUdeviceptr, unsigned long long) = nullptr;
  CUresult (*addr_free)(CUdeviceptr, size_t) = nullptr;
  CUresult (*mem_map)(CUdeviceptr, size_t, size_t, CUmemGenericAllocationHandle, unsigned long long) = nullptr;
  CUresult (*mem_unmap)(CUdeviceptr, size_t) = nullptr;
  CUresult (*set_access)(CUdeviceptr, size_t, const CUmemAccessDesc*, size_t) = nullptr;
  CUresult (*export_handle)(void*, CUmemGenericAllocationHandle, CUmemAllocationHandleType, unsigned long long) = nullptr;
  CUresult (*import_handle)(CUmemGenericAllocationHandle*, void*, CUmemAllocationHandleType) = nullptr;
  CUresult (*dev_attr)(int*, CUdevice_attribute, CUdevice) = nullptr;
};
CuApi& cuapi() {
  static CuApi a;
  static bool tried = false;
  if (!tried) {
    tried = true;
    auto get = [](const char* name, void** fn) {
      cudaDriverEntryPointQueryResult q;
      return cudaGetDriverEntryPoint(name, fn, cudaEnableDefault, &q) == cudaSuccess && q == cudaDriverEntryPointSuccess;
    };
    bool ok = true;
    ok &= get("cuMulticastCreate", (void**)&a.mc_create);
    ok &= get("cuMulticastAddDevice", (void**)&a.mc_add_device);
    ok &= get("cuMulticastBindMem", (void**)&a.mc_bind_mem);
    ok &= get("cuMulticastUnbind", (void**)&a.mc_unbind);
    ok &= get("cuMulticastGetGranularity", (void**)&a.mc_granularity);
    ok &= get("cuMemCreate", (void**)&a.mem_create);
    ok &= get("cuMemRelease", (void**)&a.mem_release);
    ok &= get("cuMemGetAllocationGranularity", (void**)&a.mem_granularity);
    ok &= get("cuMemAddressReserve", (void**)&a.addr_reserve);
    ok &= get("cuMemAddressFree", (void**)&a.addr_free);
    ok &= get("cuMemMap", (void**)&a.mem_map);
    ok &= get("cuMemUnmap", (void**)&a.mem_unmap);
    ok &= get("cuMemSetAccess", (void**)&a.set_access);
    ok &= get("cuMemExportToShareableHandle", (void**)&a.export_handle);
    ok &= get("cuMemImportFromShareableHandle", (void**)&a.import_handle);
    ok &= get("cuDeviceGetAttribute", (void**)&a.dev_attr);
    a.ok = ok;
    cudaGetLastError();
  }
  return a;
}
#define CU(call)                                                                                  \
  do {                                                                                            \
    CUresult r_ = (call);                                                                         \
    if (r_ != CUDA_SUCCESS)                                                                       \
      return fail(COEX_CUDA_ERROR, std::string(#call) + ": CUresult " + std::to_string((int)r_)); \
  } while (0)

CUmulticastObjectProp nvls_prop(size_t bytes, int world) {
  CUmulticastObjectProp mp;
  memset(&mp, 0, sizeof(mp));
  mp.numDevices = (unsigned)world;
  mp.size = bytes;
  mp.handleTypes = CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR;
  return mp;
}
void nvls_release(coex_ctx* c) {
  if (c->nv_mode == RED_P2P) {
    for (int r = 0; r < c->nv_world && r < kMaxPeers; ++r)
      if (c->nv_peer[r] && c->nv_peer[r] != c->nv_local) cudaIpcCloseMemHandle(c->nv_peer[r]);
    if (c->nv_p2p_own && c->nv_local) cudaFree(c->nv_local);
    if (c->nv_gen) cudaFree(c->nv_gen);
    return;
  }
  if (c->nv_local || c->nv_mc_handle) {           // NVLS region: unmap both aliases, unbind, release
    CuApi& a = cuapi();
    if (c->nv_mc) { a.mem_unmap((CUdeviceptr)c->nv_mc, c->nv_bytes); a.addr_free((CUdeviceptr)c->nv_mc, c->nv_bytes); }
    if (c->nv_local) {
      a.mem_unmap((CUdeviceptr)c->nv_local, c->nv_bytes);
      a.addr_free((CUdeviceptr)c->nv_local, c->nv_bytes);
      a.mc_unbind(c->nv_mc_handle, (CUdevice)c->device, 0, c->nv_bytes);
    }
    if (c->nv_mem_handle) a.mem_release(c->nv_mem_handle);
    if (c->nv_mc_handle) a.mem_release(c->nv_mc_handle);
    if (c->nv_gen) cudaFree(c->nv_gen);
  }
}
}  // namespace
extern "C" {

int coex_nvls_supported(coex_ctx* c, int* out) {
  *out = 0;
  CuApi& a = cuapi();
  if (!a.ok) return COEX_OK;
  int v = 0;
  if (a.dev_attr(&v, CU_DEVICE_ATTRIBUTE_MULTICAST_SUPPORTED, (CUdevice)c->device) == CUDA_SUCCESS) *out = v;
  return COEX_OK;
}

// Rank 0: the team's multicast object (world devices, >= bytes per device, rounded to the
// recommended granularity), exported as a POSIX fd for the other ranks (pidfd_getfd).
int coex_nvls_create(coex_ctx* c, int64_t bytes, int world, int64_t* out_pid_fd) {
  CuApi& a = cuapi();
  if (!a.ok) return fail(COEX_CUDA_ERROR, "driver multicast API not available");
  if (c->nv_mc_handle) return fail(COEX_INVALID, "NVLS region already created");
  CK(cudaSetDevice(c->device));
  size_t want = (size_t)bytes + kNvlsFlagBytes, gran = 0;
  CUmulticastObjectProp mp = nvls_prop(want, world);
  CU(a.mc_granularity(&gran, &mp, CU_MULTICAST_GRANULARITY_RECOMMENDED));
  want = (want + gran - 1) / gran * gran;
  mp.size = want;
  CUmemGenericAllocationHandle h;
  CU(a.mc_create(&h, &mp));
  c->nv_mc_handle = h;
  c->nv_bytes = want;
  c->nv_world = world;
  c->nv_creator = 1;
  int fd = -1;
  CU(a.export_handle(&fd, h, CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR, 0));
  out_pid_fd[0] = (int64_t)getpid();
  out_pid_fd[1] = fd;
  out_pid_fd[2] = (int64_t)want;
  return COEX_OK;
}

// Every rank: join the team (ranks > 0 import the creator's fd first), add this device.
int coex_nvls_attach(coex_ctx* c, int64_t pid, int64_t fd, int64_t bytes, int world) {
  CuApi& a = cuapi();
  if (!a.ok) return fail(COEX_CUDA_ERROR, "driver multicast API not available");
  CK(cudaSetDevice(c->device));
  if (!c->nv_creator) {
    const int pfd = (int)syscall(434 /* pidfd_open */, (pid_t)pid, 0);
    if (pfd < 0) return fail(COEX_CUDA_ERROR, "pidfd_open failed: " + std::string(strerror(errno)));
    const int lfd = (int)syscall(438 /* pidfd_getfd */, pfd, (int)fd, 0);
    close(pfd);
    if (lfd < 0) return fail(COEX_CUDA_ERROR, "pidfd_getfd failed: " + std::string(strerror(errno)));
    CUmemGenericAllocationHandle h;
    CUresult r = a.import_handle(&h, (void*)(uintptr_t)lfd, CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR);
    close(lfd);
    if (r != CUDA_SUCCESS) return fail(COEX_CUDA_ERROR, "cuMemImportFromShareableHandle: " + std::to_string((int)r));
    c->nv_mc_handle = h;
    c->nv_bytes = (size_t)bytes;
    c->nv_world = world;
  }
  CU(a.mc_add_device(c->nv_mc_handle, (CUdevice)c->device));
  c->nv_attached = 1;
  return COEX_OK;
}

// Every rank, after all ranks attached: this rank's physical copy bound to the object, both
// mapped (unicast + multicast), flags zeroed.  The host barrier after it precedes any pass.
int coex_nvls_bind(coex_ctx* c) {
  CuApi& a = cuapi();
  if (!c->nv_attached) return fail(COEX_INVALID, "coex_nvls_bind before coex_nvls_attach");
  CK(cudaSetDevice(c->device));
  CUmemAllocationProp ap;
  memset(&ap, 0, sizeof(ap));
  ap.type = CU_MEM_ALLOCATION_TYPE_PINNED;
  ap.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
  ap.location.id = c->device;
  size_t g = 0;
  CU(a.mem_granularity(&g, &ap, CU_MEM_ALLOC_GRANULARITY_RECOMMENDED));
  if (c->nv_bytes % g) return fail(COEX_INVALID, "NVLS size not a multiple of the allocation granularity");
  CUmemGenericAllocationHandle mem;
  CU(a.mem_create(&mem, c->nv_bytes, &ap, 0));
  c->nv_mem_handle = mem;
  CUmemAccessDesc ad;
  memset(&ad, 0, sizeof(ad));
  ad.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
  ad.location.id = c->device;
  ad.flags = CU_MEM_ACCESS_FLAGS_PROT_READWRITE;
  CUdeviceptr uc = 0, mc = 0;
  CU(a.addr_reserve(&uc, c->nv_bytes, g, 0, 0));
  CU(a.mem_map(uc, c->nv_bytes, 0, mem, 0));
  CU(a.set_access(uc, c->nv_bytes, &ad, 1));
  CU(a.mc_bind_mem(c->nv_mc_handle, 0, mem, 0, c->nv_bytes, 0));
  CU(a.addr_reserve(&mc, c->nv_bytes, g, 0, 0));
  CU(a.mem_map(mc, c->nv_bytes, 0, c->nv_mc_handle, 0));
  CU(a.set_access(mc, c->nv_bytes, &ad, 1));
  c->nv_local = (char*)uc;
  c->nv_mc = (char*)mc;
  c->nv_mode = RED_MC;
  CK(cudaMalloc(&c->nv_gen, sizeof(unsigned int) * kNvlsSlots));
  CK(cudaMemset(c->nv_gen, 0, sizeof(unsigned int) * kNvlsSlots));
  CK(cudaMemset(c->nv_local, 0, c->nv_bytes));
  CK(cudaDeviceSynchronize());
  return COEX_OK;
}

int coex_nvls_info(coex_ctx* c, int64_t* out3) {
  out3[0] = c->nv_local != nullptr ? (int64_t)(c->nv_bytes - kNvlsFlagBytes) : 0;
  out3[1] = c->nv_world;
  out3[2] = c->nv_mode;
  return COEX_OK;
}

// RED_P2P transport (no multicast object): this rank's region (flags zeroed), exported as a
// CUDA IPC handle (64 bytes) for the peers.
int coex_p2p_create(coex_ctx* c, int64_t bytes, uint8_t* out_handle64) {
  if (c->nv_local) return fail(COEX_INVALID, "gradient region already set up");
  CK(cudaSetDevice(c->device));
  const size_t want = ((size_t)bytes + kNvlsFlagBytes + 255) & ~(size_t)255;
  CK(cudaMalloc(&c->nv_local, want));
  c->nv_p2p_own = true;
  c->nv_bytes = want;
  CK(cudaMemset(c->nv_local, 0, want));
  cudaIpcMemHandle_t h;
  CK(cudaIpcGetMemHandle(&h, c->nv_local));
  memcpy(out_handle64, &h, sizeof(h) < 64 ? sizeof(h) : 64);
  return COEX_OK;
}

// Every rank, with all ranks' handles (rank order, 64 bytes each): open the peers' regions.
int coex_p2p_open(coex_ctx* c, const uint8_t* handles, int world) {
  if (!c->nv_local || !c->nv_p2p_own) return fail(COEX_INVALID, "coex_p2p_open before coex_p2p_create");
  if (world < 1 || world > kMaxPeers) return fail(COEX_INVALID, "P2P gradient region: 1..8 ranks");
  CK(cudaSetDevice(c->device));
  for (int r = 0; r < world; ++r) {
    if (r == c->rank) {
      c->nv_peer[r] = c->nv_local;
      continue;
    }
    cudaIpcMemHandle_t h;
    memcpy(&h, handles + 64 * r, sizeof(h));
    void* ptr = nullptr;
    CK(cudaIpcOpenMemHandle(&ptr, h, cudaIpcMemLazyEnablePeerAccess));
    c->nv_peer[r] = (char*)ptr;
  }
  c->nv_world = world;
  c->nv_mode = RED_P2P;
  CK(cudaMalloc(&c->nv_gen, sizeof(unsigned int) * kNvlsSlots));
  CK(cudaMemset(c->nv_gen, 0, sizeof(unsigned int) * kNvlsSlots));
  CK(cudaDeviceSynchronize());
  return COEX_OK;
}

int coex_nccl_unique_id(uint8_t* out128) {
  NcclApi& n = nccl();
  if (!n.ok) return fail(COEX_CUDA_ERROR, "libnccl.so.2 not found");
  nccl_uid_t id;
  int r = n.get_unique_id(&id);
  if (r) return fail(COEX_CUDA_ERROR, std::string("ncclGetUniqueId: ") + (n.error_string ? n.error_string(r) : ""));
  memcpy(out128, id.internal, 128);
  return COEX_OK;
}

int coex_ctx_init_comm(coex_ctx* c, int rank, int world, const uint8_t* uid128) {
  NcclApi& n = nccl();
  if (!n.ok) return fail(COEX_CUDA_ERROR, "libnccl.so.2 not found");
  nccl_uid_t id;
  memcpy(id.internal, uid128, 128);
  CK(cudaSetDevice(c->device));
  int r = n.comm_init_rank(&c->comm, world, id, rank);
  if (r) return fail(COEX_CUDA_ERROR, std::string("ncclCommInitRank: ") + (n.error_string ? n.error_string(r) : ""));
  c->rank = rank;
  c->world = world;
  if (!c->cap_stream) CK(cudaStreamCreateWithFlags(&c->cap_stream, cudaStreamNonBlocking));
  return COEX_OK;
}

int coex_ctx_set_trace(coex_ctx* c, int capacity) {
  if (c->active) return fail(COEX_IN_FLIGHT_PASS, "set_trace during a pass");
  CK(cudaStreamSynchronize(c->stream));
  if (c->d_trace) {
    cudaFree(c->d_trace);
    c->d_trace = nullptr;
  }
  c->trace_cap = capacity > 0 ? capacity : 0;
  if (c->trace_cap) CK(cudaMalloc(&c->d_trace, sizeof(unsigned long long) * 2 * c->trace_cap));
  unsigned long long* tp = c->d_trace;
  int cap = c->trace_cap;
  CK(cudaMemcpy((char*)c->d_state + offsetof(DevState, trace), &tp, sizeof(tp), cudaMemcpyHostToDevice));
  CK(cudaMemcpy((char*)c->d_state + offsetof(DevState, trace_cap), &cap, sizeof(cap), cudaMemcpyHostToDevice));
  return COEX_OK;
}

int coex_ctx_read_trace(coex_ctx* c, uint64_t* out, int64_t cap, int64_t* n) {
  if (c->active) return fail(COEX_IN_FLIGHT_PASS, "read_trace during a pass");
  int tn = 0;
  CK(cudaStreamSynchronize(c->stream));
  CK(cudaMemcpy(&tn, (char*)c->d_state + offsetof(DevState, trace_n), sizeof(int), cudaMemcpyDeviceToHost));
  if (tn > c->trace_cap) tn = c->trace_cap;
  int64_t m = tn < cap ? tn : cap;
  if (m > 0) CK(cudaMemcpy(out, c->d_trace, sizeof(uint64_t) * 2 * m, cudaMemcpyDeviceToHost));
  *n = m;
  return COEX_OK;
}

int coex_ctx_event_record(coex_ctx* c, int slot) {
  if (slot < 0 || slot >= 64) return fail(COEX_INVALID, "event slot out of range");
  if (!c->events[slot]) CK(cudaEventCreate(&c->events[slot]));
  CK(cudaEventRecord(c->events[slot], c->stream));
  return COEX_OK;
}

int coex_ctx_event_elapsed(coex_ctx* c, int a, int b, double* ms) {
  if (a < 0 || a >= 64 || b < 0 || b >= 64 || !c->events[a] || !c->events[b])
    return fail(COEX_INVALID, "event slot not recorded");
  CK(cudaEventSynchronize(c->events[b]));
  float f = 0.f;
  CK(cudaEventElapsedTime(&f, c->events[a], c->events[b]));
  *ms = f;
  return COEX_OK;
}

// =============================================================== tensors
int coex_tensor_put(coex_ctx* c, int ndim, const int64_t* shape, const double* data, int64_t* id) {
  return coex_tensor_put_index(c, ndim, shape, data, 0.0, id);
}

int coex_tensor_put_index(coex_ctx* c, int ndim, const int64_t* shape, const double* data, double index_v,
                          int64_t* id) {
  if (ndim < 0 || ndim > COEX_MAX_RANK) return fail(COEX_INVALID, "rank out of range");
  TRec t;
  t.ndim = ndim;
  for (int i = 0; i < ndim; ++i) t.shape[i] = shape[i];
  t.numel = numel_of(ndim, shape);
  int rc = alloc_buf(c, t.numel * c->esize, &t.buf);
  if (rc) return rc;
  if (t.numel > 0) {
    rc = ensure_stage(c, t.numel);
    if (rc) return rc;
    CK(cudaStreamSynchronize(c->stream));        // staging buffer reuse
    memcpy(c->h_stage, data, t.numel * sizeof(double));
    if (is_f64(c) && !(index_v > 0.0)) {
      CK(cudaMemcpyAsync(t.buf->ptr, c->h_stage, t.numel * 8, cudaMemcpyHostToDevice, c->stream));
    } else {
      double* dtmp;
      CK(cudaMallocAsync(&dtmp, t.numel * 8, c->stream));
      CK(cudaMemcpyAsync(dtmp, c->h_stage, t.numel * 8, cudaMemcpyHostToDevice, c->stream));
      if (is_f64(c))
        k_from_f64<double><<<grid_for(t.numel), 256, 0, c->stream>>>(dtmp, (double*)t.buf->ptr, t.numel, index_v);
      else
        k_from_f64<float><<<grid_for(t.numel), 256, 0, c->stream>>>(dtmp, (float*)t.buf->ptr, t.numel, index_v);
      CK(cudaGetLastError());
      CK(cudaFreeAsync(dtmp, c->stream));
    }
  }
  *id = new_handle(c, t);
  return COEX_OK;
}

int coex_tensor_synth(coex_ctx* c, uint64_t state, int ndim, const int64_t* shape, int64_t* id) {
  return coex_tensor_synth_index(c, state, ndim, shape, 0.0, id);
}

int coex_tensor_synth_index(coex_ctx* c, uint64_t state, int ndim, const int64_t* shape, double index_v,
                            int64_t* id) {
  if (ndim < 0 || ndim > COEX_MAX_RANK) return fail(COEX_INVALID, "rank out of range");
  TRec t;
  t.ndim = ndim;
  for (int i = 0; i < ndim; ++i) t.shape[i] = shape[i];
  t.numel = numel_of(ndim, shape);
  int rc = alloc_buf(c, t.numel * c->esize, &t.buf);
  if (rc) return rc;
  if (t.numel > 0) {
    SynthParams p{};
    p.jump = c->d_jump;
    p.state = state;
    p.n = t.numel;
    p.iv = index_v;
    p.out.buf[0] = t.buf->ptr;
    const int64_t per_block = (int64_t)kSynthThreads * kSynthRun;
    int64_t blocks = (t.numel + per_block - 1) / per_block;
    dim3 g((unsigned)(blocks < kNumSMs * 4 ? blocks : kNumSMs * 4));
    Launch L;
    if (is_f64(c)) L.set((void*)k_synth<double>, g, dim3(kSynthThreads), p);
    else L.set((void*)k_synth<float>, g, dim3(kSynthThreads), p);
    rc = launch_now(c, L);
    if (rc) return rc;
  }
  *id = new_handle(c, t);
  return COEX_OK;
}

int coex_tensor_info(coex_ctx* c, int64_t id, int* ndim, int64_t* shape) {
  TRec* t = get_t(c, id);
  if (!t) return fail(COEX_INVALID, "unknown tensor id");
  *ndim = t->ndim;
  for (int i = 0; i < t->ndim; ++i) shape[i] = t->shape[i];
  return COEX_OK;
}

static int read_buf(coex_ctx* c, const void* dptr, int64_t numel, double* out) {
  if (numel == 0) return COEX_OK;
  int rc = ensure_stage(c, numel);
  if (rc) return rc;
  CK(cudaMemcpyAsync(c->h_stage, dptr, numel * c->esize, cudaMemcpyDeviceToHost, c->stream));
  CK(cudaStreamSynchronize(c->stream));
  if (is_f64(c)) {
    memcpy(out, c->h_stage, numel * 8);
  } else {
    const float* f = (const float*)c->h_stage;
    for (int64_t i = 0; i < numel; ++i) out[i] = (double)f[i];
  }
  return COEX_OK;
}

int coex_tensor_get(coex_ctx* c, int64_t id, double* out, int64_t cap, int* ndim, int64_t* shape) {
  TRec* t = get_t(c, id);
  if (!t) return fail(COEX_INVALID, "unknown tensor id");
  if (cap < t->numel) return fail(COEX_INVALID, "output buffer too small");
  *ndim = t->ndim;
  for (int i = 0; i < t->ndim; ++i) shape[i] = t->shape[i];
  return read_buf(c, t->buf ? t->buf->ptr : nullptr, t->numel, out);
}

int coex_tensor_free(coex_ctx* c, int64_t id) {
  auto it = c->tensors.find(id);
  if (it == c->tensors.end()) return fail(COEX_INVALID, "unknown tensor id");
  release(c, it->second.buf);
  c->tensors.erase(it);
  return COEX_OK;
}

}  // extern "C"

namespace {
// Eager op: spec from tensor records; scratch (bf16 MatMul operands) and extension-op
// workspace allocated stream-ordered around the launches.
int eager_spec(coex_ctx* c, int kind, const coex_attrs* attrs, int nin, const TRec* in, const TRec& o, OpSpec* s) {
  s->kind = kind;
  s->nin = nin;
  for (int i = 0; i < nin; ++i) {
    s->in[i].direct = in[i].buf ? in[i].buf->ptr : nullptr;
    s->in_ndim[i] = in[i].ndim;
    memcpy(s->in_shape[i], in[i].shape, sizeof(int64_t) * in[i].ndim);
  }
  s->out_ndim = o.ndim;
  memcpy(s->out_shape, o.shape, sizeof(int64_t) * o.ndim);
  if (attrs) {
    s->attr_n = attrs->n;
    memcpy(s->attr_dims, attrs->dims, sizeof(int64_t) * COEX_MAX_RANK);
    s->value = attrs->value;
  }
  s->out.buf[0] = o.buf->ptr;
  return COEX_OK;
}

int eager_scratch(coex_ctx* c, OpSpec* s) {
  if (needs_scratch(c, s->kind)) {
    size_t ba, bb;
    scratch_bytes(c, *s, &ba, &bb);
    CK(cudaMallocAsync(&s->scratch[0], ba, c->stream));
    CK(cudaMallocAsync(&s->scratch[1], bb, c->stream));
    const int64_t M = s->trans_a ? s->in_shape[0][1] : s->in_shape[0][0];
    const int64_t K = s->trans_a ? s->in_shape[0][0] : s->in_shape[0][1];
    const int64_t N = s->trans_b ? s->in_shape[1][0] : s->in_shape[1][1];
    const size_t wb = matmul_split_ws_c(c, M, N, K);
    if (wb) CK(cudaMallocAsync((void**)&s->ws, wb, c->stream));
  }
  if (is_ext_compute(s->kind)) {
    Launch tmp[kMaxLaunches];
    int n = 0;
    size_t wb = 0, pzb = 0;
    int rc = build_xop(c, *s, tmp, &n, &wb, &pzb);
    if (rc) return rc;
    if (wb < 256) wb = 256;          // a non-null workspace marks the build pass
    CK(cudaMallocAsync((void**)&s->ws, wb, c->stream));
    if (pzb) {
      CK(cudaMallocAsync((void**)&s->pz, pzb, c->stream));
      CK(cudaMemsetAsync(s->pz, 0, pzb, c->stream));
    }
  }
  return COEX_OK;
}

void eager_free(coex_ctx* c, OpSpec* s) {
  if (s->scratch[0]) cudaFreeAsync(s->scratch[0], c->stream);
  if (s->scratch[1]) cudaFreeAsync(s->scratch[1], c->stream);
  if (s->ws) cudaFreeAsync(s->ws, c->stream);
  if (s->pz) cudaFreeAsync(s->pz, c->stream);
  s->scratch[0] = s->scratch[1] = nullptr;
  s->ws = s->pz = nullptr;
}
}  // namespace

extern "C" {

int coex_exec_op(coex_ctx* c, int kind, const coex_attrs* attrs, int nin, const int64_t* in_ids,
                 int64_t* out_id) {
  if (c->active) return fail(COEX_IN_FLIGHT_PASS, "eager op while a pass is in flight");
  if (nin < 0 || nin > kMaxIn) return fail(COEX_BAD_ATTRS, "wrong number of tensor inputs");
  TRec in[kMaxIn];
  for (int i = 0; i < nin; ++i) {
    TRec* t = get_t(c, in_ids[i]);
    if (!t) return fail(COEX_INVALID, "unknown input tensor id");
    in[i] = *t;
  }
  TRec o;
  int rc = infer(kind, attrs, nin, in, &o.ndim, o.shape);
  if (rc) return rc;
  o.numel = numel_of(o.ndim, o.shape);
  if (kind == COEX_RESHAPE || kind == COEX_ASSIGN_VAR) {       // views: share the buffer
    o.buf = in[0].buf;
    o.buf->refs++;
    *out_id = new_handle(c, o);
    return COEX_OK;
  }
  rc = alloc_buf(c, o.numel * c->esize, &o.buf);
  if (rc) return rc;
  OpSpec s;
  eager_spec(c, kind, attrs, nin, in, o, &s);
  if (o.numel > 0 || kind == COEX_SUM || kind == COEX_MEAN) {
    rc = eager_scratch(c, &s);
    Launch L[kMaxLaunches];
    int nL = 0;
    if (rc == COEX_OK) rc = build_launches(c, s, L, &nL);
    for (int i = 0; rc == COEX_OK && i < nL; ++i) rc = launch_now(c, L[i]);
    eager_free(c, &s);
    if (rc) {
      release(c, o.buf);
      return rc;
    }
  }
  *out_id = new_handle(c, o);
  return COEX_OK;
}

int coex_exec_op_timed(coex_ctx* c, int kind, const coex_attrs* attrs, int nin, const int64_t* in_ids, int reps,
                       double* avg_ms) {
  if (reps < 1) return fail(COEX_INVALID, "reps must be >= 1");
  int64_t out;
  int rc = coex_exec_op(c, kind, attrs, nin, in_ids, &out);     // warm-up + output buffer
  if (rc) return rc;
  TRec in[kMaxIn];
  for (int i = 0; i < nin; ++i) in[i] = *get_t(c, in_ids[i]);
  TRec* o = get_t(c, out);
  OpSpec s;
  eager_spec(c, kind, attrs, nin, in, *o, &s);
  rc = eager_scratch(c, &s);
  if (rc) return rc;
  Launch L[kMaxLaunches];
  int nL = 0;
  rc = build_launches(c, s, L, &nL);
  if (rc) return rc;
  rc = coex_ctx_event_record(c, 62);
  if (rc) return rc;
  for (int r = 0; r < reps; ++r) {
    for (int i = 0; i < nL; ++i) {
      rc = launch_now(c, L[i]);
      if (rc) return rc;
    }
  }
  rc = coex_ctx_event_record(c, 63);
  if (rc) return rc;
  double ms = 0;
  rc = coex_ctx_event_elapsed(c, 62, 63, &ms);
  *avg_ms = ms / reps;
  eager_free(c, &s);
  coex_tensor_free(c, out);
  return rc;
}

// Per-launch device time of one op (roofline evidence for multi-kernel ops): every launch of
// the op's lowering is repeated `reps` times back to back between CUDA events on the context
// stream, after one full warm run that fills the op's scratch.
int coex_exec_op_profile(coex_ctx* c, int kind, const coex_attrs* attrs, int nin, const int64_t* in_ids, int reps,
                         double* ms, int* nlaunch, char* names, int name_cap) {
  if (reps < 1) return fail(COEX_INVALID, "reps must be >= 1");
  int64_t out;
  int rc = coex_exec_op(c, kind, attrs, nin, in_ids, &out);
  if (rc) return rc;
  TRec in[kMaxIn];
  for (int i = 0; i < nin; ++i) in[i] = *get_t(c, in_ids[i]);
  TRec* o = get_t(c, out);
  OpSpec s;
  eager_spec(c, kind, attrs, nin, in, *o, &s);
  rc = eager_scratch(c, &s);
  if (rc) return rc;
  Launch L[kMaxLaunches];
  int nL = 0;
  rc = build_launches(c, s, L, &nL);
  for (int i = 0; rc == COEX_OK && i < nL; ++i) rc = launch_now(c, L[i]);
  for (int j = 0; rc == COEX_OK && j < nL; ++j) {
    rc = coex_ctx_event_record(c, 62);
    for (int r = 0; rc == COEX_OK && r < reps; ++r) rc = launch_now(c, L[j]);
    if (rc == COEX_OK) rc = coex_ctx_event_record(c, 63);
    double t = 0;
    if (rc == COEX_OK) rc = coex_ctx_event_elapsed(c, 62, 63, &t);
    ms[j] = t / reps;
    const char* nm = nullptr;
    if (names != nullptr && name_cap > 0) {
      if (cudaFuncGetName(&nm, L[j].fn) != cudaSuccess || nm == nullptr) nm = "?";
      snprintf(names + (size_t)j * name_cap, name_cap, "%s", nm);
    }
  }
  *nlaunch = nL;
  eager_free(c, &s);
  coex_tensor_free(c, out);
  return rc;
}

// Fused causal attention outside a graph (kernel-level parity and ncu captures of
// attn_tc.cuh; the step graph reaches the same kernels through T_ATTN).  Forward: in = {q, k,
// v} fp32 [BH][T][64] -> out = {O [BH][T][64], lse [BH][T]}.  Backward: in = {q, k, v, O, dO,
// lse} -> out = {dQ, dK, dV}.  reps > 0: the kernels are re-launched reps times between CUDA
// events after the first run and *avg_ms receives the per-repetition time.
int coex_flash_attn(coex_ctx* c, int backward, const int64_t* in_ids, int BH, int T, double scale, int reps,
                    int64_t* out_ids, double* avg_ms) {
  if (c->active) return fail(COEX_IN_FLIGHT_PASS, "eager op while a pass is in flight");
  if (c->esize != 4) return fail(COEX_BAD_ATTRS, "flash attention: fp32 / bf16 precision modes only");
  if (BH < 1 || T < FA_BLK || T % FA_BLK) return fail(COEX_BAD_ATTRS, "flash attention: T a multiple of 128");
  const int nin = backward ? 6 : 3;
  const float* ptr[6];
  for (int i = 0; i < nin; ++i) {
    TRec* t = get_t(c, in_ids[i]);
    const int64_t want = (int64_t)BH * T * (i == 5 ? 1 : FA_D);
    if (!t || t->numel != want) return fail(COEX_SHAPE_MISMATCH, "flash attention: operand size");
    ptr[i] = (const float*)t->buf->ptr;
  }
  if (int e = fa_set_attrs()) return e;
  auto in_of = [](const void* p) { In x{}; x.direct = p; return x; };
  auto out_of = [](void* p) { Out o{}; o.buf[0] = p; return o; };
  const int nout = backward ? 3 : 2;
  TRec o[3];
  for (int i = 0; i < nout; ++i) {
    const bool lse = !backward && i == 1;
    o[i].ndim = lse ? 2 : 3;
    o[i].shape[0] = BH;
    o[i].shape[1] = T;
    o[i].shape[2] = FA_D;
    o[i].numel = (int64_t)BH * T * (lse ? 1 : FA_D);
    int rc = alloc_buf(c, o[i].numel * 4, &o[i].buf);
    if (rc) return rc;
  }
  FaParams fp{};
  fp.ds = c->d_state;
  fp.BH = BH;
  fp.T = T;
  fp.H = 1;
  fp.rs = FA_D;
  fp.scale = (float)scale;
  fp.q = in_of(ptr[0]);
  fp.k = in_of(ptr[1]);
  fp.v = in_of(ptr[2]);
  Buf *delta = nullptr, *tiles = nullptr;
  int rc = alloc_buf(c, (int64_t)fa_tiles_bytes(BH, T), &tiles);
  if (rc) return rc;
  fp.tiles = (unsigned char*)tiles->ptr;
  const unsigned pb = fa_prep_blocks(fp);
  Launch L[4];
  int nL = 0;
  if (!backward) {
    fp.lse = (float*)o[1].buf->ptr;
    fp.out = out_of(o[0].buf->ptr);
    L[nL++].set((void*)k_fa_prep_qkv, dim3(pb, 3), dim3(256), fp);
    L[nL].set((void*)k_fa_fwd, dim3(fa_fwd_blocks(fp)), dim3(FA_THREADS), fp);
    L[nL++].smem = kFaFwdSmem;
  } else {
    rc = alloc_buf(c, (int64_t)BH * T * 4, &delta);
    if (rc) return rc;
    fp.o = in_of(ptr[3]);
    fp.dout = in_of(ptr[4]);
    fp.lse = (float*)ptr[5];
    fp.delta = (float*)delta->ptr;
    fp.out = out_of(o[0].buf->ptr);
    fp.out2 = out_of(o[1].buf->ptr);
    fp.out3 = out_of(o[2].buf->ptr);
    const unsigned blocks = (unsigned)(BH * (T / FA_BLK));
    L[nL++].set((void*)k_fa_prep_qkv, dim3(pb, 3), dim3(256), fp);
    L[nL++].set((void*)k_fa_prep_do, dim3(pb), dim3(256), fp);
    L[nL].set((void*)k_fa_bwd_kv, dim3(blocks), dim3(FA_THREADS), fp);
    L[nL++].smem = kFaKvSmem;
    L[nL].set((void*)k_fa_bwd_q, dim3(blocks), dim3(FA_THREADS), fp);
    L[nL++].smem = kFaQSmem;
  }
  for (int i = 0; rc == COEX_OK && i < nL; ++i) rc = launch_now(c, L[i]);
  if (rc == COEX_OK && getenv("COEX_FA_DBG") && !backward) {   // one instrumented forward: CTA 0 clocks
    long long* dbg = nullptr;
    CK(cudaMalloc(&dbg, 4096 * sizeof(long long)));
    CK(cudaMemset(dbg, 0, 4096 * sizeof(long long)));
    FaParams dp = fp;
    dp.dbg = dbg;
    Launch D;
    D.set((void*)k_fa_fwd, dim3(fa_fwd_blocks(fp)), dim3(FA_THREADS), dp);
    D.smem = kFaFwdSmem;
    rc = launch_now(c, D);
    CK(cudaStreamSynchronize(c->stream));
    std::vector<long long> h(4096);
    CK(cudaMemcpy(h.data(), dbg, 4096 * sizeof(long long), cudaMemcpyDeviceToHost));
    cudaFree(dbg);
    const long long t0 = h[0];
    for (int role = 0; role < 4; ++role) {
      printf("FA_DBG role %d:", role);
      for (int i = 0; i < 1024; ++i)
        if (h[role * 1024 + i]) printf(" %d:%lld", i, h[role * 1024 + i] - t0);
      printf("\n");
    }
    fflush(stdout);
  }
  // timed repetitions: the per-call work (tile preparation included; backward: the q / k / v
  // tiles its forward would have left are rebuilt, the only launch not in the step's backward)
  if (rc == COEX_OK && reps > 0) {
    rc = coex_ctx_event_record(c, 62);
    for (int r = 0; rc == COEX_OK && r < reps; ++r)
      for (int i = backward ? 1 : 0; rc == COEX_OK && i < nL; ++i) rc = launch_now(c, L[i]);
    if (rc == COEX_OK) rc = coex_ctx_event_record(c, 63);
    double ms = 0;
    if (rc == COEX_OK) rc = coex_ctx_event_elapsed(c, 62, 63, &ms);
    if (avg_ms) *avg_ms = ms / reps;
  }
  if (delta) release(c, delta);
  release(c, tiles);
  for (int i = 0; i < nout; ++i) {
    if (rc) {
      release(c, o[i].buf);
      continue;
    }
    out_ids[i] = new_handle(c, o[i]);
  }
  return rc;
}

// =============================================================== variables
int coex_var_define(coex_ctx* c, const char* name, int64_t tid, int* var_index) {
  TRec* t = get_t(c, tid);
  if (!t) return fail(COEX_INVALID, "unknown tensor id");
  auto it = c->var_index.find(name);
  int idx;
  if (it == c->var_index.end()) {
    if ((int)c->vars.size() >= kMaxVars) return fail(COEX_INVALID, "too many variables");
    idx = (int)c->vars.size();
    c->vars.push_back(Var());
    c->vars[idx].name = name;
    c->var_index[name] = idx;
  } else {
    idx = it->second;
    release(c, c->vars[idx].t.buf);
  }
  c->vars[idx].t = *t;
  c->vars[idx].t.buf->refs++;
  *var_index = idx;
  return set_var_cur(c, idx);
}

int coex_var_read(coex_ctx* c, int idx, int64_t* tid) {
  if (idx < 0 || idx >= (int)c->vars.size()) return fail(COEX_BAD_ATTRS, "unknown variable");
  if (c->active) return fail(COEX_IN_FLIGHT_PASS, "variable read during a pass");
  TRec t = c->vars[idx].t;
  t.buf->refs++;
  *tid = new_handle(c, t);
  return COEX_OK;
}

int coex_var_assign(coex_ctx* c, int idx, int64_t tid) {
  if (idx < 0 || idx >= (int)c->vars.size()) return fail(COEX_BAD_ATTRS, "unknown variable");
  if (c->active) return fail(COEX_IN_FLIGHT_PASS, "variable assign during a pass");
  TRec* t = get_t(c, tid);
  if (!t) return fail(COEX_INVALID, "unknown tensor id");
  Buf* old = c->vars[idx].t.buf;
  c->vars[idx].t = *t;
  c->vars[idx].t.buf->refs++;
  release(c, old);
  return set_var_cur(c, idx);
}

int coex_var_info(coex_ctx* c, int idx, int* ndim, int64_t* shape) {
  if (idx < 0 || idx >= (int)c->vars.size()) return fail(COEX_BAD_ATTRS, "unknown variable");
  *ndim = c->vars[idx].t.ndim;
  for (int i = 0; i < *ndim; ++i) shape[i] = c->vars[idx].t.shape[i];
  return COEX_OK;
}

int coex_var_rollback(coex_ctx* c) {
  if (c->active) return fail(COEX_IN_FLIGHT_PASS, "rollback during a pass");
  return COEX_OK;   // the overlay lives only inside a pass; a cancelled pass never commits
}

}  // extern "C"

// =============================================================== symbolic programs
namespace {

enum PlanTag : int64_t { T_SEQ = 1, T_OP = 2, T_PTR = 3, T_FEED = 4, T_FETCH = 5, T_SWITCH = 6, T_WHILE = 7, T_CHAIN = 8,
                         T_ALLREDUCE = 9, T_XOP = 10, T_MCHAIN = 11, T_ATTN = 12, T_JOIN = 13,
                         T_NVLS_AR = 14, T_NVLS_ZERO = 15 };
constexpr int64_t kPlanMagic = 0xC0E8B200;
constexpr int64_t kPlanVersion = 4;

struct FeedSlot {
  int64_t slot;
  void* buf;
  void** cell;
  FeedRecord* rec;
};

}  // namespace

struct coex_prog {
  coex_ctx* ctx = nullptr;
  cudaGraph_t graph = nullptr;
  cudaGraphExec_t exec = nullptr;
  char* arena = nullptr;              // node / slot buffers
  size_t arena_bytes = 0;
  void** cells = nullptr;             // device pointer cells
  void** cells_init = nullptr;        // their build-time values (k_pass_begin resets them)
  void* spare = nullptr;              // zero-filled stand-in for cells without a buffer of their own
  int64_t ncells = 0;
  FeedRecord* recs = nullptr;
  unsigned int* late = nullptr;       // late-publication counters
  int64_t n_kernel_nodes = 0, n_cond_nodes = 0, n_compute = 0, n_collectives = 0, n_guards = 0;
  int64_t n_nvls_fused = 0;           // GEMMs whose epilogue reduces into the NVLS region
  std::vector<int> commit_vars;
  std::vector<int64_t> commit_bytes;
  std::unordered_map<int, std::vector<int64_t>> var_shapes;   // shape id -> dims
  // pass state (host side)
  bool running = false;
  unsigned long long pass_id = 0;
  int64_t dec_n = 0, feed_n = 0;
  size_t feed_off = 0;
  int64_t fetch_read = 0;
  std::unordered_map<int64_t, int64_t> fetch_count;             // node -> entries seen
  std::unordered_map<int64_t, std::vector<int64_t>> fetch_idx;  // node -> ring indices
  std::vector<std::vector<double>> fetch_copy;                  // payload snapshots
  std::vector<void*> workspaces;                                // extension-op workspaces
  size_t ws_bytes = 0;
};

namespace {

struct Builder {
  coex_ctx* c;
  coex_prog* p;
  const int64_t* w;
  int64_t n;
  int64_t pos = 0;
  std::vector<char*> bufs;
  std::vector<int64_t> sizes;      // buffer bytes (views: bytes to the parent's end)
  std::vector<std::pair<char*, char*>> nv_red;   // NVLS: output ranges reduced by GEMM epilogues
  int64_t n_late = 0;
  std::string err;
  char* scratch = nullptr;         // scratch shared by the program's ops (they run in stream order)
  size_t scratch_cap = 0;

  // A scratch region of >= bytes; grows geometrically (earlier ops keep the smaller region
  // they were built with, so the total stays below twice the largest request).
  char* shared_scratch(size_t bytes) {
    if (bytes < 256) bytes = 256;
    if (bytes > scratch_cap) {
      size_t cap = scratch_cap * 2 > bytes ? scratch_cap * 2 : bytes;
      void* q = nullptr;
      if (cudaMalloc(&q, cap) != cudaSuccess) {
        cudaGetLastError();
        cap = bytes;
        if (cudaMalloc(&q, cap) != cudaSuccess) {
          cudaGetLastError();
          throw std::runtime_error("cudaMalloc(shared scratch): out of memory");
        }
      }
      p->workspaces.push_back(q);
      p->ws_bytes += cap;
      scratch = (char*)q;
      scratch_cap = cap;
    }
    return scratch;
  }

  // One chain program (T_CHAIN word after its tag) into q.
  void parse_chain(ChainParams& q) {
    memset(&q, 0, sizeof(q));
    q.ds = c->d_state;
    q.n = next();
    q.red = (int)next();
    q.red_reg = (int)next();
    q.red_buf = buf(next());
    q.red_npub = (int)next();
    for (int i = 0; i < kChainPub; ++i) {
      int64_t ci = next();
      q.red_pub[i] = i < q.red_npub ? pubcell(ci) : nullptr;
    }
    const int64_t late = next();
    q.nin = (int)next();
    for (int i = 0; i < kChainIn; ++i) {
      int64_t ci = next();
      q.in[i] = (i < q.nin) ? operand(ci) : In{nullptr, nullptr, nullptr};
      q.in_scalar[i] = (unsigned char)next();
    }
    q.nops = (int)next();
    for (int i = 0; i < kChainOps; ++i) {
      q.ops[i].op = (unsigned char)next();
      q.ops[i].dst = (unsigned char)next();
      q.ops[i].a = (unsigned char)next();
      q.ops[i].b = (unsigned char)next();
    }
    q.nout = (int)next();
    for (int j = 0; j < kChainOut; ++j) {
      q.out_reg[j] = (unsigned char)next();
      q.out_buf[j] = buf(next());
      q.npub[j] = (unsigned char)next();
      for (int i = 0; i < kChainPub; ++i) {
        int64_t ci = next();
        q.pub[j][i] = (j < q.nout && i < q.npub[j]) ? pubcell(ci) : nullptr;
      }
    }
    if (q.nin > kChainIn || q.nops > kChainOps || q.nout > kChainOut) throw std::runtime_error("chain too wide");
    q.late = late ? p->late + (n_late++) : nullptr;
  }

  int64_t next() {
    if (pos >= n) throw std::runtime_error("plan truncated");
    return w[pos++];
  }
  void** cell(int64_t i) {
    if (i < 0 || i >= p->ncells) throw std::runtime_error("bad cell index");
    return p->cells + i;
  }
  // operand codes: >= 0 program cell; -1 none; -(1000 + v) variable v (overlay, then committed)
  In operand(int64_t ci) {
    In x{nullptr, nullptr, nullptr};
    if (ci >= 0) {
      x.cell = cell(ci);
    } else if (ci <= -1000 && ci > -2000) {
      const int64_t v = -1000 - ci;
      if (v >= kMaxVars) throw std::runtime_error("bad variable operand");
      x.cell = c->d_var_cur + v;
      x.ovl = c->d_var_ovl + v;
    } else if (ci != -1) {
      throw std::runtime_error("bad operand code");
    }
    return x;
  }
  // publish codes: >= 0 program cell; -(2000 + v) variable v's overlay slot (a folded AssignVar)
  void** pubcell(int64_t ci) {
    if (ci >= 0) return cell(ci);
    if (ci <= -2000) {
      const int64_t v = -2000 - ci;
      if (v >= kMaxVars) throw std::runtime_error("bad variable publish code");
      return c->d_var_ovl + v;
    }
    throw std::runtime_error("bad publish code");
  }
  char* buf(int64_t i) {
    if (i < 0) return nullptr;
    if (i >= (int64_t)bufs.size()) throw std::runtime_error("bad buffer index");
    return bufs[i];
  }

  std::unordered_map<cudaGraphNode_t, bool> kernel_nodes;   // nodes created by add_kernel
  bool pdl = true;
  int64_t cancel_every = 64;        // kernel nodes per cancel-guarded segment (0: no guards)
  std::vector<std::pair<cudaGraph_t, cudaGraphNode_t>> pending_ar;   // async collectives not yet joined

  // Kernel node after `*prev`.  Kernel -> kernel edges are programmatic (PDL): the node is
  // scheduled while its predecessor's last wave drains and synchronises in COEX_PDL_ENTER.
  // NCCL all-reduce captured on a side stream into a child graph node after *prev.
  int add_allreduce(cudaGraph_t g, cudaGraphNode_t* prev, void* b, int64_t count, int dtype, int op) {
    NcclApi& n = nccl();
    if (!n.ok || c->comm == nullptr) throw std::runtime_error("all-reduce in a plan without a communicator");
    cudaGraph_t child;
    CK(cudaStreamBeginCapture(c->cap_stream, cudaStreamCaptureModeRelaxed));
    int r = n.all_reduce(b, b, (size_t)count, dtype, op, c->comm, c->cap_stream);
    cudaError_t ce = cudaStreamEndCapture(c->cap_stream, &child);
    if (r || ce != cudaSuccess) throw std::runtime_error("capturing ncclAllReduce failed");
    cudaGraphNode_t node;
    ce = cudaGraphAddChildGraphNode(&node, g, *prev ? prev : nullptr, *prev ? 1 : 0, child);
    cudaGraphDestroy(child);
    if (ce != cudaSuccess) throw std::runtime_error(std::string("child graph node: ") + cudaGetErrorString(ce));
    *prev = node;
    p->n_collectives++;
    return COEX_OK;
  }

  // ---- NVLS fusion (nvls.cuh) ----
  bool in_nv(const void* q) const {
    return c->nv_local != nullptr && (const char*)q >= c->nv_local + kNvlsFlagBytes &&
           (const char*)q < c->nv_local + c->nv_bytes;
  }
  // An op whose Out is an NVLS bucket member and whose result comes from ONE tcgen05 GEMM
  // (plain or split-K, no bias, no scatter / batch / triangle): the GEMM epilogue adds its
  // tiles into the multicast alias, the split-K reduction launch is dropped (every K slice
  // adds), and the range is recorded as already reduced for the bucket's all-reduce.
  void nvls_fuse(const Out& o, Launch* L, int* nL) {
    if (!in_nv(o.buf[0]) || o.pingpong) return;
    int gi = -1, ng = 0;
    for (int i = 0; i < *nL; ++i)
      if (L[i].tc_dest == 1) { gi = i; ++ng; }
    if (ng != 1 || L[gi].fn_red == nullptr) return;
    TcGemmParams* gp = (TcGemmParams*)L[gi].params;
    if (gp->has_bias || gp->cv.phases > 1 || gp->batch > 1 || gp->tri_out || gp->tri_a) return;
    for (int i = 0; i < *nL; ++i)
      if (L[i].tc_dest == 2 && ((SplitReduceParams*)L[i].params)->has_bias) return;
    const size_t bytes = (size_t)gp->M * (size_t)gp->N * 4;
    char* lo = (char*)o.buf[0];
    if (lo + bytes > c->nv_local + c->nv_bytes) return;
    L[gi].fn = L[gi].fn_red;
    L[gi].grid = dim3(L[gi].red_grid);
    L[gi].smem = L[gi].red_smem;
    gp->red.mode = c->nv_mode;
    if (c->nv_mode == RED_MC) {
      gp->red.npeers = 1;
      gp->red.delta[0] = (long long)(c->nv_mc - c->nv_local);
    } else {
      gp->red.npeers = c->nv_world;
      for (int r = 0; r < c->nv_world; ++r) gp->red.delta[r] = (long long)(c->nv_peer[r] - c->nv_local);
    }
    gp->raw = nullptr;
    int k = 0;
    for (int i = 0; i < *nL; ++i)
      if (L[i].tc_dest != 2) {
        if (k != i) L[k] = L[i];
        ++k;
      }
    *nL = k;
    nv_red.push_back({lo, lo + bytes});
    p->n_nvls_fused++;
  }
  int nvls_barrier(cudaGraph_t g, cudaGraphNode_t* prev) {
    const int slot = c->nv_next_slot++ % kNvlsSlots;
    NvlsBarrierParams q{};
    q.ds = c->d_state;
    q.mode = c->nv_mode;
    q.world = c->nv_world;
    if (c->nv_mode == RED_MC) q.flag_arrive[0] = (unsigned int*)c->nv_mc + slot;
    else for (int r = 0; r < c->nv_world; ++r) q.flag_arrive[r] = (unsigned int*)c->nv_peer[r] + slot;
    q.flag_local = (unsigned int*)c->nv_local + slot;
    q.gen = c->nv_gen + slot;
    Launch L;
    L.set((void*)k_nvls_barrier, dim3(1), dim3(32), q);
    return add_kernel(g, prev, L);
  }

  int add_kernel(cudaGraph_t g, cudaGraphNode_t* prev, Launch& L) {
    if (L.fn == nullptr && L.ar_buf != nullptr)
      return add_allreduce(g, prev, L.ar_buf, L.ar_count, L.ar_f64 ? kNcclDouble : kNcclFloat, kNcclSum);
    cudaKernelNodeParams kp = {};
    kp.func = L.fn;
    kp.gridDim = L.grid;
    kp.blockDim = L.block;
    kp.sharedMemBytes = (unsigned)L.smem;
    kp.kernelParams = L.argv();
    cudaGraphNode_t node;
    if (pdl && *prev && kernel_nodes.count(*prev)) {
      CK(cudaGraphAddKernelNode(&node, g, nullptr, 0, &kp));
      cudaGraphEdgeData ed;
      memset(&ed, 0, sizeof(ed));
      ed.from_port = cudaGraphKernelNodePortProgrammatic;
      ed.type = cudaGraphDependencyTypeProgrammatic;
      CK(cudaGraphAddDependencies_v2(g, prev, &node, &ed, 1));
    } else {
      CK(cudaGraphAddKernelNode(&node, g, *prev ? prev : nullptr, *prev ? 1 : 0, &kp));
    }
    kernel_nodes[node] = true;
    *prev = node;
    p->n_kernel_nodes++;
    return COEX_OK;
  }

  void read_out(Out& o) {
    int64_t b0 = next(), b1 = next();
    o.buf[0] = buf(b0);
    o.buf[1] = buf(b1);
    o.pingpong = (int)next();
    int64_t late = next();
    int64_t np = next();
    if (np > kMaxPub) throw std::runtime_error("too many publish cells");
    o.npub = (int)np;
    for (int i = 0; i < kMaxPub; ++i) {
      int64_t ci = next();
      o.pub[i] = (i < np) ? pubcell(ci) : nullptr;
    }
    o.late = late ? p->late + (n_late++) : nullptr;
  }

  // A straight-line list.  With cancel guards on (COEX_CANCEL_EVERY > 0, default 64) the
  // list is cut into segments of about that many kernel nodes, each the body of an IF
  // conditional set by a k_guard that reads the host's cancel word: a cancelled pass skips
  // every later segment.  All-reduce child graphs stay at the list's own level.
  int seq(cudaGraph_t g, cudaGraphNode_t* prev) {
    if (next() != T_SEQ) throw std::runtime_error("expected SEQ");
    int64_t items = next();
    cudaGraph_t body = nullptr;
    cudaGraphNode_t bprev = nullptr;
    int64_t seg0 = 0;
    auto close = [&]() -> int {
      if (body && bprev == nullptr) {            // segment without nodes: keep the body non-empty
        cudaGraphNode_t e;
        CK(cudaGraphAddEmptyNode(&e, body, nullptr, 0));
      }
      body = nullptr;
      return COEX_OK;
    };
    for (int64_t i = 0; i < items; ++i) {
      const int64_t tag = pos < n ? w[pos] : -1;
      const bool guardable = cancel_every > 0 && tag != T_ALLREDUCE && tag != T_JOIN && tag != T_NVLS_AR &&
                             tag != T_NVLS_ZERO;
      if (body && (!guardable || p->n_kernel_nodes - seg0 >= cancel_every)) {
        int rc = close();
        if (rc) return rc;
      }
      if (guardable && !body) {
        cudaGraphConditionalHandle h;
        CK(cudaGraphConditionalHandleCreate(&h, g, 0, 0));
        GuardParams gp{c->d_state, c->d_mb, h};
        Launch L;
        L.set((void*)k_guard, dim3(1), dim3(1), gp);
        int rc = add_kernel(g, prev, L);
        if (rc) return rc;
        cudaGraphNodeParams cp = {};
        cp.type = cudaGraphNodeTypeConditional;
        cp.conditional.handle = h;
        cp.conditional.type = cudaGraphCondTypeIf;
        cp.conditional.size = 1;
        cudaGraphNode_t node;
        CK(cudaGraphAddNode(&node, g, prev, 1, &cp));
        p->n_guards++;
        *prev = node;
        body = cp.conditional.phGraph_out[0];
        bprev = nullptr;
        seg0 = p->n_kernel_nodes;
      }
      int rc = body ? item(body, &bprev) : item(g, prev);
      if (rc) return rc;
    }
    return close();
  }

  int item(cudaGraph_t g, cudaGraphNode_t* prev) {
    int64_t tag = next();
    switch (tag) {
      case T_OP: {
        OpSpec s;
        s.ds = c->d_state;
        s.kind = (int)next();
        next();  // node id (diagnostics)
        for (int i = 0; i < 2; ++i) {
          int64_t ci = next();
          s.in[i] = operand(ci);
        }
        for (int i = 0; i < 2; ++i) {
          s.in_ndim[i] = (int)next();
          for (int d = 0; d < COEX_MAX_RANK; ++d) s.in_shape[i][d] = next();
        }
        s.out_ndim = (int)next();
        for (int d = 0; d < COEX_MAX_RANK; ++d) s.out_shape[d] = next();
        s.attr_n = (int)next();
        for (int d = 0; d < COEX_MAX_RANK; ++d) s.attr_dims[d] = next();
        int64_t vbits = next();
        memcpy(&s.value, &vbits, 8);
        s.trans_a = (int)next();
        s.trans_b = (int)next();
        s.scratch[0] = buf(next());
        s.scratch[1] = buf(next());
        s.in_conv[0] = (int)next();
        s.in_conv[1] = (int)next();
        {
          const int64_t bc = next();                // fused bias_add (GEMM epilogue), -1: none
          if (bc != -1) {
            s.in[2] = operand(bc);
            s.bias = 1;
          }
          s.shadow = buf(next());                   // elementwise: bf16 GEMM-operand copy, -1: none
          s.skip_f32 = (int)next();

        }
        read_out(s.out);
        s.nin = 2;
        if (needs_scratch(c, s.kind)) {           // bf16 MatMul: split-K slices when the tile grid is small
          const int64_t M = s.trans_a ? s.in_shape[0][1] : s.in_shape[0][0];
          const int64_t K = s.trans_a ? s.in_shape[0][0] : s.in_shape[0][1];
          const int64_t N = s.trans_b ? s.in_shape[1][0] : s.in_shape[1][1];
          const size_t wb = matmul_split_ws_c(c, M, N, K);
          if (wb) s.ws = shared_scratch(wb);
        }
        Launch L[kMaxLaunches];
        int nL = 0;
        int rc = build_launches(c, s, L, &nL);
        if (rc) return rc;
        nvls_fuse(s.out, L, &nL);
        p->n_compute += nL;
        for (int i = 0; i < nL; ++i) {
          rc = add_kernel(g, prev, L[i]);
          if (rc) return rc;
        }
        return COEX_OK;
      }
      case T_XOP: {
        OpSpec s;
        s.ds = c->d_state;
        s.kind = (int)next();
        next();  // node id (diagnostics)
        s.nin = (int)next();
        if (s.nin < 1 || s.nin > kMaxIn || !is_ext_compute(s.kind)) throw std::runtime_error("bad extension op");
        for (int i = 0; i < kMaxIn; ++i) {
          int64_t ci = next();
          s.in[i] = i < s.nin ? operand(ci) : In{nullptr, nullptr, nullptr};
        }
        for (int i = 0; i < kMaxIn; ++i) {
          s.in_ndim[i] = (int)next();
          for (int d = 0; d < COEX_MAX_RANK; ++d) s.in_shape[i][d] = next();
        }
        s.out_ndim = (int)next();
        for (int d = 0; d < COEX_MAX_RANK; ++d) s.out_shape[d] = next();
        s.attr_n = (int)next();
        for (int d = 0; d < COEX_MAX_RANK; ++d) s.attr_dims[d] = next();
        int64_t vbits = next();
        memcpy(&s.value, &vbits, 8);
        read_out(s.out);
        if (s.kind == kBnBwdFused || s.kind == kLnBwdFused) {
          read_out(s.out2);
          read_out(s.out3);
        } else if (s.kind == kBnAct || s.kind == kCeFused) {
          read_out(s.out2);
        }
        s.shadow = buf(next());
        for (int i = 0; i < kMaxIn; ++i) s.in_shadow[i] = buf(next());
        for (int i = 0; i < kMaxIn; ++i) s.in_conv[i] = (int)next();
        Launch L[kMaxLaunches];
        int nL = 0;
        size_t wb = 0, pzb = 0;
        int rc = build_xop(c, s, L, &nL, &wb, &pzb);
        if (rc) return rc;
        s.ws = shared_scratch(wb);   // non-null: marks the build pass
        if (pzb) {
          void* pz = nullptr;
          CK(cudaMalloc(&pz, pzb));
          CK(cudaMemset(pz, 0, pzb));
          p->workspaces.push_back(pz);
          p->ws_bytes += pzb;
          s.pz = (char*)pz;
        }
        rc = build_xop(c, s, L, &nL, &wb, &pzb);
        if (rc) return rc;
        nvls_fuse(s.out, L, &nL);
        p->n_compute += nL;
        for (int i = 0; i < nL; ++i) {
          rc = add_kernel(g, prev, L[i]);
          if (rc) return rc;
        }
        return COEX_OK;
      }
      case T_ATTN: {                                // fused causal attention (attn_tc.cuh)
        const int64_t mode = next();
        FaParams fp{};
        fp.ds = c->d_state;
        fp.BH = (int)next();
        fp.T = (int)next();
        fp.H = (int)next();
        fp.rs = next();
        {
          int64_t sb = next();
          double sc;
          memcpy(&sc, &sb, 8);
          fp.scale = (float)sc;
        }
        fp.lse = (float*)buf(next());
        fp.delta = (float*)buf(next());
        fp.tiles = (unsigned char*)buf(next());
        for (int i = 0; i < 3; ++i) fp.sh[i] = (__nv_bfloat16*)buf(next());   // -1 -> nullptr
        fp.q = operand(next());
        fp.k = operand(next());
        fp.v = operand(next());
        fp.o = operand(next());
        fp.dout = operand(next());
        fp.pa = fp.q;
        fp.pb = fp.k;
        if (is_f64(c) || fp.T % FA_BLK != 0 || fp.H < 1 || fp.BH % fp.H != 0)
          throw std::runtime_error("flash attention: bf16 mode, T % 128, BH % H");
        if (int e = fa_set_attrs()) return e;
        p->n_compute++;
        const unsigned pb = fa_prep_blocks(fp);
        if (mode == 0) {
          read_out(fp.out);
          Launch L0, L1;
          L0.set((void*)k_fa_prep_qkv, dim3(pb, 3), dim3(256), fp);
          L1.set((void*)k_fa_fwd, dim3(fa_fwd_blocks(fp)), dim3(FA_THREADS), fp);
          L1.smem = kFaFwdSmem;
          int rc = add_kernel(g, prev, L0);
          if (!rc) rc = add_kernel(g, prev, L1);
          return rc;
        }
        read_out(fp.out);
        read_out(fp.out2);
        read_out(fp.out3);
        const unsigned blocks = (unsigned)(fp.BH * (fp.T / FA_BLK));
        Launch L0, L1, L2;
        L0.set((void*)k_fa_prep_do, dim3(pb), dim3(256), fp);
        L1.set((void*)k_fa_bwd_kv, dim3(blocks), dim3(FA_THREADS), fp);
        L1.smem = kFaKvSmem;
        L2.set((void*)k_fa_bwd_q, dim3(blocks), dim3(FA_THREADS), fp);
        L2.smem = kFaQSmem;
        int rc = add_kernel(g, prev, L0);
        if (!rc) rc = add_kernel(g, prev, L1);
        if (!rc) rc = add_kernel(g, prev, L2);
        return rc;
      }
      case T_MCHAIN: {                              // independent chains, one launch
        const int64_t cnt = next();
        if (cnt < 1 || cnt > kMaxMultiChain) throw std::runtime_error("bad multi-chain count");
        MultiChainParams* mq = new MultiChainParams();
        memset(mq, 0, sizeof(*mq));
        mq->ds = c->d_state;
        mq->count = (int)cnt;
        int64_t blocks = 0;
        for (int64_t j = 0; j < cnt; ++j) {
          if (next() != T_CHAIN) throw std::runtime_error("multi-chain member is not a chain");
          parse_chain(mq->c[j]);
          if (mq->c[j].red) throw std::runtime_error("multi-chain member reduces");
          mq->off[j] = (int)blocks;
          blocks += grid_for(mq->c[j].n).x;
        }
        mq->off[cnt] = (int)blocks;
        Launch L;
        if (is_f64(c)) L.set((void*)k_chain_multi<double>, dim3((unsigned)blocks), dim3(256), *mq);
        else L.set((void*)k_chain_multi<float>, dim3((unsigned)blocks), dim3(256), *mq);
        delete mq;
        p->n_compute++;
        return add_kernel(g, prev, L);
      }
      case T_CHAIN: {
        ChainParams q;
        parse_chain(q);
        Launch L;
        if (q.red) {
          if (is_f64(c)) L.set((void*)k_chain_reduce<double, true>, dim3(1), dim3(256), q);
          else L.set((void*)k_chain_reduce<float, false>, dim3(1), dim3(256), q);
        } else {
          if (is_f64(c)) L.set((void*)k_chain<double>, grid_for(q.n), dim3(256), q);
          else L.set((void*)k_chain<float>, grid_for(q.n), dim3(256), q);
        }
        p->n_compute++;
        return add_kernel(g, prev, L);
      }
      case T_ALLREDUCE: {
        void* b = buf(next());
        const int64_t count = next();
        const int64_t avg = next();
        const int64_t async = next();
        // the collective is captured on a side stream into a child graph node (a child node
        // keeps conditional bodies simple).  async (gradient buckets): a side branch off the
        // chain -- the following compute does not wait for it; a later T_JOIN (placed by the
        // planner before the first reader) does
        if (!async)
          return add_allreduce(g, prev, b, count, is_f64(c) ? kNcclDouble : kNcclFloat, avg ? kNcclAvg : kNcclSum);
        cudaGraphNode_t branch = *prev;
        int rc = add_allreduce(g, &branch, b, count, is_f64(c) ? kNcclDouble : kNcclFloat, avg ? kNcclAvg : kNcclSum);
        if (rc) return rc;
        pending_ar.push_back({g, branch});
        return COEX_OK;
      }
      case T_NVLS_ZERO: {                           // list start: red targets zeroed on every rank
        char* lo = buf(next());
        const int64_t last = next();
        if (last < 0 || last >= (int64_t)bufs.size()) throw std::runtime_error("bad NVLS zero range");
        char* hi = bufs[last] + sizes[last];
        if (!in_nv(lo) || !in_nv(hi - 1) || hi <= lo) throw std::runtime_error("NVLS zero range outside the region");
        NvlsZeroParams q{};
        q.ds = c->d_state;
        q.p = (float4*)lo;
        q.n4 = (int64_t)((hi - lo + 15) / 16);
        Launch L;
        L.set((void*)k_nvls_zero, grid_for(q.n4), dim3(256), q);
        int rc = add_kernel(g, prev, L);
        if (rc) return rc;
        return nvls_barrier(g, prev);               // no rank adds before every copy is zero
      }
      case T_NVLS_AR: {                             // bucket over the multicast region
        char* lo = buf(next());
        const int64_t count = next();
        const int64_t avg = next();
        const int64_t async = next();
        char* hi = lo + count * 4;
        if (is_f64(c) || !in_nv(lo) || !in_nv(hi - 1)) throw std::runtime_error("bad NVLS bucket");
        // spans of the bucket the GEMM epilogues did not reduce (other producers' outputs)
        std::vector<std::pair<char*, char*>> red;
        for (auto& r : nv_red)
          if (r.second > lo && r.first < hi) red.push_back(r);
        std::sort(red.begin(), red.end());
        if (avg && !red.empty()) throw std::runtime_error("NVLS average bucket with GEMM-reduced members");
        std::vector<NvlsSpan> spans;
        char* cur = lo;
        for (auto& r : red) {
          if (r.first > cur) spans.push_back({(long long)((cur - c->nv_local) / 4), (long long)((r.first - cur) / 4)});
          if (r.second > cur) cur = (char*)(((uintptr_t)r.second + 15) & ~(uintptr_t)15);   // padding to the next buffer
        }
        if (cur < hi) spans.push_back({(long long)((cur - c->nv_local) / 4), (long long)((hi - cur + 3) / 4)});
        cudaGraphNode_t branch = *prev;
        cudaGraphNode_t* at = async ? &branch : prev;
        int rc = nvls_barrier(g, at);               // every rank's producers (and reds) are done
        if (rc) return rc;
        if (!spans.empty()) {
          for (size_t s0 = 0; s0 < spans.size(); s0 += kNvlsMaxSpans) {
            NvlsAllReduceParams q{};
            q.ds = c->d_state;
            q.mode = c->nv_mode;
            if (c->nv_mode == RED_MC) q.base[0] = (float*)c->nv_mc;
            else for (int r = 0; r < c->nv_world; ++r) q.base[r] = (float*)c->nv_peer[r];
            q.rank = c->rank;
            q.world = c->nv_world;
            q.scale = avg ? 1.0f / (float)c->nv_world : 1.0f;
            long long tot = 0;
            for (size_t j = s0; j < spans.size() && j < s0 + kNvlsMaxSpans; ++j) {
              q.spans[q.nspans++] = spans[j];
              tot += spans[j].n;
            }
            Launch L;
            L.set((void*)k_nvls_allreduce, grid_for(tot / 4 / (c->nv_world > 0 ? c->nv_world : 1) + 1), dim3(256), q);
            rc = add_kernel(g, at, L);
            if (rc) return rc;
          }
          rc = nvls_barrier(g, at);                 // every rank's stores landed
          if (rc) return rc;
        }
        p->n_collectives++;
        if (async) pending_ar.push_back({g, branch});
        return COEX_OK;
      }
      case T_JOIN: {                                // chain += every pending collective of this graph
        std::vector<cudaGraphNode_t> deps;
        if (*prev) deps.push_back(*prev);
        std::vector<std::pair<cudaGraph_t, cudaGraphNode_t>> keep;
        for (auto& pr : pending_ar) {
          if (pr.first == g) deps.push_back(pr.second);
          else keep.push_back(pr);
        }
        pending_ar.swap(keep);
        if (deps.size() <= 1) return COEX_OK;
        cudaGraphNode_t node;
        CK(cudaGraphAddEmptyNode(&node, g, deps.data(), deps.size()));
        *prev = node;
        return COEX_OK;
      }
      case T_PTR: {
        PtrParams q{};
        q.ds = c->d_state;
        q.op = (int)next();
        next();  // node id
        int64_t ci = next();
        q.a = operand(ci);
        int64_t vi = next();
        q.shape_id = (int)next();
        if (vi >= 0) {
          q.var_cur = c->d_var_cur + vi;
          q.var_ovl = c->d_var_ovl + vi;
          q.var_ovl_shape = c->d_var_ovl_shape + vi;
        }
        read_out(q.out);
        Launch L;
        L.set((void*)k_ptr, dim3(1), dim3(1), q);
        return add_kernel(g, prev, L);
      }
      case T_FEED: {
        FeedWaitParams q{};
        q.ds = c->d_state;
        q.mb = c->d_mb;
        q.slot = next();
        q.numel = next();
        q.ndim = (int)next();
        for (int d = 0; d < COEX_MAX_RANK; ++d) q.shape[d] = next();
        q.buf = buf(next());
        q.cell = cell(next());
        q.rec = p->recs + (int64_t)next();
        q.is_f64 = is_f64(c);
        {                                      // index feed: TO_INDEX fused into the feed
          int64_t vbits = next();
          memcpy(&q.iv, &vbits, 8);
        }
        Launch L;
        L.set((void*)k_feed_wait, dim3(1), dim3(1), q);
        int rc = add_kernel(g, prev, L);
        if (rc) return rc;
        if (q.numel > 1 || q.ndim > 0) {
          FeedFillParams f{};
          f.ds = c->d_state;
          f.rec = q.rec;
          f.arena = c->d_feed_arena;
          f.jump = c->d_jump;
          f.n = q.numel;
          f.buf = q.buf;
          f.iv = q.iv;
          const int64_t per_block = (int64_t)kSynthThreads * kSynthRun;
          int64_t blocks = (q.numel + per_block - 1) / per_block;
          if (blocks < 1) blocks = 1;
          dim3 gd((unsigned)(blocks < kNumSMs * 4 ? blocks : kNumSMs * 4));
          Launch F;
          if (is_f64(c)) F.set((void*)k_feed_fill<double>, gd, dim3(kSynthThreads), f);
          else F.set((void*)k_feed_fill<float>, gd, dim3(kSynthThreads), f);
          rc = add_kernel(g, prev, F);
        }
        return rc;
      }
      case T_FETCH: {
        FetchParams q{};
        q.ds = c->d_state;
        q.mb = c->d_mb;
        q.node = next();
        q.a = operand(next());
        q.numel = next();
        q.ndim = (int)next();
        for (int d = 0; d < COEX_MAX_RANK; ++d) q.shape[d] = next();
        q.arena = c->d_fetch_arena;
        q.arena_cap = c->fetch_cap;
        q.elsize = (int)c->esize;
        Launch L;
        L.set((void*)k_fetch, dim3(1), dim3(256), q);
        return add_kernel(g, prev, L);
      }
      case T_SWITCH: {
        int64_t branch = next();
        int64_t ncases = next();
        cudaGraphConditionalHandle h;
        CK(cudaGraphConditionalHandleCreate(&h, g, 0, 0));
        DecideParams d{};
        d.ds = c->d_state;
        d.mb = c->d_mb;
        d.handle = h;
        d.id = branch;
        d.kind = 0;
        d.skip_value = (int)ncases;
        Launch L;
        L.set((void*)k_decide, dim3(1), dim3(1), d);
        int rc = add_kernel(g, prev, L);
        if (rc) return rc;
        cudaGraphNodeParams cp = {};
        cp.type = cudaGraphNodeTypeConditional;
        cp.conditional.handle = h;
        cp.conditional.type = cudaGraphCondTypeSwitch;
        cp.conditional.size = (unsigned)ncases;
        cudaGraphNode_t node;
        CK(cudaGraphAddNode(&node, g, prev, 1, &cp));
        p->n_cond_nodes++;
        for (int64_t k = 0; k < ncases; ++k) {
          cudaGraphNode_t bprev = nullptr;
          rc = seq(cp.conditional.phGraph_out[k], &bprev);
          if (rc) return rc;
        }
        *prev = node;
        return COEX_OK;
      }
      case T_WHILE: {
        int64_t loop = next();
        cudaGraphConditionalHandle h;
        CK(cudaGraphConditionalHandleCreate(&h, g, 0, 0));
        DecideParams d{};
        d.ds = c->d_state;
        d.mb = c->d_mb;
        d.handle = h;
        d.id = loop;
        d.kind = 1;
        d.skip_value = 0;
        Launch L;
        L.set((void*)k_decide, dim3(1), dim3(1), d);
        int rc = add_kernel(g, prev, L);
        if (rc) return rc;
        cudaGraphNodeParams cp = {};
        cp.type = cudaGraphNodeTypeConditional;
        cp.conditional.handle = h;
        cp.conditional.type = cudaGraphCondTypeWhile;
        cp.conditional.size = 1;
        cudaGraphNode_t node;
        CK(cudaGraphAddNode(&node, g, prev, 1, &cp));
        p->n_cond_nodes++;
        cudaGraph_t body = cp.conditional.phGraph_out[0];
        cudaGraphNode_t bprev = nullptr;
        rc = seq(body, &bprev);
        if (rc) return rc;
        Launch L2;    // Loop-Cond at the end of the body: next LoopDecision
        L2.set((void*)k_decide, dim3(1), dim3(1), d);
        rc = add_kernel(body, &bprev, L2);
        if (rc) return rc;
        *prev = node;
        return COEX_OK;
      }
      default:
        throw std::runtime_error("unknown plan tag " + std::to_string(tag));
    }
  }
};

}  // namespace

extern "C" {

int coex_prog_build(coex_ctx* c, const int64_t* plan, int64_t nwords, const double* consts, int64_t nconsts,
                    coex_prog** out) {
  if (c->active) return fail(COEX_IN_FLIGHT_PASS, "prog_build during a pass");
  coex_prog* p = new coex_prog();
  p->ctx = c;
  Builder b{c, p, plan, nwords};
  {
    const char* e = getenv("COEX_PDL");
    b.pdl = !(e && e[0] == '0');
    const char* ce = getenv("COEX_CANCEL_EVERY");
    if (ce) b.cancel_every = atoll(ce);
    // data parallel over several ranks: every rank must run every collective it reaches, so
    // straight-line segments are not guarded (a rank that observes its cancel earlier than
    // its peers would skip an all-reduce they already entered); spinners still stop
    if (c->comm != nullptr && c->world > 1) b.cancel_every = 0;
  }
  try {
    if (b.next() != kPlanMagic || b.next() != kPlanVersion) throw std::runtime_error("bad plan header");
    const int64_t nbufs = b.next();
    std::vector<int64_t> sizes(nbufs);
    size_t total = 0;
    // a negative entry is a VIEW: -(1 + parent << 40 + byte offset) into an earlier buffer
    // (planner _arm_views: arm-exclusive activations of a SwitchCase share one region)
    for (int64_t i = 0; i < nbufs; ++i) sizes[i] = b.next();
    // NVLS plans: the listed buffers (sum-reduced gradient bucket members) live in the
    // context's multicast-mapped region instead of the arena, in index order
    const int64_t n_nv = b.next();
    std::vector<char> in_nv(nbufs, 0);
    for (int64_t i = 0; i < n_nv; ++i) {
      const int64_t bi = b.next();
      if (bi < 0 || bi >= nbufs || sizes[bi] < 0) throw std::runtime_error("bad NVLS buffer");
      in_nv[bi] = 1;
    }
    if (n_nv > 0 && c->nv_local == nullptr) throw std::runtime_error("NVLS plan without an NVLS region");
    for (int64_t i = 0; i < nbufs; ++i)
      if (sizes[i] >= 0 && !in_nv[i]) total += ((size_t)sizes[i] + 255) & ~(size_t)255;
    p->arena_bytes = total;
    size_t nv_off = kNvlsFlagBytes;
    if (total) CK(cudaMalloc(&p->arena, total));
    size_t off = 0;
    for (int64_t i = 0; i < nbufs; ++i) {
      if (sizes[i] < 0) {
        const int64_t v = -sizes[i] - 1, parent = v >> 40, boff = v & ((1ll << 40) - 1);
        if (parent < 0 || parent >= i || sizes[parent] < 0 || boff >= sizes[parent])
          throw std::runtime_error("bad buffer view");
        b.bufs.push_back((char*)b.bufs[parent] + boff);
        sizes[i] = sizes[parent] - boff;            // bound for the spare below
        continue;
      }
      if (in_nv[i]) {
        if (nv_off + (size_t)sizes[i] > c->nv_bytes) throw std::runtime_error("NVLS region too small for the plan");
        b.bufs.push_back(c->nv_local + nv_off);
        nv_off += ((size_t)sizes[i] + 255) & ~(size_t)255;
        continue;
      }
      b.bufs.push_back(p->arena + off);
      off += ((size_t)sizes[i] + 255) & ~(size_t)255;
    }
    b.sizes = sizes;
    p->ncells = b.next();
    std::vector<void*> init(p->ncells > 0 ? p->ncells : 1, nullptr);
    for (int64_t i = 0; i < p->ncells; ++i) init[i] = b.buf(b.next());
    // cells without a buffer (pointer ops, merged bindings of pointer ops) start at a
    // zero-filled spare as large as any tensor the program touches: a cancelled pass that
    // skipped their publisher still hands its readers valid memory
    size_t spare = 256;
    for (int64_t i = 0; i < nbufs; ++i) spare = std::max(spare, (size_t)sizes[i]);
    for (const auto& v : c->vars) spare = std::max(spare, (size_t)(v.t.numel > 0 ? v.t.numel : 1) * c->esize);
    CK(cudaMalloc(&p->spare, spare));
    CK(cudaMemset(p->spare, 0, spare));
    for (int64_t i = 0; i < p->ncells; ++i)
      if (init[i] == nullptr) init[i] = p->spare;
    CK(cudaMalloc(&p->cells, sizeof(void*) * (p->ncells > 0 ? p->ncells : 1)));
    CK(cudaMalloc(&p->cells_init, sizeof(void*) * (p->ncells > 0 ? p->ncells : 1)));
    CK(cudaMemcpy(p->cells, init.data(), sizeof(void*) * p->ncells, cudaMemcpyHostToDevice));
    CK(cudaMemcpy(p->cells_init, init.data(), sizeof(void*) * p->ncells, cudaMemcpyHostToDevice));
    const int64_t nrecs = b.next();
    CK(cudaMalloc(&p->recs, sizeof(FeedRecord) * (nrecs > 0 ? nrecs : 1)));
    const int64_t nlate = b.next();
    CK(cudaMalloc(&p->late, sizeof(unsigned int) * (nlate > 0 ? nlate : 1)));
    CK(cudaMemset(p->late, 0, sizeof(unsigned int) * (nlate > 0 ? nlate : 1)));
    // constant buffers (FILL nodes are evaluated once here)
    const int64_t nfill = b.next();
    for (int64_t i = 0; i < nfill; ++i) {
      int64_t bi = b.next(), cnt = b.next(), ci = b.next();
      if (ci < 0 || ci >= nconsts) throw std::runtime_error("bad const index");
      OpSpec s;
      s.kind = COEX_FILL;
      s.out_ndim = 1;
      s.out_shape[0] = cnt;
      s.value = consts[ci];
      s.out.buf[0] = b.buf(bi);
      if (cnt > 0) {
        Launch L;
        int rc = build_launch(c, s, &L);
        if (rc == COEX_OK) rc = launch_now(c, L);
        if (rc) throw std::runtime_error(g_err);
      }
    }
    // variables committed by this program
    const int64_t ncommit = b.next();
    if (ncommit > kMaxVars) throw std::runtime_error("too many assigned variables");
    for (int64_t i = 0; i < ncommit; ++i) {
      p->commit_vars.push_back((int)b.next());
      p->commit_bytes.push_back(b.next());
    }
    const int64_t nshapes = b.next();
    for (int64_t i = 0; i < nshapes; ++i) {
      int sid = (int)b.next();
      int64_t nd = b.next();
      std::vector<int64_t> dims;
      for (int64_t d = 0; d < nd; ++d) dims.push_back(b.next());
      p->var_shapes[sid] = dims;
    }
    CK(cudaGraphCreate(&p->graph, 0));
    cudaGraphNode_t prev = nullptr;
    {
      BeginParams bp{c->d_state, c->d_mb, c->d_var_ovl, (int)c->vars.size() > 0 ? (int)kMaxVars : 0};
      bp.nvars = kMaxVars;
      bp.cells = p->cells;
      bp.cells_init = p->cells_init;
      bp.ncells = p->ncells;
      Launch L;
      L.set((void*)k_pass_begin, dim3(1), dim3(256), bp);
      int rc = b.add_kernel(p->graph, &prev, L);
      if (rc) throw std::runtime_error(g_err);
    }
    int rc = b.seq(p->graph, &prev);
    if (rc) throw std::runtime_error(g_err);
    {
      GateParams gp{c->d_state, c->d_mb};
      Launch L;
      L.set((void*)k_commit_gate, dim3(1), dim3(1), gp);
      rc = b.add_kernel(p->graph, &prev, L);
      if (rc) throw std::runtime_error(g_err);
    }
    for (size_t base = 0; base < p->commit_vars.size(); base += kMaxCommit) {   // kMaxCommit per launch
      CommitParams cp{};
      cp.ds = c->d_state;
      cp.n = (int)std::min((size_t)kMaxCommit, p->commit_vars.size() - base);
      for (int i = 0; i < cp.n; ++i) {
        cp.var_index[i] = p->commit_vars[base + i];
        cp.bytes[i] = p->commit_bytes[base + i];
      }
      cp.var_cur = c->d_var_cur;
      cp.var_ovl = c->d_var_ovl;
      cp.var_spare = c->d_var_spare;
      Launch L;
      int64_t maxb = 0;
      for (int i = 0; i < cp.n; ++i) maxb = cp.bytes[i] > maxb ? cp.bytes[i] : maxb;
      int64_t gx = (maxb / 16 + 255) / 256;
      gx = gx < 1 ? 1 : (gx > kNumSMs ? kNumSMs : gx);
      L.set((void*)k_commit, dim3((unsigned)gx, cp.n), dim3(256), cp);
      rc = b.add_kernel(p->graph, &prev, L);
      if (rc) throw std::runtime_error(g_err);
    }
    {
      EndParams ep{c->d_state, c->d_mb, c->d_var_ovl, c->d_var_ovl_shape, (int)c->vars.size()};
      Launch L;
      L.set((void*)k_pass_end, dim3(1), dim3(32), ep);
      rc = b.add_kernel(p->graph, &prev, L);
      if (rc) throw std::runtime_error(g_err);
    }
    if (b.pos != nwords) throw std::runtime_error("trailing plan words");
    cudaError_t e = cudaGraphInstantiate(&p->exec, p->graph, 0);
    if (e != cudaSuccess) throw std::runtime_error(std::string("cudaGraphInstantiate: ") + cudaGetErrorString(e));
    e = cudaStreamSynchronize(c->stream);
    if (e != cudaSuccess) throw std::runtime_error(std::string("build sync: ") + cudaGetErrorString(e));
  } catch (const std::exception& ex) {
    coex_prog_destroy(p);
    return fail(COEX_INVALID, std::string("coex_prog_build: ") + ex.what() + (g_err.empty() ? "" : " / " + g_err));
  }
  *out = p;
  return COEX_OK;
}

int coex_prog_destroy(coex_prog* p) {
  if (p == nullptr) return COEX_OK;
  coex_ctx* c = p->ctx;
  if (c && c->active == p) return fail(COEX_IN_FLIGHT_PASS, "destroying a running program");
  if (c) cudaStreamSynchronize(c->stream);
  if (p->exec) cudaGraphExecDestroy(p->exec);
  if (p->graph) cudaGraphDestroy(p->graph);
  if (p->arena) cudaFree(p->arena);
  if (p->cells) cudaFree(p->cells);
  if (p->cells_init) cudaFree(p->cells_init);
  if (p->spare) cudaFree(p->spare);
  if (p->recs) cudaFree(p->recs);
  if (p->late) cudaFree(p->late);
  for (void* w : p->workspaces) cudaFree(w);
  delete p;
  return COEX_OK;
}

int coex_prog_nvls(coex_prog* p, int64_t* fused) {
  *fused = p ? p->n_nvls_fused : 0;
  return COEX_OK;
}

int coex_prog_info(coex_prog* p, int64_t* nk, int64_t* nc, int64_t* ab) {
  *nk = p->n_kernel_nodes;
  *nc = p->n_cond_nodes;
  *ab = (int64_t)(p->arena_bytes + p->ws_bytes);
  return COEX_OK;
}

// =============================================================== passes
static double now_s() {
  return std::chrono::duration<double>(std::chrono::steady_clock::now().time_since_epoch()).count();
}

int coex_pass_begin(coex_prog* p) {
  coex_ctx* c = p->ctx;
  if (c->active) return fail(COEX_IN_FLIGHT_PASS, "a pass is already in flight");
  // spare buffers for the variables this program may commit
  for (size_t i = 0; i < p->commit_vars.size(); ++i) {
    Var& v = c->vars[p->commit_vars[i]];
    size_t need = (size_t)p->commit_bytes[i];
    if (v.spare && (v.spare->refs != 1 || v.spare->bytes < need)) {
      release(c, v.spare);
      v.spare = nullptr;
    }
    if (!v.spare) {
      int rc = alloc_buf(c, need, &v.spare);
      if (rc) return rc;
    }
    c->h_var_spare[p->commit_vars[i]] = v.spare->ptr;
  }
  if (!p->commit_vars.empty())
    CK(cudaMemcpyAsync(c->d_var_spare, c->h_var_spare, sizeof(void*) * c->vars.size(), cudaMemcpyHostToDevice,
                       c->stream));
  p->pass_id = ++c->pass_counter;
  p->dec_n = p->feed_n = 0;
  p->feed_off = 0;
  p->fetch_read = 0;
  p->fetch_count.clear();
  p->fetch_idx.clear();
  p->fetch_copy.clear();
  c->mb->done = 0;
  c->mb->dec_consumed = 0;
  c->mb->feed_consumed = 0;
  c->mb->pass_id = p->pass_id;
  std::atomic_thread_fence(std::memory_order_seq_cst);
  CK(cudaGraphLaunch(p->exec, c->stream));
  c->kernel_count += p->n_compute;
  c->active = p;
  p->running = true;
  return COEX_OK;
}

static int publish_wait(coex_prog* p, volatile long long* consumed, int64_t next_idx, int cap) {
  coex_ctx* c = p->ctx;
  double t0 = 0;
  while (next_idx - *consumed >= cap) {
    if (t0 == 0) t0 = now_s();
    if (c->mb->done == p->pass_id) return fail(COEX_CHANNEL_CLOSED, "pass ended while the host was publishing");
    if (now_s() - t0 > c->timeout_s) return fail(COEX_CHANNEL_CLOSED, "ring full: device not consuming");
  }
  return COEX_OK;
}

static int push_decision(coex_prog* p, int kind, int64_t id, int value) {
  coex_ctx* c = p->ctx;
  if (c->active != p) return fail(COEX_CHANNEL_CLOSED, "no pass in flight");
  int rc = publish_wait(p, &c->mb->dec_consumed, p->dec_n, kDecCap);
  if (rc) return rc;
  DecEntry* e = &c->mb->dec[p->dec_n % kDecCap];
  e->id = id;
  e->kind = kind;
  e->value = value;
  std::atomic_thread_fence(std::memory_order_release);
  e->seq = seq_of(p->pass_id, p->dec_n);
  p->dec_n++;
  return COEX_OK;
}

int coex_pass_case(coex_prog* p, int64_t branch_id, int32_t case_index) {
  return push_decision(p, 0, branch_id, case_index);
}
int coex_pass_loop(coex_prog* p, int64_t loop_id, int32_t cont) { return push_decision(p, 1, loop_id, cont ? 1 : 0); }

static int push_feed(coex_prog* p, int64_t slot, int type, int ndim, const int64_t* shape, const double* data,
                     uint64_t state, const void* dptr) {
  coex_ctx* c = p->ctx;
  if (c->active != p) return fail(COEX_CHANNEL_CLOSED, "no pass in flight");
  if (ndim < 0 || ndim > COEX_MAX_RANK) return fail(COEX_INVALID, "rank out of range");
  int rc = publish_wait(p, &c->mb->feed_consumed, p->feed_n, kFeedCap);
  if (rc) return rc;
  FeedEntry* e = &c->mb->feed[p->feed_n % kFeedCap];
  const int64_t n = numel_of(ndim, shape);
  e->slot = slot;
  e->ndim = ndim;
  for (int d = 0; d < ndim; ++d) e->shape[d] = shape[d];
  e->type = type;
  e->state = state;
  e->dptr = dptr;
  if (type == FEED_HOST && n == 1 && ndim == 0) {
    e->type = FEED_SCALAR;
    e->scalar = data[0];
  } else if (type == FEED_HOST) {
    if (p->feed_off + (size_t)n > c->feed_cap) return fail(COEX_CHANNEL_CLOSED, "feed arena exhausted this pass");
    memcpy(c->feed_arena + p->feed_off, data, n * sizeof(double));
    e->off = p->feed_off;
    p->feed_off += ((size_t)n + 1) & ~(size_t)1;
  }
  std::atomic_thread_fence(std::memory_order_release);
  e->seq = seq_of(p->pass_id, p->feed_n);
  p->feed_n++;
  return COEX_OK;
}

int coex_pass_feed(coex_prog* p, int64_t slot, int ndim, const int64_t* shape, const double* data) {
  return push_feed(p, slot, FEED_HOST, ndim, shape, data, 0, nullptr);
}
int coex_pass_feed_mapped(coex_prog* p, int64_t slot, int ndim, const int64_t* shape, const double* data) {
  coex_ctx* c = p->ctx;
  const char* d = (const char*)data;
  const size_t bytes = (size_t)numel_of(ndim, shape) * sizeof(double);
  for (const auto& r : c->pinned) {
    if (d >= r.first && d + bytes <= r.first + r.second) {
      void* dev = nullptr;
      CK(cudaHostGetDevicePointer(&dev, r.first, 0));
      return push_feed(p, slot, FEED_MAPPED, ndim, shape, nullptr, 0, (const char*)dev + (d - r.first));
    }
  }
  return fail(COEX_INVALID, "coex_pass_feed_mapped: payload is not inside a registered host range");
}
int coex_host_register(coex_ctx* c, void* ptr, int64_t bytes) {
  if (ptr == nullptr || bytes <= 0) return fail(COEX_INVALID, "coex_host_register: empty range");
  CK(cudaHostRegister(ptr, (size_t)bytes, cudaHostRegisterMapped | cudaHostRegisterReadOnly));
  c->pinned.emplace_back((char*)ptr, (size_t)bytes);
  return COEX_OK;
}
int coex_host_unregister(coex_ctx* c, void* ptr) {
  for (size_t i = 0; i < c->pinned.size(); ++i) {
    if (c->pinned[i].first == (char*)ptr) {
      cudaStreamSynchronize(c->stream);
      CK(cudaHostUnregister(ptr));
      c->pinned.erase(c->pinned.begin() + (long)i);
      return COEX_OK;
    }
  }
  return fail(COEX_INVALID, "coex_host_unregister: range not registered");
}
int coex_pass_feed_synth(coex_prog* p, int64_t slot, uint64_t state, int ndim, const int64_t* shape) {
  return push_feed(p, slot, FEED_SYNTH, ndim, shape, nullptr, state, nullptr);
}
int coex_pass_feed_tensor(coex_prog* p, int64_t slot, int64_t tid) {
  TRec* t = get_t(p->ctx, tid);
  if (!t) return fail(COEX_INVALID, "unknown tensor id");
  return push_feed(p, slot, FEED_DEVICE, t->ndim, t->shape, nullptr, 0, t->buf ? t->buf->ptr : nullptr);
}

int coex_pass_fetch(coex_prog* p, int64_t node, int64_t occ, double* out, int64_t cap, int* ndim, int64_t* shape) {
  coex_ctx* c = p->ctx;
  if (c->active != p) return fail(COEX_CHANNEL_CLOSED, "no pass in flight");
  double t0 = 0;
  while (true) {
    auto it = p->fetch_idx.find(node);
    if (it != p->fetch_idx.end() && (int64_t)it->second.size() > occ) {
      const FetchEntry* e = &c->mb->fetch[it->second[occ] % kFetchCap];
      const std::vector<double>& data = p->fetch_copy[it->second[occ]];
      if (cap < e->numel) return fail(COEX_INVALID, "fetch buffer too small");
      *ndim = e->ndim;
      for (int d = 0; d < e->ndim; ++d) shape[d] = e->shape[d];
      memcpy(out, data.data(), sizeof(double) * e->numel);
      return COEX_OK;
    }
    // drain newly published entries in order
    const FetchEntry* e = &c->mb->fetch[p->fetch_read % kFetchCap];
    if (e->seq == seq_of(p->pass_id, p->fetch_read)) {
      std::atomic_thread_fence(std::memory_order_acquire);
      std::vector<double> v(e->numel);
      if (c->prec == COEX_F64) {
        memcpy(v.data(), c->fetch_arena + e->off, sizeof(double) * e->numel);
      } else {
        const float* f = (const float*)(c->fetch_arena + e->off);
        for (int64_t i = 0; i < e->numel; ++i) v[i] = (double)f[i];
      }
      p->fetch_copy.push_back(std::move(v));
      p->fetch_idx[e->node].push_back(p->fetch_read);
      p->fetch_read++;
      continue;
    }
    if (c->mb->done == p->pass_id) {
      int st = c->mb->status;
      if (st == 3) return fail(COEX_DECISION_MISMATCH, "device reported a decision mismatch");
      if (st == 9) return fail(COEX_SHAPE_MISS, "fed shape differs from the graph specialisation");
      return fail(COEX_CHANNEL_CLOSED, "pass ended without the requested fetch");
    }
    if (t0 == 0) t0 = now_s();
    else if (now_s() - t0 > c->timeout_s) return fail(COEX_CHANNEL_CLOSED, "fetch timed out");
  }
}

int coex_pass_cancel(coex_prog* p) {
  coex_ctx* c = p->ctx;
  if (c->active != p) return COEX_OK;
  c->mb->cancel = p->pass_id;
  std::atomic_thread_fence(std::memory_order_seq_cst);
  return COEX_OK;
}

int coex_pass_wait(coex_prog* p, coex_pass_stats* st) {
  coex_ctx* c = p->ctx;
  if (c->active != p) return fail(COEX_CHANNEL_CLOSED, "no pass in flight");
  if (c->mb->cancel != p->pass_id && c->mb->done != p->pass_id) {
    int rc = push_decision(p, 2, -1, 0);          // commit token: the skeleton reached StepEnd
    if (rc) return rc;
  }
  double t0 = now_s();
  while (c->mb->done != p->pass_id) {
    if (now_s() - t0 > c->timeout_s) {
      c->mb->cancel = p->pass_id;     // unblock any spinner, then report
      cudaStreamSynchronize(c->stream);
      c->active = nullptr;
      p->running = false;
      return fail(COEX_CHANNEL_CLOSED, "pass did not finish before the timeout");
    }
  }
  std::atomic_thread_fence(std::memory_order_acquire);
  CK(cudaStreamSynchronize(c->stream));
  c->active = nullptr;
  p->running = false;
  const Mailbox* mb = c->mb;
  if (st) {
    st->committed = mb->committed;
    st->status = mb->status;
    st->exec_ms = mb->exec_ns * 1e-6;
    st->stall_ms = mb->stall_ns * 1e-6;
    st->ops = mb->ops;
    st->fetches = mb->fetches;
    st->dirty_mask = mb->dirty_mask;
  }
  if (mb->committed) {
    // host bookkeeping of committed variables: the spare became the value
    for (size_t i = 0; i < p->commit_vars.size(); ++i) {
      int vi = p->commit_vars[i];
      if (vi >= kMaxVars || !((mb->dirty[vi / 64] >> (vi % 64)) & 1ull)) continue;
      Var& v = c->vars[vi];
      Buf* old = v.t.buf;
      v.t.buf = v.spare;
      v.spare = (old && old->refs == 1) ? old : nullptr;
      if (v.spare == nullptr) release(c, old);
      // graph-mode assignments are shape-stable (the planner rejects shape changes)
      c->h_var_cur[vi] = v.t.buf->ptr;
    }
  }
  if (mb->status == 3) return fail(COEX_DECISION_MISMATCH, "device reported a decision mismatch");
  return mb->committed ? COEX_OK : COEX_CANCELLED;
}

}  // extern "C"
