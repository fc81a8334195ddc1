/*
 * coex_b200.h -- C-ABI of the B200 symbolic-execution backend (libcoexb200.so).
 *
 * Drop-in boundary for the reference's symbolic executor.  The reference (a
 * pure-Python package, /root/reference/pkg) has no FFI; its boundary for this
 * path is the Python surface each entry point below replaces:
 *
 *   coex_exec_op            <- coex.tensor.execute_kernel     pkg/src/coex/tensor.py:246-291
 *   coex_tensor_put/get     <- coex.tensor.Tensor marshalling pkg/src/coex/tensor.py:69-102
 *   coex_tensor_synth       <- coex.dataset.SyntheticDataset.next  pkg/src/coex/dataset.py:44-51
 *   coex_var_*              <- graph_runner.VariableStore / snapshot_vars / rollback
 *   coex_prog_build         <- graph_gen.structure output (SymProgram) consumed by run_pass
 *   coex_pass_begin/_wait   <- graph_runner.run_pass (Committed | Cancelled)
 *   coex_pass_case/_loop    <- ChannelSet.decisions push (CaseDecision / LoopDecision)
 *   coex_pass_feed*         <- ChannelSet.feeds push
 *   coex_pass_fetch         <- ChannelSet.fetches pop
 *   coex_pass_cancel        <- ChannelSet.cancel
 *
 * Status codes map 1:1 onto the reference's exception classes
 * (pkg/src/coex/errors.py:6-90); coex_last_error() returns the message of the
 * last failing call on the calling thread.  All data crosses the ABI as
 * float64 (the reference's only dtype, tensor.py:1-11); the device stores it in
 * the context's precision.  Every call is made from one host thread (the
 * orchestrator/skeleton thread); the GPU plays the runner thread.
 */
#ifndef COEX_B200_H
#define COEX_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum coex_status {
  COEX_OK = 0,
  COEX_SHAPE_MISMATCH = 1,   /* errors.ShapeMismatch */
  COEX_BAD_ATTRS = 2,        /* errors.BadAttrs */
  COEX_DECISION_MISMATCH = 3,/* errors.DecisionMismatch */
  COEX_CHANNEL_CLOSED = 4,   /* errors.ChannelClosed (peer failed / timeout) */
  COEX_CANCELLED = 5,        /* pass ended Cancelled */
  COEX_IN_FLIGHT_PASS = 6,   /* errors.InFlightPass */
  COEX_BUDGET = 7,           /* errors.BudgetExceeded */
  COEX_CUDA_ERROR = 8,       /* device / driver failure */
  COEX_SHAPE_MISS = 9,       /* fed shape differs from the graph's specialisation */
  COEX_INVALID = 10          /* bad handle / argument */
};

/* OpKind codes (order of coex.tensor.OpKind, tensor.py:30-44), followed by the extension
 * op set for configs C2-C5 (no reference counterpart -- semantics in
 * oracle/kernels.py).  Extension ops take up to 3 tensor inputs; convolutions carry
 * [kernel, stride, pad] in coex_attrs.dims[0..2]; NHWC layout, weights [k*k*Cin, Cout]. */
enum coex_opkind {
  COEX_MATMUL = 0, COEX_ADD, COEX_SUB, COEX_MUL, COEX_NEG, COEX_RELU, COEX_SIGMOID,
  COEX_SUM, COEX_MEAN, COEX_TRANSPOSE, COEX_RESHAPE, COEX_FILL, COEX_READ_VAR, COEX_ASSIGN_VAR,
  COEX_CONV2D = 14,        /* (x [N,H,W,C], w [k*k*C, F]) -> [N,Ho,Wo,F] */
  COEX_CONV2D_T,           /* (x [N,H,W,C], w [k*k*F, C]) -> [N,(H-1)s-2p+k,..,F] (conv2d input grad) */
  COEX_CONV2D_DW,          /* (x [N,H,W,C], dy [N,Ho,Wo,F]) -> [k*k*C, F] (conv2d weight grad) */
  COEX_BATCHNORM,          /* (x [..,C], gamma [C], beta [C]) -> batch-statistics normalisation */
  COEX_BATCHNORM_DX,       /* (x, gamma, dy) -> dx */
  COEX_BN_DGAMMA,          /* (x, dy) -> [C] = sum_rows(dy * xhat) */
  COEX_SUM_ROWS,           /* (x [..,C]) -> [C] */
  COEX_TANH, COEX_LEAKY_RELU, COEX_RELU_GRAD, COEX_LEAKY_RELU_GRAD, COEX_BCE_TERM,
  /* transformer extension (config C4): coex_attrs.dims[0] = vocab (embedding_dw),
   * coex_attrs.value = softmax scale (causal_softmax, softmax_grad) */
  COEX_TO_INDEX = 26,      /* (u, V) -> clip(floor((u+1)/2*V), 0, V-1) */
  COEX_EMBEDDING,          /* (table [V, d], ids [..]) -> [.., d] */
  COEX_EMBEDDING_DW,       /* (ids [..], dy [.., d]) -> [V, d] scatter-add */
  COEX_LAYERNORM,          /* (x [.., d], gamma [d], beta [d]) */
  COEX_LAYERNORM_DX,       /* (x, gamma, dy) -> dx */
  COEX_LN_DGAMMA,          /* (x, dy) -> [d] */
  COEX_BIAS_ADD,           /* (x [.., d], b [d]) */
  COEX_GELU, COEX_GELU_GRAD,
  COEX_BMM, COEX_BMM_NT, COEX_BMM_TN,   /* batched a.b, a.b^T, a^T.b ([B, ., .]) */
  COEX_CAUSAL_SOFTMAX,     /* (x [.., T, T]) -> row softmax of scale*x over j <= i */
  COEX_SOFTMAX_GRAD,       /* (y, dy) -> scale*y*(dy - sum(dy*y)) */
  COEX_CROSS_ENTROPY,      /* (logits [R, V], ids [R]) -> mean loss */
  COEX_CROSS_ENTROPY_GRAD, /* -> (softmax - onehot) / R */
  /* relative attention (config C5, Music Transformer) */
  COEX_REL_SKEW = 42,      /* (x [.., T, T]) -> y[i, j] = x[i, T-1-i+j] for j <= i, else 0 */
  COEX_REL_UNSKEW,         /* adjoint: dx[i, m] = dy[i, m-(T-1)+i] for m >= T-1-i, else 0 */
  /* ResNet-50 / SDPoint (config C3): coex_attrs.dims = [kernel, stride, pad] */
  COEX_CONV2D_DX = 44,     /* (dy, w [k*k*C, F], x [N,H,W,C]) -> conv2d's input gradient, x's shape */
  COEX_MAXPOOL,            /* (x) -> [N,Ho,Wo,C], -inf padding */
  COEX_MAXPOOL_GRAD,       /* (x, dy) -> dy routed to each window's first argmax */
  COEX_AVGPOOL,            /* (x) -> window sum / k^2, zero padding */
  COEX_AVGPOOL_GRAD,       /* (x, dy) -> covering dy sum / k^2 */
  COEX_GLOBAL_AVGPOOL,     /* (x [N,H,W,C]) -> [N,C] */
  COEX_GLOBAL_AVGPOOL_GRAD,/* (x, dy [N,C]) -> dy / (H*W) broadcast */
  /* general extension ops: Adam's elementwise sqrt / div; data movement; axis reductions
   * (coex_attrs.dims = [axis, start, length] for slice, [axis] for concat / sum_axis) */
  COEX_SQRT = 51,          /* (x) -> sqrt(x) */
  COEX_DIV,                /* (a, b) -> a / b, rank-0 broadcast */
  COEX_SLICE,              /* (x) -> x[.., start:start+length, ..] along axis */
  COEX_CONCAT,             /* (a, b) -> joined along axis */
  COEX_SUM_AXIS,           /* (x) -> sequential sum along axis (axis removed) */
  COEX_NUM_KINDS
};

/* Device storage / arithmetic precision of a context. */
enum coex_precision {
  COEX_F64 = 0,   /* parity mode: bitwise equal to the reference except Sigmoid (<= few ulp) */
  COEX_F32 = 1,   /* fp32 storage and arithmetic (<= 1e-5 relative) */
  COEX_BF16 = 2   /* fp32 storage, MatMul on tcgen05 with bf16 operands (<= 2e-2 relative) */
};

#define COEX_MAX_RANK 8

typedef struct coex_ctx coex_ctx;
typedef struct coex_prog coex_prog;

/* Op attributes: perm (TRANSPOSE), target_shape (RESHAPE), shape + value (FILL). */
typedef struct coex_attrs {
  int32_t n;                      /* entries used in dims */
  int64_t dims[COEX_MAX_RANK];
  double value;                   /* FILL value */
} coex_attrs;

typedef struct coex_pass_stats {
  int32_t committed;              /* 1 = Committed, 0 = Cancelled */
  int32_t status;                 /* coex_status of the device side */
  double exec_ms;                 /* device time of the pass (begin..end kernels) */
  double stall_ms;                /* device time spent waiting on decisions/feeds */
  int64_t ops;                    /* compute kernels executed */
  int64_t fetches;                /* fetch entries published */
  uint64_t dirty_mask;            /* vars committed by this pass (first 64 var indices) */
} coex_pass_stats;

const char* coex_last_error(void);
const char* coex_version(void);
/* Launch shape of the tcgen05 bf16 GEMM for an [M,K] x [K,N] MatMul (tile width bn, split-K
 * count, 1 = two CTAs per SM): host-only query for tests / tuning (no context needed). */
int coex_gemm_plan(int64_t M, int64_t N, int64_t K, int allow_split, int* bn, int* splits, int* duo);

/* ---- context ---- */
int coex_ctx_create(int device, int precision, coex_ctx** out);
int coex_ctx_destroy(coex_ctx* ctx);
int coex_ctx_sync(coex_ctx* ctx);
int coex_ctx_set_timeout(coex_ctx* ctx, double seconds);
/* Number of compute kernels this context launched eagerly or replayed in graphs. */
int64_t coex_ctx_kernel_count(coex_ctx* ctx);

/* ---- data parallelism (one process per GPU; NCCL over NVLink, loaded at run time) ----
 * Rank 0 calls coex_nccl_unique_id, the host plumbing (torch.distributed) broadcasts the 128
 * bytes, every rank calls coex_ctx_init_comm.  Plans of a sharded SymProgram then contain
 * all-reduce nodes (ncclAllReduce captured into the pass graph). */
int coex_nccl_unique_id(uint8_t* out128);
int coex_ctx_init_comm(coex_ctx* ctx, int rank, int world, const uint8_t* uid128);

/* ---- GEMM -> all-reduce fusion over NVLink SHARP multicast (csrc/nvls.cuh) ----
 * Replaces the NCCL gradient buckets of a data-parallel plan (the reference has no
 * distributed path).  Set-up, once per context, with a host
 * barrier (torch.distributed) between the steps:
 *   rank 0: coex_nvls_create(bytes, world) -> {pid, fd, rounded bytes} (broadcast them);
 *   every rank: coex_nvls_attach(pid, fd, bytes, world); barrier; coex_nvls_bind; barrier.
 * Plans built afterwards place sum-reduced gradient buckets in the region: their GEMM
 * producers add into the multicast alias from the epilogue (multimem.red), other members
 * are reduced by a one-shot multimem.ld_reduce / multimem.st kernel. */
int coex_nvls_supported(coex_ctx* ctx, int* out);          /* CU_DEVICE_ATTRIBUTE_MULTICAST_SUPPORTED */
int coex_nvls_create(coex_ctx* ctx, int64_t bytes, int world, int64_t* out_pid_fd_bytes);
int coex_nvls_attach(coex_ctx* ctx, int64_t pid, int64_t fd, int64_t bytes, int world);
int coex_nvls_bind(coex_ctx* ctx);
int coex_nvls_info(coex_ctx* ctx, int64_t* out3);          /* {usable bytes (0: none), world, mode 1 MC / 2 P2P} */
/* Same protocol without a multicast object (cuMulticastCreate unavailable): each rank's
 * region is a cudaMalloc exported by CUDA IPC; the epilogues add into every peer's copy over
 * NVLink.  rank: coex_p2p_create -> 64-byte handle; all-gather; coex_p2p_open(all handles). */
int coex_p2p_create(coex_ctx* ctx, int64_t bytes, uint8_t* out_handle64);
int coex_p2p_open(coex_ctx* ctx, const uint8_t* handles, int world);
int coex_prog_nvls(coex_prog* prog, int64_t* fused_gemms); /* GEMMs reducing in their epilogue */

/* ---- timing on the context's stream (bench.py; CUDA events, not host clocks) ---- */
int coex_ctx_event_record(coex_ctx* ctx, int slot);               /* slot in [0, 64) */
int coex_ctx_event_elapsed(coex_ctx* ctx, int a, int b, double* ms);
/* Launch one op `reps` times back to back between two events; average device ms per launch. */
int coex_exec_op_timed(coex_ctx* ctx, int kind, const coex_attrs* attrs, int nin, const int64_t* in_ids,
                       int reps, double* avg_ms);

/* Per-launch profile of one op's lowering (up to 6 launches): average device ms of each launch
 * repeated `reps` times; kernel names into names[j * name_cap]. */
int coex_exec_op_profile(coex_ctx* ctx, int kind, const coex_attrs* attrs, int nin, const int64_t* in_ids,
                         int reps, double* ms, int* nlaunch, char* names, int name_cap);

/* Fused causal attention (csrc/attn_tc.cuh, tcgen05; fp32 / bf16 modes) outside a graph: the
 * kernels the step graph runs for a planner attention group (T_ATTN) -- SURVEY §8(f)2; no
 * reference counterpart (its op set is closed, pkg/src/coex/tensor.py:30-44), parity is against
 * the unfused composition bmm_nt -> causal_softmax -> bmm (oracle/kernels.py).  Head dim 64, T a
 * multiple of 128, fp32 [BH][T][64] operands.  backward = 0: in {q, k, v} -> out {O, lse [BH][T]}
 * (lse in log2 units of scale*q.k); backward = 1: in {q, k, v, O, dO, lse} -> out {dQ, dK, dV}.
 * reps > 0 re-launches the kernels reps times between CUDA events: *avg_ms per repetition. */
int coex_flash_attn(coex_ctx* ctx, int backward, const int64_t* in_ids, int BH, int T, double scale, int reps,
                    int64_t* out_ids, double* avg_ms);

/* Device-side per-kernel stamps (%globaltimer, kernel kind) for the next passes (0 = off).
 * coex_ctx_read_trace returns n (time_ns, kind) pairs of the last pass. */
int coex_ctx_set_trace(coex_ctx* ctx, int capacity);
int coex_ctx_read_trace(coex_ctx* ctx, uint64_t* out_pairs, int64_t cap, int64_t* n);

/* ---- tensors (eager side) ---- */
int coex_tensor_put(coex_ctx* ctx, int ndim, const int64_t* shape, const double* data, int64_t* id);
int coex_tensor_synth(coex_ctx* ctx, uint64_t state, int ndim, const int64_t* shape, int64_t* id);
/* Index inputs: the same, with TO_INDEX(u, index_v) (pkg tensor extension, oracle
 * clip(floor((u+1)/2*V), 0, V-1)) applied to each f64 value before it is stored in the compute
 * precision -- an fp32-rounded u can move floor() across an integer.  index_v <= 0: plain put. */
int coex_tensor_put_index(coex_ctx* ctx, int ndim, const int64_t* shape, const double* data, double index_v,
                          int64_t* id);
int coex_tensor_synth_index(coex_ctx* ctx, uint64_t state, int ndim, const int64_t* shape, double index_v,
                            int64_t* id);
int coex_tensor_get(coex_ctx* ctx, int64_t id, double* out, int64_t cap, int* ndim, int64_t* shape);
int coex_tensor_info(coex_ctx* ctx, int64_t id, int* ndim, int64_t* shape);
int coex_tensor_free(coex_ctx* ctx, int64_t id);
int coex_exec_op(coex_ctx* ctx, int kind, const coex_attrs* attrs, int nin, const int64_t* in_ids,
                 int64_t* out_id);

/* ---- variable store ---- */
int coex_var_define(coex_ctx* ctx, const char* name, int64_t tensor_id, int* var_index);
int coex_var_read(coex_ctx* ctx, int var_index, int64_t* tensor_id);
int coex_var_assign(coex_ctx* ctx, int var_index, int64_t tensor_id);
int coex_var_info(coex_ctx* ctx, int var_index, int* ndim, int64_t* shape);
int coex_var_rollback(coex_ctx* ctx);

/* ---- symbolic programs ---- */
/* plan: int64 words produced by the host planner (paper_2201_09210_b200/planner.py). */
int coex_prog_build(coex_ctx* ctx, const int64_t* plan, int64_t nwords, const double* consts,
                    int64_t nconsts, coex_prog** out);
int coex_prog_destroy(coex_prog* prog);
int coex_prog_info(coex_prog* prog, int64_t* n_kernel_nodes, int64_t* n_cond_nodes, int64_t* arena_bytes);

/* ---- one pass (one co-execution step) ---- */
int coex_pass_begin(coex_prog* prog);
int coex_pass_case(coex_prog* prog, int64_t branch_id, int32_t case_index);
int coex_pass_loop(coex_prog* prog, int64_t loop_id, int32_t cont);
int coex_pass_feed(coex_prog* prog, int64_t slot, int ndim, const int64_t* shape, const double* data);
int coex_pass_feed_synth(coex_prog* prog, int64_t slot, uint64_t state, int ndim, const int64_t* shape);
int coex_pass_feed_tensor(coex_prog* prog, int64_t slot, int64_t tensor_id);
/* Host payload already in registered (pinned, mapped) memory: the feed kernel reads it in
 * place over the bus -- no staging copy into the feed arena.  `data` must lie inside a range
 * registered with coex_host_register. */
int coex_pass_feed_mapped(coex_prog* prog, int64_t slot, int ndim, const int64_t* shape, const double* data);
/* Page-lock and map a host range for coex_pass_feed_mapped (cudaHostRegister, read-only). */
int coex_host_register(coex_ctx* ctx, void* ptr, int64_t bytes);
int coex_host_unregister(coex_ctx* ctx, void* ptr);
int coex_pass_fetch(coex_prog* prog, int64_t node_id, int64_t occurrence, double* out, int64_t cap,
                    int* ndim, int64_t* shape);
int coex_pass_cancel(coex_prog* prog);
int coex_pass_wait(coex_prog* prog, coex_pass_stats* stats);

#ifdef __cplusplus
}
#endif
#endif /* COEX_B200_H */
