"""The B200 backend: ctypes binding of libcoexb200.so (include/coex_b200.h).

* :class:`B200Backend` implements the backend protocol of :mod:`.runner_api`
  on the device: eager ops for imperative / tracing / replay steps, the device
  variable store, and symbolic passes.
* :class:`B200Program` caches one CUDA graph per shape signature of a
  SymProgram (built by :mod:`.planner`, instantiated by ``coex_prog_build``).
* :class:`B200Pass` is the skeleton's side of one pass: decisions and feeds
  are published to the pinned mapped rings, fetches spin on the fetch ring.
  Lazy mode withholds publication (and the launch) until a fetch or StepEnd.

There is no CPU fallback: constructing a backend without the built library or
without a CUDA device raises.
"""

from __future__ import annotations

import ctypes
import os
import struct

import numpy as np

from .dataset import SyntheticTensor
from .errors import STATUS, ChannelClosed, CoexError, DeviceError, ShapeMiss
from .planner import Planner, slot_code
from .runner_api import PassResult
from .tensor import CONV_ATTR_KINDS, OpKind, Tensor, shape_size
from .trace_graph import CaseDecision, LoopDecision

_F64 = struct.Struct("<d")
LIB_NAME = "libcoexb200.so"
MAX_RANK = 8
PRECISIONS = {"f64": 0, "fp32": 1, "bf16": 2}


class CoexAttrs(ctypes.Structure):
    _fields_ = [("n", ctypes.c_int32), ("dims", ctypes.c_int64 * MAX_RANK), ("value", ctypes.c_double)]


class CoexPassStats(ctypes.Structure):
    _fields_ = [("committed", ctypes.c_int32), ("status", ctypes.c_int32), ("exec_ms", ctypes.c_double),
                ("stall_ms", ctypes.c_double), ("ops", ctypes.c_int64), ("fetches", ctypes.c_int64),
                ("dirty_mask", ctypes.c_uint64)]


_P = ctypes.c_void_p
_I64 = ctypes.c_int64
_I64P = ctypes.POINTER(ctypes.c_int64)
_DP = ctypes.POINTER(ctypes.c_double)
_IP = ctypes.POINTER(ctypes.c_int)

SIGNATURES = {
    "coex_last_error": (ctypes.c_char_p, []),
    "coex_version": (ctypes.c_char_p, []),
    "coex_gemm_plan": (ctypes.c_int, [_I64, _I64, _I64, ctypes.c_int, ctypes.POINTER(ctypes.c_int),
                                      ctypes.POINTER(ctypes.c_int), ctypes.POINTER(ctypes.c_int)]),
    "coex_ctx_create": (ctypes.c_int, [ctypes.c_int, ctypes.c_int, ctypes.POINTER(_P)]),
    "coex_ctx_destroy": (ctypes.c_int, [_P]),
    "coex_ctx_sync": (ctypes.c_int, [_P]),
    "coex_ctx_set_timeout": (ctypes.c_int, [_P, ctypes.c_double]),
    "coex_ctx_kernel_count": (_I64, [_P]),
    "coex_ctx_event_record": (ctypes.c_int, [_P, ctypes.c_int]),
    "coex_ctx_event_elapsed": (ctypes.c_int, [_P, ctypes.c_int, ctypes.c_int, _DP]),
    "coex_exec_op_timed": (ctypes.c_int, [_P, ctypes.c_int, ctypes.POINTER(CoexAttrs), ctypes.c_int, _I64P,
                                          ctypes.c_int, _DP]),
    "coex_exec_op_profile": (ctypes.c_int, [_P, ctypes.c_int, ctypes.POINTER(CoexAttrs), ctypes.c_int, _I64P,
                                            ctypes.c_int, _DP, ctypes.POINTER(ctypes.c_int), ctypes.c_char_p,
                                            ctypes.c_int]),
    "coex_flash_attn": (ctypes.c_int, [_P, ctypes.c_int, _I64P, ctypes.c_int, ctypes.c_int, ctypes.c_double,
                                       ctypes.c_int, _I64P, _DP]),
    "coex_nccl_unique_id": (ctypes.c_int, [ctypes.c_char_p]),
    "coex_ctx_init_comm": (ctypes.c_int, [_P, ctypes.c_int, ctypes.c_int, ctypes.c_char_p]),
    "coex_nvls_supported": (ctypes.c_int, [_P, ctypes.POINTER(ctypes.c_int)]),
    "coex_nvls_create": (ctypes.c_int, [_P, ctypes.c_int64, ctypes.c_int, ctypes.POINTER(ctypes.c_int64)]),
    "coex_nvls_attach": (ctypes.c_int, [_P, ctypes.c_int64, ctypes.c_int64, ctypes.c_int64, ctypes.c_int]),
    "coex_nvls_bind": (ctypes.c_int, [_P]),
    "coex_nvls_info": (ctypes.c_int, [_P, ctypes.POINTER(ctypes.c_int64)]),
    "coex_prog_nvls": (ctypes.c_int, [_P, ctypes.POINTER(ctypes.c_int64)]),
    "coex_p2p_create": (ctypes.c_int, [_P, ctypes.c_int64, ctypes.c_char_p]),
    "coex_p2p_open": (ctypes.c_int, [_P, ctypes.c_char_p, ctypes.c_int]),
    "coex_ctx_set_trace": (ctypes.c_int, [_P, ctypes.c_int]),
    "coex_ctx_read_trace": (ctypes.c_int, [_P, ctypes.POINTER(ctypes.c_uint64), _I64, _I64P]),
    "coex_tensor_put": (ctypes.c_int, [_P, ctypes.c_int, _I64P, _DP, _I64P]),
    "coex_tensor_synth": (ctypes.c_int, [_P, ctypes.c_uint64, ctypes.c_int, _I64P, _I64P]),
    "coex_tensor_put_index": (ctypes.c_int, [_P, ctypes.c_int, _I64P, _DP, ctypes.c_double, _I64P]),
    "coex_tensor_synth_index": (ctypes.c_int, [_P, ctypes.c_uint64, ctypes.c_int, _I64P, ctypes.c_double, _I64P]),
    "coex_tensor_get": (ctypes.c_int, [_P, _I64, _DP, _I64, _IP, _I64P]),
    "coex_tensor_info": (ctypes.c_int, [_P, _I64, _IP, _I64P]),
    "coex_tensor_free": (ctypes.c_int, [_P, _I64]),
    "coex_exec_op": (ctypes.c_int, [_P, ctypes.c_int, ctypes.POINTER(CoexAttrs), ctypes.c_int, _I64P, _I64P]),
    "coex_var_define": (ctypes.c_int, [_P, ctypes.c_char_p, _I64, _IP]),
    "coex_var_read": (ctypes.c_int, [_P, ctypes.c_int, _I64P]),
    "coex_var_assign": (ctypes.c_int, [_P, ctypes.c_int, _I64]),
    "coex_var_info": (ctypes.c_int, [_P, ctypes.c_int, _IP, _I64P]),
    "coex_var_rollback": (ctypes.c_int, [_P]),
    "coex_prog_build": (ctypes.c_int, [_P, _I64P, _I64, _DP, _I64, ctypes.POINTER(_P)]),
    "coex_prog_destroy": (ctypes.c_int, [_P]),
    "coex_prog_info": (ctypes.c_int, [_P, _I64P, _I64P, _I64P]),
    "coex_pass_begin": (ctypes.c_int, [_P]),
    "coex_pass_case": (ctypes.c_int, [_P, _I64, ctypes.c_int32]),
    "coex_pass_loop": (ctypes.c_int, [_P, _I64, ctypes.c_int32]),
    "coex_pass_feed": (ctypes.c_int, [_P, _I64, ctypes.c_int, _I64P, _DP]),
    "coex_pass_feed_synth": (ctypes.c_int, [_P, _I64, ctypes.c_uint64, ctypes.c_int, _I64P]),
    "coex_pass_feed_tensor": (ctypes.c_int, [_P, _I64, _I64]),
    "coex_pass_feed_mapped": (ctypes.c_int, [_P, _I64, ctypes.c_int, _I64P, _DP]),
    "coex_host_register": (ctypes.c_int, [_P, ctypes.c_void_p, _I64]),
    "coex_host_unregister": (ctypes.c_int, [_P, ctypes.c_void_p]),
    "coex_pass_fetch": (ctypes.c_int, [_P, _I64, _I64, _DP, _I64, _IP, _I64P]),
    "coex_pass_cancel": (ctypes.c_int, [_P]),
    "coex_pass_wait": (ctypes.c_int, [_P, ctypes.POINTER(CoexPassStats)]),
}

_LIB = None


def lib_path() -> str:
    return os.path.join(os.path.dirname(os.path.abspath(__file__)), LIB_NAME)


def load_library():
    """Load the in-tree libcoexb200.so; raise (no fallback) when it is missing."""
    global _LIB
    if _LIB is None:
        path = lib_path()
        if not os.path.exists(path):
            raise DeviceError(f"{path} is not built; run __graft_entry__.build() "
                              "(there is no CPU fallback for the B200 backend)")
        lib = ctypes.CDLL(path)
        for name, (res, args) in SIGNATURES.items():
            fn = getattr(lib, name)
            fn.restype = res
            fn.argtypes = args
        _LIB = lib
    return _LIB


def _check(rc: int):
    if rc != 0:
        msg = _LIB.coex_last_error().decode(errors="replace")
        raise STATUS.get(rc, CoexError)(msg)


def _shape_arr(shape):
    a = (ctypes.c_int64 * MAX_RANK)()
    for i, d in enumerate(shape):
        a[i] = int(d)
    return a


def _attrs(kind: OpKind, attrs: dict) -> CoexAttrs:
    at = CoexAttrs()
    if kind is OpKind.TRANSPOSE:
        dims = attrs["perm"]
    elif kind is OpKind.RESHAPE:
        dims = attrs["target_shape"]
    elif kind is OpKind.FILL:
        dims = attrs["shape"]
        at.value = float(attrs["value"])
    elif kind in CONV_ATTR_KINDS:
        dims = attrs["conv"]
    elif kind in (OpKind.EMBEDDING_DW, OpKind.SLICE, OpKind.CONCAT, OpKind.SUM_AXIS):
        dims = attrs["dims"]
    elif kind in (OpKind.CAUSAL_SOFTMAX, OpKind.SOFTMAX_GRAD):
        dims = ()
        at.value = float(attrs["value"])
    elif kind is OpKind.CROSS_ENTROPY_GRAD:
        dims = ()
        at.value = float(attrs.get("rows", 0.0))
    else:
        dims = ()
    if len(dims) > MAX_RANK:
        raise CoexError(f"rank {len(dims)} exceeds {MAX_RANK}")
    at.n = len(dims)
    for i, d in enumerate(dims):
        at.dims[i] = int(d)
    return at


def gemm_plan(M: int, N: int, K: int, allow_split: bool = True) -> tuple:
    """(tile width, split-K count, two-CTA variant) the runtime picks for a bf16 MatMul."""
    lib = load_library()
    bn, sp, duo = ctypes.c_int(), ctypes.c_int(), ctypes.c_int()
    _check(lib.coex_gemm_plan(M, N, K, int(allow_split), ctypes.byref(bn), ctypes.byref(sp), ctypes.byref(duo)))
    return bn.value, sp.value, bool(duo.value)


class DevTensor:
    """A device tensor handle owned by a context (freed on GC)."""

    __slots__ = ("be", "id", "shape", "__weakref__")

    def __init__(self, be, tid: int, shape: tuple):
        self.be = be
        self.id = tid
        self.shape = tuple(shape)

    def __del__(self):
        be = self.be
        if be is not None and be.ctx is not None and _LIB is not None:
            _LIB.coex_tensor_free(be.ctx, self.id)

    def size(self):
        return shape_size(self.shape)


class B200Backend:
    """Backend protocol (runner_api.py) on one B200 through libcoexb200.so."""

    name = "b200"

    def __init__(self, device: int = 0, precision: str = "f64", timeout_s: float = 120.0, dp=None):
        self.lib = load_library()
        self.dp = dp
        if precision not in PRECISIONS:
            raise ValueError(f"precision must be one of {sorted(PRECISIONS)}")
        self.precision = precision
        self.esize = 8 if precision == "f64" else 4
        ctx = _P()
        _check(self.lib.coex_ctx_create(device, PRECISIONS[precision], ctypes.byref(ctx)))
        self.ctx = ctx
        self.lib.coex_ctx_set_timeout(ctx, timeout_s)
        self.var_idx: dict = {}
        self._vshape: dict = {}
        self.active = None
        self.op_log = None            # list: record (kind, attrs, input shapes) of eager ops
        self.nvls_bytes = 0           # NVLS gradient region (csrc/nvls.cuh); 0 = NCCL buckets
        self.nvls_mode = "none"
        if dp is not None and (dp.world > 1 or dp.force):
            self._init_comm()
            if precision != "f64" and self._nvls_wanted():
                self._init_nvls(int(os.environ.get("COEX_NVLS_MB", "1024")) << 20)

    def _nvls_wanted(self) -> bool:
        """COEX_NVLS=0: off; 1: on (multicast, else the P2P transport -- also for a forced
        1-rank group); p2p: the P2P transport; unset: on when the group spans several GPUs and
        a multicast object can be created (P2P reductions send R x the bytes of the
        switch-reduced path, so the default then falls back to the NCCL buckets)."""
        mode = os.environ.get("COEX_NVLS", "")
        if mode == "0":
            return False
        if mode in ("1", "p2p"):
            return True
        ok = ctypes.c_int(0)
        _check(self.lib.coex_nvls_supported(self.ctx, ctypes.byref(ok)))
        return bool(ok.value) and self.dp.world > 1

    def _init_nvls(self, nbytes: int):
        """GEMM -> all-reduce fusion region over the data-parallel group (csrc/nvls.cuh,
        include/coex_b200.h).  Multicast: rank 0 creates the object and exports a POSIX fd,
        every rank imports it (pidfd_getfd) and adds its device, then binds its own copy, with
        host barriers between the phases.  P2P: every rank exports its region by CUDA IPC and
        opens the others'."""
        world, mode = self.dp.world, os.environ.get("COEX_NVLS", "")
        if world > 1:                 # (torch is already up under torchrun; a 1-rank group never imports it)
            import torch.distributed as dist
        info = (ctypes.c_int64 * 3)()
        vals = [0, 0, 0, 0]
        if mode != "p2p" and self.dp.rank == 0:
            if self.lib.coex_nvls_create(self.ctx, nbytes, world, info) == 0:
                vals = [1, int(info[0]), int(info[1]), int(info[2])]
        if world > 1:
            obj = [vals]
            dist.broadcast_object_list(obj, src=0)
            vals = obj[0]
        def agree(ok: bool) -> bool:
            """every rank's verdict (a rank that cannot import the fd -- e.g. pidfd_getfd
            refused by the ptrace policy -- sends the whole group back to NCCL)"""
            if world == 1:
                return ok
            flags = [None] * world
            dist.all_gather_object(flags, bool(ok))
            return all(flags)

        if vals[0] and agree(self.lib.coex_nvls_attach(self.ctx, vals[1], vals[2], vals[3], world) == 0):
            if not agree(self.lib.coex_nvls_bind(self.ctx) == 0):
                raise DeviceError("NVLS multicast bind failed on some rank: " +
                                  self.lib.coex_last_error().decode(errors="replace"))
        elif vals[0] and mode != "1":
            return                                   # multicast unusable on some rank: NCCL buckets
        elif mode in ("1", "p2p"):
            h = ctypes.create_string_buffer(64)
            _check(self.lib.coex_p2p_create(self.ctx, nbytes, h))
            handles = [bytes(h.raw)]
            if world > 1:
                handles = [None] * world
                dist.all_gather_object(handles, bytes(h.raw))
            allh = ctypes.create_string_buffer(b"".join(handles), 64 * world)
            _check(self.lib.coex_p2p_open(self.ctx, allh, world))
            if world > 1:
                dist.barrier()
        else:
            return                                   # no multicast: NCCL buckets
        out = (ctypes.c_int64 * 3)()
        _check(self.lib.coex_nvls_info(self.ctx, out))
        self.nvls_bytes = int(out[0])
        self.nvls_mode = {1: "multicast", 2: "p2p"}.get(int(out[2]), "none")

    def _init_comm(self):
        """NCCL communicator over the caller's torch.distributed group (rank 0 makes the id)."""
        uid = ctypes.create_string_buffer(128)
        if self.dp.world > 1:
            import torch.distributed as dist
            if self.dp.rank == 0:
                _check(self.lib.coex_nccl_unique_id(uid))
            obj = [bytes(uid.raw)]
            dist.broadcast_object_list(obj, src=0)
            uid = ctypes.create_string_buffer(obj[0], 128)
        else:
            _check(self.lib.coex_nccl_unique_id(uid))
        _check(self.lib.coex_ctx_init_comm(self.ctx, self.dp.rank, self.dp.world, uid))

    def close(self):
        if self.ctx is not None:
            for prog in getattr(self, "_programs", []):   # graphs, arenas and workspaces first
                prog.close()
            self._programs = []
            self.lib.coex_ctx_destroy(self.ctx)      # also unregisters pinned host ranges
            self.ctx = None
            self._pinned = []

    def kernel_count(self) -> int:
        return int(self.lib.coex_ctx_kernel_count(self.ctx))

    def sync(self):
        _check(self.lib.coex_ctx_sync(self.ctx))

    def event(self, slot: int):
        """Record CUDA event ``slot`` on the context's stream."""
        _check(self.lib.coex_ctx_event_record(self.ctx, slot))

    def elapsed_ms(self, a: int, b: int) -> float:
        ms = ctypes.c_double()
        _check(self.lib.coex_ctx_event_elapsed(self.ctx, a, b, ctypes.byref(ms)))
        return ms.value

    STAMP_KINDS = {0: "begin", 1: "elementwise", 2: "reduce", 3: "transpose", 4: "matmul", 5: "ptr-op",
                   6: "decide", 7: "feed-wait", 8: "feed-fill", 9: "fetch", 10: "commit-gate", 11: "commit",
                   12: "end", 13: "fused chain", 14: "im2col", 15: "col2im", 16: "bf16 cvt", 17: "colstats",
                   18: "bn apply", 19: "split-K reduce", 20: "causal softmax", 21: "softmax grad",
                   22: "cross-entropy", 23: "bias add", 24: "layernorm", 25: "embedding", 26: "column sum",
                   27: "rel skew", 28: "pooling", 29: "axis op", 30: "cancel guard",
                   31: "attention fwd", 32: "attention prep", 33: "attention dK/dV", 34: "attention dQ",
                   35: "nvls all-reduce"}

    def set_trace(self, capacity: int):
        """Enable device-side per-kernel stamps (0 disables)."""
        _check(self.lib.coex_ctx_set_trace(self.ctx, capacity))

    def read_trace(self) -> list:
        """[(t_ns, kind, after_wait)] of the last pass."""
        cap = 8192
        buf = (ctypes.c_uint64 * (2 * cap))()
        n = ctypes.c_int64()
        _check(self.lib.coex_ctx_read_trace(self.ctx, buf, cap, ctypes.byref(n)))
        return [(buf[2 * i], buf[2 * i + 1] & 63, bool(buf[2 * i + 1] & 64)) for i in range(n.value)]

    def time_op(self, kind: OpKind, attrs: dict, values: list, reps: int = 50) -> float:
        """Average device ms of one launch of ``kind`` (CUDA events on the context stream)."""
        devs = [self.put(v) for v in values]
        at = _attrs(kind, attrs)
        ids = (ctypes.c_int64 * 3)(*[d.id for d in devs], *([0] * (3 - len(devs))))
        ms = ctypes.c_double()
        _check(self.lib.coex_exec_op_timed(self.ctx, kind.code, ctypes.byref(at), len(devs), ids, reps,
                                           ctypes.byref(ms)))
        return ms.value

    def flash_attention(self, values: list, scale: float, backward: bool = False, reps: int = 0):
        """Fused causal attention (csrc/attn_tc.cuh) eagerly: forward ``[q, k, v]`` -> ``(O, lse)``,
        backward ``[q, k, v, O, dO, lse]`` -> ``(dQ, dK, dV)``; fp32 ``[BH, T, 64]`` operands.
        With ``reps`` > 0 also the average device ms of one (re-launched) repetition."""
        devs = [v if isinstance(v, DevTensor) else self.put(v) for v in values]
        BH, T = devs[0].shape[0], devs[0].shape[1]
        ids = (ctypes.c_int64 * 6)(*[d.id for d in devs], *([0] * (6 - len(devs))))
        outs = (ctypes.c_int64 * 3)()
        ms = ctypes.c_double()
        _check(self.lib.coex_flash_attn(self.ctx, 1 if backward else 0, ids, BH, T, float(scale), reps, outs,
                                        ctypes.byref(ms)))
        if backward:
            res = tuple(DevTensor(self, outs[i], (BH, T, 64)) for i in range(3))
        else:
            res = (DevTensor(self, outs[0], (BH, T, 64)), DevTensor(self, outs[1], (BH, T)))
        return (res, ms.value) if reps > 0 else res

    def profile_op(self, kind: OpKind, attrs: dict, values: list, reps: int = 20) -> list:
        """[(kernel name, average device ms)] for every launch of the op's lowering."""
        import re
        devs = [self.put(v) for v in values]
        at = _attrs(kind, attrs)
        ids = (ctypes.c_int64 * 3)(*[d.id for d in devs], *([0] * (3 - len(devs))))
        ms = (ctypes.c_double * 8)()
        n = ctypes.c_int()
        cap = 256
        names = ctypes.create_string_buffer(8 * cap)
        _check(self.lib.coex_exec_op_profile(self.ctx, kind.code, ctypes.byref(at), len(devs), ids, reps, ms,
                                             ctypes.byref(n), names, cap))
        out = []
        for j in range(n.value):
            raw = names.raw[j * cap:(j + 1) * cap].split(b"\0", 1)[0].decode(errors="replace")
            m = re.search(r"(k_[A-Za-z0-9_]+)", raw)
            out.append((m.group(1) if m else raw, ms[j]))
        return out

    # ------------------------------------------------------------ eager side
    def put(self, t) -> DevTensor:
        if isinstance(t, DevTensor):
            return t
        tid = ctypes.c_int64()
        if isinstance(t, SyntheticTensor):
            _check(self.lib.coex_tensor_synth(self.ctx, t.state, len(t.shape), _shape_arr(t.shape), ctypes.byref(tid)))
            return DevTensor(self, tid.value, t.shape)
        if not isinstance(t, Tensor):
            raise TypeError(f"cannot put {type(t).__name__}")
        data = np.ascontiguousarray(t.data, dtype=np.float64)
        _check(self.lib.coex_tensor_put(self.ctx, len(t.shape), _shape_arr(t.shape),
                                        data.ctypes.data_as(_DP), ctypes.byref(tid)))
        return DevTensor(self, tid.value, t.shape)

    def put_index(self, t, v: float) -> DevTensor:
        """TO_INDEX(t, v) of a host-side input (synthetic or host tensor), evaluated in f64 on
        the device while the values are converted to the compute precision (the op itself
        would see fp32/bf16-rounded values; include/coex_b200.h coex_tensor_put_index)."""
        tid = ctypes.c_int64()
        if isinstance(t, SyntheticTensor):
            _check(self.lib.coex_tensor_synth_index(self.ctx, t.state, len(t.shape), _shape_arr(t.shape), float(v),
                                                    ctypes.byref(tid)))
            return DevTensor(self, tid.value, t.shape)
        data = np.ascontiguousarray(t.data, dtype=np.float64)
        _check(self.lib.coex_tensor_put_index(self.ctx, len(t.shape), _shape_arr(t.shape),
                                              data.ctypes.data_as(_DP), float(v), ctypes.byref(tid)))
        return DevTensor(self, tid.value, t.shape)

    def get(self, v) -> Tensor:
        if isinstance(v, Tensor):
            return v
        if isinstance(v, SyntheticTensor):
            return v.materialize()
        out = np.empty(max(shape_size(v.shape), 1), dtype=np.float64)
        nd = ctypes.c_int()
        shp = (ctypes.c_int64 * MAX_RANK)()
        _check(self.lib.coex_tensor_get(self.ctx, v.id, out.ctypes.data_as(_DP), out.size, ctypes.byref(nd), shp))
        return Tensor._wrap(out[:shape_size(v.shape)].reshape(v.shape))

    def exec_op(self, kind: OpKind, attrs: dict, values: list) -> DevTensor:
        devs = [self.put(v) for v in values]
        if self.op_log is not None:
            self.op_log.append((kind, dict(attrs), tuple(tuple(d.shape) for d in devs)))
        at = _attrs(kind, attrs)
        ids = (ctypes.c_int64 * 3)(*[d.id for d in devs], *([0] * (3 - len(devs))))
        out = ctypes.c_int64()
        _check(self.lib.coex_exec_op(self.ctx, kind.code, ctypes.byref(at), len(devs), ids, ctypes.byref(out)))
        nd = ctypes.c_int()
        shp = (ctypes.c_int64 * MAX_RANK)()
        _check(self.lib.coex_tensor_info(self.ctx, out.value, ctypes.byref(nd), shp))
        return DevTensor(self, out.value, tuple(shp[i] for i in range(nd.value)))

    # ------------------------------------------------------------ variables
    def var_define(self, name: str, value):
        d = self.put(value)
        idx = ctypes.c_int()
        _check(self.lib.coex_var_define(self.ctx, name.encode(), d.id, ctypes.byref(idx)))
        self.var_idx[name] = idx.value
        self._vshape[name] = tuple(d.shape)

    def var_read(self, name: str) -> DevTensor:
        tid = ctypes.c_int64()
        _check(self.lib.coex_var_read(self.ctx, self.var_idx[name], ctypes.byref(tid)))
        return DevTensor(self, tid.value, self._vshape[name])

    def var_assign(self, name: str, value):
        d = self.put(value)
        _check(self.lib.coex_var_assign(self.ctx, self.var_idx[name], d.id))
        self._vshape[name] = tuple(d.shape)

    def var_shape(self, name: str) -> tuple:
        return self._vshape[name]

    def var_shapes(self) -> dict:
        return dict(self._vshape)

    # ------------------------------------------------------------ pinned host inputs
    def pin(self, array) -> None:
        """Page-lock and map a host f64 array (cudaHostRegister) so that feeding it in a pass
        is one bus crossing read by the feed kernel instead of a staging copy plus a read.
        The array must stay alive (the backend keeps a reference) and unchanged while passes
        may read it."""
        a = np.asarray(array)
        if a.dtype != np.float64 or not a.flags["C_CONTIGUOUS"] or a.nbytes == 0:
            raise CoexError("pin: a non-empty C-contiguous float64 array is required")
        if not hasattr(self, "_pinned"):
            self._pinned = []
        _check(self.lib.coex_host_register(self.ctx, ctypes.c_void_p(a.ctypes.data), a.nbytes))
        self._pinned.append((a.ctypes.data, a.nbytes, a))

    def is_pinned(self, a) -> bool:
        p, n = a.ctypes.data, a.nbytes
        return any(b <= p and p + n <= b + m for b, m, _ in getattr(self, "_pinned", ()))

    def snapshot_vars(self) -> dict:
        if self.active is not None:
            from .errors import InFlightPass
            raise InFlightPass("snapshot_vars during an in-flight pass")
        return {name: self.get(self.var_read(name)) for name in self.var_idx}

    def rollback(self):
        _check(self.lib.coex_var_rollback(self.ctx))

    # ------------------------------------------------------------ symbolic side
    def compile(self, sp, tg) -> "B200Program":
        prog = self._compile(sp, tg)
        if not hasattr(self, "_programs"):
            self._programs = []
        # a regenerated SymProgram supersedes the earlier ones: release their graphs and
        # device memory now (a program asked for a pass again rebuilds on demand)
        for old in self._programs:
            old.close()
        self._programs.append(prog)
        return prog

    def _compile(self, sp, tg) -> "B200Program":
        return B200Program(self, sp, tg)

    def begin_pass(self, prog: "B200Program", lazy: bool = False) -> "B200Pass":
        return B200Pass(self, prog, lazy)


class B200Program:
    """A SymProgram with its CUDA graphs, one per shape signature."""

    def __init__(self, be: B200Backend, sp, tg):
        self.be = be
        self.sp = sp
        self.tg = tg
        self.graphs: dict = {}
        self.feed_shape: dict = {}       # slot -> expected shape (observed hints, updated on misses)
        self.dp_plan = None
        self.varying: set = set()        # feed slots whose speculated constant missed
        for n in tg.all_nodes():
            if n.typ == "op":
                for pos, s in n.feed_shapes.items():
                    self.feed_shape[(n.id, pos)] = tuple(s)
        self.last_plan = None

    def specialise(self):
        """The (graph handle, plan) for the current variable shapes."""
        vsh = {n: self.be.var_shape(n) for n in self.be.var_idx}
        self.consts = self._const_slots()
        key = (tuple(sorted(vsh.items())), tuple(sorted(self.feed_shape.items())),
               tuple(sorted(self.consts.items())))
        hit = self.graphs.get(key)
        if hit is not None:
            return hit
        plan = self._plan(vsh)
        words = np.asarray(plan.words, dtype=np.int64)
        consts = np.asarray(plan.consts if plan.consts else [0.0], dtype=np.float64)
        handle = _P()
        _check(self.be.lib.coex_prog_build(self.be.ctx, words.ctypes.data_as(_I64P), words.size,
                                           consts.ctypes.data_as(_DP), len(plan.consts), ctypes.byref(handle)))
        self.graphs[key] = (handle, plan)
        self.last_plan = plan
        return handle, plan

    def _const_slots(self) -> dict:
        """Fed rank-0 host scalars that had one value in every trace: baked into the graph."""
        from .trace_graph import VARIES
        out = {}
        for n in self.tg.all_nodes():
            if n.typ != "op":
                continue
            for pos, v in n.feed_values.items():
                slot = (n.id, pos)
                if v is not VARIES and slot not in self.varying and tuple(n.feed_shapes.get(pos, (0,))) == ():
                    out[slot] = v
        return out

    def _plan(self, vsh):
        be = self.be
        bf16 = be.precision == "bf16"
        dp = be.dp
        if dp is not None and (dp.world > 1 or dp.force):
            from .dp import local_feed_shapes, shard_program
            from .planner import NeedsReplicated
            gshapes = Planner(self.sp, self.tg, be.var_idx, vsh, self.feed_shape, be.esize).infer_shapes()
            dplan = shard_program(self.sp, self.feed_shape, gshapes, dp.batch, dp.world, force=dp.force)
            self.dp_plan = dplan
            if not dplan.replicated:
                try:
                    plan = Planner(dplan.sp, self.tg, be.var_idx, vsh, local_feed_shapes(self.feed_shape, dplan),
                                   be.esize, bf16=bf16, force_store=dplan.allreduce_nodes,
                                   const_slots=self.consts, nvls_bytes=be.nvls_bytes).build()
                    plan.feed_shapes = dict(self.feed_shape)        # host checks global shapes
                    plan.sharded = set(dplan.sharded_slots)
                    plan.dp = dplan
                    return plan
                except NeedsReplicated as e:
                    dplan.replicated, dplan.reason = True, str(e)
        return Planner(self.sp, self.tg, be.var_idx, vsh, self.feed_shape, be.esize, bf16=bf16,
                       const_slots=self.consts).build()

    def info(self, handle) -> dict:
        nk, nc, ab, nv = ctypes.c_int64(), ctypes.c_int64(), ctypes.c_int64(), ctypes.c_int64()
        self.be.lib.coex_prog_info(handle, ctypes.byref(nk), ctypes.byref(nc), ctypes.byref(ab))
        self.be.lib.coex_prog_nvls(handle, ctypes.byref(nv))
        return {"kernel_nodes": nk.value, "conditional_nodes": nc.value, "arena_bytes": ab.value,
                "nvls_fused_gemms": nv.value}

    def close(self):
        for handle, _ in self.graphs.values():
            self.be.lib.coex_prog_destroy(handle)
        self.graphs.clear()


class B200Pass:
    """Skeleton-side channel of one in-flight pass (ChannelSet)."""

    def __init__(self, be: B200Backend, prog: B200Program, lazy: bool):
        self.be = be
        self.lib = be.lib
        self.prog = prog
        self.lazy = lazy
        self.handle, self.plan = prog.specialise()
        self.launched = False
        self.pending: list = []
        self.keep: list = []             # device tensors fed by pointer must outlive the pass
        self.cancelled = False
        self.result = None
        if not lazy:
            self._launch()

    def _launch(self):
        if self.be.active is not None:
            raise ChannelClosed("another pass is in flight")
        _check(self.lib.coex_pass_begin(self.handle))
        self.be.active = self
        self.launched = True

    def _flush(self):
        if not self.launched:
            self._launch()
        for fn, args in self.pending:
            _check(fn(*args))
        self.pending.clear()

    def _do(self, fn, *args):
        if self.lazy:
            self.pending.append((fn, (self.handle,) + args))
        else:
            _check(fn(self.handle, *args))

    def decide(self, d):
        if isinstance(d, CaseDecision):
            self._do(self.lib.coex_pass_case, d.branch_id, d.case_index)
        elif isinstance(d, LoopDecision):
            self._do(self.lib.coex_pass_loop, d.loop_id, 1 if d.cont else 0)
        else:
            raise CoexError(f"unknown decision {d!r}")

    def feed(self, slot, v):
        c = self.plan.const_slots.get(slot)
        if c is not None:
            if isinstance(v, Tensor) and v.shape == () and v.data.tobytes() == _F64.pack(c):
                return                                     # speculated constant holds: nothing to send
            self.prog.varying.add(slot)
            raise ShapeMiss(f"feed slot {slot}: value differs from the constant baked into the graph")
        want = self.plan.feed_shapes.get(slot)
        shape = tuple(v.shape)
        if want is None or tuple(want) != shape:
            self.prog.feed_shape[slot] = shape           # next specialisation uses the observed shape
            raise ShapeMiss(f"feed slot {slot}: shape {shape} but the graph expects {want}")
        code = slot_code(slot)
        if slot in getattr(self.plan, "sharded", ()):
            from .dp import shard_value
            dp = self.be.dp
            if isinstance(v, DevTensor):
                v = self.be.get(v)
            v = shard_value(v, dp.rank, dp.world)
            shape = tuple(v.shape)
        if isinstance(v, DevTensor):
            self.keep.append(v)
            self._do(self.lib.coex_pass_feed_tensor, code, v.id)
        elif isinstance(v, SyntheticTensor):
            self._do(self.lib.coex_pass_feed_synth, code, ctypes.c_uint64(v.state), len(shape), _shape_arr(shape))
        else:
            data = np.ascontiguousarray(v.data, dtype=np.float64)
            self.keep.append(data)
            if self.be.is_pinned(data):      # registered host memory: read in place by the feed kernel
                self._do(self.lib.coex_pass_feed_mapped, code, len(shape), _shape_arr(shape),
                         data.ctypes.data_as(_DP))
            else:
                self._do(self.lib.coex_pass_feed, code, len(shape), _shape_arr(shape), data.ctypes.data_as(_DP))

    def fetch(self, nid: int, k: int) -> Tensor:
        if self.lazy:
            self._flush()
        shp_expect = self.plan.node_shapes[nid]
        out = np.empty(max(shape_size(shp_expect), 1), dtype=np.float64)
        nd = ctypes.c_int()
        shp = (ctypes.c_int64 * MAX_RANK)()
        _check(self.lib.coex_pass_fetch(self.handle, nid, k, out.ctypes.data_as(_DP), out.size, ctypes.byref(nd), shp))
        shape = tuple(shp[i] for i in range(nd.value))
        return Tensor._wrap(out[:shape_size(shape)].reshape(shape))

    def cancel(self):
        self.cancelled = True
        if self.launched:
            self.lib.coex_pass_cancel(self.handle)

    def wait(self) -> PassResult:
        if self.result is not None:
            return self.result
        if not self.launched:
            if self.cancelled:
                self.result = PassResult(False)
                return self.result
            self._flush()
        elif self.lazy:
            self._flush()
        st = CoexPassStats()
        rc = self.lib.coex_pass_wait(self.handle, ctypes.byref(st))
        self.be.active = None
        self.keep.clear()
        if rc not in (0, 5):
            msg = self.lib.coex_last_error().decode(errors="replace")
            self.result = PassResult(False, st.exec_ms, st.stall_ms, st.ops, st.fetches, error=msg)
            if rc == 3:
                raise STATUS[rc](msg)
            return self.result
        self.result = PassResult(bool(st.committed), st.exec_ms, st.stall_ms, st.ops, st.fetches)
        return self.result
