"""Device plan for one SymProgram specialisation.

Turns a :class:`~.graph_gen.SymProgram` plus a shape signature (variable shapes
at pass begin, fed shapes per feed slot) into the int64 plan consumed by
``coex_prog_build`` (csrc/runtime.cu ``Builder``), which builds one CUDA graph.

Memory model:
* every ExecOp node id owns one output buffer (two when the node can read its
  own previous output, e.g. a loop-carried ``x = matmul(x, w)``); tail-duplicated
  instances of a node share it, since at most one instance runs per position;
* every value is reached through a *cell* (a device word holding a pointer):
  ``vcell[node]`` holds the node's latest output; an input with several
  candidate producers reads ``bcell[candidate set]``, which every candidate
  writes when it executes -- "latest candidate wins", the phi rule the cursor
  enforces on the host;
* RESHAPE / READ_VAR / ASSIGN_VAR only move pointers; FILL nodes are constants
  evaluated once at build time;
* each feed slot owns a buffer and a cell (re-pointed for device-resident feeds).

Transpose folding: a 2-D TRANSPOSE whose only consumers are MatMuls (and which
is not fetched) is not materialised -- the MatMul reads the operand transposed.
"""

from __future__ import annotations

import os
import struct
from dataclasses import dataclass, field

from .errors import ShapeMiss
from .graph_gen import ExecOp, InputFeed, OutputFetch, SwitchCase, SymProgram, UnrolledLoop, While
from .tensor import BMM_KINDS, CONV_ATTR_KINDS, CONV_KINDS, OpKind, flops_of, infer_shape, shape_size

MAGIC = 0xC0E8B200
VERSION = 4
T_SEQ, T_OP, T_PTR, T_FEED, T_FETCH, T_SWITCH, T_WHILE, T_CHAIN, T_ALLREDUCE, T_XOP, T_MCHAIN = 1, 2, 3, 4, 5, 6, 7, 8, 9, 10, 11
T_ATTN = 12               # fused causal attention (csrc attn_tc.cuh): forward / backward of one layer
T_JOIN = 13               # the chain waits for every asynchronous all-reduce issued so far in its list
T_NVLS_AR = 14            # gradient bucket over the NVLS multicast region (csrc/nvls.cuh)
T_NVLS_ZERO = 15          # list start: the region's red targets zeroed on every rank + barrier
AR_BUCKET_BYTES = int(os.environ.get("COEX_AR_BUCKET_MB", "64")) << 20
MAX_MCHAIN = 8            # chains per k_chain_multi launch (csrc kMaxMultiChain)
PTR_ALIAS, PTR_READ_VAR, PTR_ASSIGN_VAR = 0, 1, 2
MAX_RANK = 8
MAX_PUB = 6
# extension compute ops (conv / batch-norm families) lowered by csrc/ext_ops.cuh: T_XOP items
XOP = {OpKind.CONV2D, OpKind.CONV2D_T, OpKind.CONV2D_DW, OpKind.BATCHNORM, OpKind.BATCHNORM_DX,
       OpKind.BN_DGAMMA, OpKind.SUM_ROWS,
       OpKind.EMBEDDING, OpKind.EMBEDDING_DW, OpKind.LAYERNORM, OpKind.LAYERNORM_DX, OpKind.LN_DGAMMA,
       OpKind.BIAS_ADD, OpKind.BMM, OpKind.BMM_NT, OpKind.BMM_TN, OpKind.CAUSAL_SOFTMAX, OpKind.SOFTMAX_GRAD,
       OpKind.CROSS_ENTROPY, OpKind.CROSS_ENTROPY_GRAD, OpKind.REL_SKEW, OpKind.REL_UNSKEW,
       OpKind.CONV2D_DX, OpKind.MAXPOOL, OpKind.MAXPOOL_GRAD, OpKind.AVGPOOL, OpKind.AVGPOOL_GRAD,
       OpKind.GLOBAL_AVGPOOL, OpKind.GLOBAL_AVGPOOL_GRAD, OpKind.SLICE, OpKind.CONCAT, OpKind.SUM_AXIS}
EW_CODE = {OpKind.ADD: 0, OpKind.SUB: 1, OpKind.MUL: 2, OpKind.NEG: 3, OpKind.RELU: 4, OpKind.SIGMOID: 5,
           OpKind.TANH: 7, OpKind.LEAKY_RELU: 8, OpKind.RELU_GRAD: 9, OpKind.LEAKY_RELU_GRAD: 10,
           OpKind.BCE_TERM: 11, OpKind.TO_INDEX: 12, OpKind.GELU_GRAD: 13, OpKind.GELU: 14,
           OpKind.SQRT: 15, OpKind.DIV: 16}
COMPUTE = {OpKind.MATMUL, OpKind.SUM, OpKind.MEAN, OpKind.TRANSPOSE} | set(EW_CODE) | XOP
MAX_XIN = 3
XOP_BN_BWD = 100          # fused batchnorm_dx + bn_dgamma + sum_rows (csrc COEX_BN_BWD_FUSED)
XOP_BN_ACT = 101          # batchnorm also writing relu / leaky_relu of its output (csrc kBnAct)
XOP_CE_FUSED = 102        # cross_entropy + cross_entropy_grad in one pass (csrc kCeFused)
XOP_LN_BWD = 103          # fused layernorm_dx + ln_dgamma + sum_rows (csrc kLnBwdFused)
XOP_SKEW_ADD = 104        # add(a, rel_skew(x)) in one pass (csrc kSkewAdd)
FA_HEAD = 64              # flash attention: head dim and query / key block of the tcgen05 kernels
FA_BLOCK = 128


class _ARBucket:
    """Consecutive AllReduce items of one instruction list whose node buffers are adjacent in
    the arena: ONE collective over the span (gradient bucketing), issued asynchronously."""

    def __init__(self, members: list):
        self.members = members


class _Join:
    """The chain waits for the list's asynchronous all-reduces (before their first reader)."""


class _NvlsZero:
    """List start of an NVLS plan: zero the list's bucket buffers [first, last] on every rank
    and barrier, before any GEMM epilogue adds into them (csrc/nvls.cuh)."""

    def __init__(self, first: int, last: int):
        self.first, self.last = first, last


class _Attn:
    """Stands in for one layer's attention nodes in an instruction list: mode 0 = the forward
    (S = bmm_nt(q, k), P = causal_softmax(S), O = bmm(P, v)) at O's position, mode 1 = the
    backward (dP = bmm_nt(dO, v), dS = softmax_grad(P, dP), dQ = bmm(dS, k), dK = bmm_tn(dS, q),
    dV = bmm_tn(P, dO)) at dS's position."""

    def __init__(self, mode: int, g: dict):
        self.mode = mode
        self.g = g
CHAIN_IN, CHAIN_OPS, CHAIN_OUT, CHAIN_PUB, CHAIN_REGS = 8, 16, 8, 4, 16


def slot_code(slot: tuple) -> int:
    return slot[0] * 4 + slot[1]


def _pad(shape, n=MAX_RANK) -> list:
    s = list(shape)
    if len(s) > n:
        raise ShapeMiss(f"rank {len(s)} exceeds {n}")
    return s + [0] * (n - len(s))


def _f64_bits(x: float) -> int:
    return struct.unpack("<q", struct.pack("<d", float(x)))[0]


def walk(insts):
    """Yield every instruction (pre-order), descending into cases and loop bodies."""
    for x in insts:
        yield x
        if isinstance(x, SwitchCase):
            for c in x.cases:
                yield from walk(c)
        elif isinstance(x, While):
            yield from walk(x.body)
        elif isinstance(x, UnrolledLoop):
            if x.bodies:
                yield from walk(x.bodies[0])


@dataclass
class Plan:
    words: list
    consts: list
    signature: tuple
    n_compute: int = 0
    flops: int = 0                       # algorithmic FLOPs if every instruction ran once
    node_shapes: dict = field(default_factory=dict)
    feed_shapes: dict = field(default_factory=dict)
    folded: set = field(default_factory=set)
    n_attn: int = 0                      # flash-attention groups (one forward + one backward item each)


class Planner:
    def __init__(self, sp: SymProgram, tg, var_index: dict, var_shapes: dict, feed_shapes: dict, esize: int,
                 bf16: bool = False, fuse: bool = True, force_store=(), const_slots=None, nvls_bytes: int = 0):
        self.force_store = set(force_store)
        # data parallel over an NVLS region of this many bytes (B200Backend._init_nvls): sum
        # all-reduced gradients live there, reduced by their GEMM epilogues (csrc/nvls.cuh)
        self.nvls_bytes = int(nvls_bytes) if esize == 4 else 0
        self.const_slots = dict(const_slots or {})
        self.bf16 = bf16
        self.fuse = fuse
        self.sp = sp
        self.tg = tg
        self.var_index = var_index
        self.var_shapes = dict(var_shapes)
        self.feed_shapes = dict(feed_shapes)
        self.esize = esize
        # fp32 mode with COEX_TF32=1: MatMuls run as 3xTF32 on the tensor cores (csrc/gemm_tf32.cuh)
        # with hi / lo operand planes in per-op scratch (same switch as the runtime's tf32_on;
        # off by default, see gemm_tf32.cuh for the measured accuracy)
        self.tf32 = (not bf16) and esize == 4 and os.environ.get("COEX_TF32", "0") == "1"
        self.ops = {}           # node id -> ExecOp (first instance)
        for x in walk(sp.body):
            if isinstance(x, ExecOp) and x.node_id not in self.ops:
                self.ops[x.node_id] = x

    # ------------------------------------------------------------ shapes
    def infer_shapes(self) -> dict:
        shapes: dict = {}
        vsh = dict(self.var_shapes)

        def in_shape(b):
            if b.fed:
                s = self.feed_shapes.get(b.slot)
                if s is None:
                    raise ShapeMiss(f"no shape known for feed slot {b.slot}")
                return tuple(s)
            known = [shapes[c] for c in b.cands if c in shapes]
            if not known:
                return None
            if any(k != known[0] for k in known):
                raise ShapeMiss(f"candidates {b.cands} disagree on shape")
            return known[0]

        def go(insts, final):
            for x in insts:
                if isinstance(x, ExecOp):
                    if x.kind is OpKind.READ_VAR:
                        name = x.attrs["var_name"]
                        if name not in vsh:
                            raise ShapeMiss(f"unknown variable {name!r}")
                        s = tuple(vsh[name])
                    else:
                        ins = [in_shape(b) for b in x.inputs]
                        if any(i is None for i in ins):
                            if final:
                                raise ShapeMiss(f"node {x.node_id}: input shape unknown")
                            continue
                        s = tuple(infer_shape(x.kind, x.attrs, ins)[0])
                        if x.kind is OpKind.ASSIGN_VAR:
                            name = x.attrs["var_name"]
                            if name in self.var_shapes and tuple(self.var_shapes[name]) != s:
                                raise ShapeMiss(f"assignment changes the shape of {name!r}")
                            vsh[name] = s
                    if x.node_id in shapes and shapes[x.node_id] != s:
                        raise ShapeMiss(f"node {x.node_id} has a path-dependent shape")
                    shapes[x.node_id] = s
                elif isinstance(x, SwitchCase):
                    for c in x.cases:
                        go(c, final)
                elif isinstance(x, While):
                    go(x.body, final)
                    go(x.body, final)
                elif isinstance(x, UnrolledLoop):
                    for b in x.bodies:
                        go(b, final)

        go(self.sp.body, False)
        go(self.sp.body, True)
        return shapes

    # ------------------------------------------------------------ plan
    def _nvls_lists_ok(self, insts) -> bool:
        """Every sum all-reduce of a list has its producer inside that list (so the list-start
        zeroing of the NVLS buffers precedes every epilogue that adds into them)."""
        made = {x.node_id for x in walk(insts) if isinstance(x, ExecOp)}
        for x in insts:
            if type(x).__name__ == "AllReduce" and not x.avg and x.node_id not in made:
                return False
            subs = (x.cases if isinstance(x, SwitchCase) else [x.body] if isinstance(x, While)
                    else x.bodies if isinstance(x, UnrolledLoop) else [])
            if not all(self._nvls_lists_ok(b) for b in subs):
                return False
        return True

    def build(self) -> Plan:
        shapes = self.infer_shapes()
        # NVLS: sum all-reduced (gradient) nodes get buffers in the multicast region
        self.nvls = self.nvls_bytes > 0 and AR_BUCKET_BYTES > 0 and self._nvls_lists_ok(self.sp.body)
        self.nvls_bufs = []
        ops = self.ops
        # consumers of every node id (over all bindings)
        consumers: dict = {}
        multi: dict = {}          # frozenset(cands) -> bcell index (assigned later)
        for x in walk(self.sp.body):
            if isinstance(x, ExecOp):
                for b in x.inputs:
                    if not b.fed:
                        for c in b.cands:
                            consumers.setdefault(c, []).append(x)
                        if len(b.cands) > 1:
                            multi.setdefault(frozenset(b.cands), None)
        # transpose folding: 2-D transpose consumed only (single-candidate) by matmuls, not fetched
        folded = set()
        for nid, x in ops.items():
            if x.kind is OpKind.TRANSPOSE and tuple(x.attrs["perm"]) == (1, 0) and nid not in self.sp.fetch_nodes:
                cons = consumers.get(nid, [])
                if cons and all(c.kind is OpKind.MATMUL for c in cons) and \
                        not any(nid in s for s in multi) and not x.inputs[0].fed and len(x.inputs[0].cands) == 1 \
                        and _fold_is_local(self.sp.body, nid, x.inputs[0].cands[0]):
                    folded.add(nid)
        self.folded = folded
        # index feeds: TO_INDEX(input(..), V) with V a baked constant is applied by the feed
        # kernel to the f64 value (exact ids, see csrc index_of); the node aliases the slot
        self.index_nodes = {}
        self.index_slots = {}
        for nid, x in ops.items():
            if x.kind is OpKind.TO_INDEX and x.inputs[0].fed and x.inputs[1].fed and \
                    x.inputs[1].slot in self.const_slots and float(self.const_slots[x.inputs[1].slot]) > 0:
                self.index_nodes[nid] = x.inputs[0].slot
                self.index_slots[x.inputs[0].slot] = float(self.const_slots[x.inputs[1].slot])
        self.elided_reads, self.folded_assigns = self._pointer_rewrites(consumers, multi, folded)

        bufs: list = []

        def new_buf(nbytes):
            bufs.append(max(int(nbytes), 16))
            return len(bufs) - 1

        self.new_buf = new_buf

        def new_view(parent, offset):
            """a buffer that is a byte range of another (plan word: -(1 + parent<<40 + offset))"""
            bufs.append(-(1 + (parent << 40) + int(offset)))
            return len(bufs) - 1

        cell_init: list = []

        def new_cell(buf_idx=-1):
            cell_init.append(buf_idx)
            return len(cell_init) - 1

        node_buf: dict = {}
        self._node_buf = node_buf
        vcell: dict = {}
        fills: list = []
        consts: list = []
        # all-reduced (data-parallel gradient) nodes get adjacent buffers in program order, so
        # consecutive all-reduces of a list can run as one collective over the span
        ar_order = []
        for x in walk(self.sp.body):
            if type(x).__name__ == "AllReduce" and x.node_id not in ar_order and x.node_id in ops:
                ar_order.append(x.node_id)
        self._ar_pos = {nid: i for i, nid in enumerate(ar_order)}
        ar_set = set(ar_order)
        ar_sum = {x.node_id for x in walk(self.sp.body) if type(x).__name__ == "AllReduce" and not x.avg}
        arm_view = self._arm_views(consumers, multi, folded, shapes, new_buf, new_view)
        for nid in ar_order + [n for n in ops if n not in ar_set]:
            x = ops[nid]
            n = shape_size(shapes[nid])
            if x.kind in COMPUTE and nid not in folded and nid not in self.index_nodes:
                self_dep = any((not b.fed) and nid in b.cands for b in x.inputs)
                if self.nvls and nid in ar_sum and not self_dep:
                    b0 = new_buf(n * self.esize)            # own buffer in the multicast region
                    self.nvls_bufs.append(b0)
                else:
                    b0 = arm_view[nid] if nid in arm_view else new_buf(n * self.esize)
                b1 = new_buf(n * self.esize) if self_dep else -1
                node_buf[nid] = (b0, b1, self_dep)
                vcell[nid] = new_cell(b0)
            elif x.kind is OpKind.FILL:
                b0 = new_buf(n * self.esize)
                consts.append(float(x.attrs["value"]))
                fills.append((b0, n, len(consts) - 1))
                vcell[nid] = new_cell(b0)
            else:
                vcell[nid] = new_cell(-1)
        if self.nvls and sum((max(bufs[b], 16) + 255) // 256 * 256 for b in self.nvls_bufs) > self.nvls_bytes:
            self.nvls, self.nvls_bufs = False, []            # does not fit: NCCL buckets in the arena
        self.nvls_set = set(self.nvls_bufs)
        # bf16 shadows: a softmax-type node whose output feeds batched GEMMs as operand A also
        # writes a bf16 copy, which those GEMMs read instead of converting the fp32 tensor
        self.shadow = {}
        if self.bf16:
            def gemm_use(nid):
                """nid's output is a MatMul operand (directly or through a folded transpose)."""
                for c in consumers.get(nid, []):
                    if c.kind is OpKind.MATMUL:
                        return True
                    if c.kind is OpKind.TRANSPOSE and c.node_id in folded:
                        return True
                return False

            for nid, x in ops.items():
                if x.kind is OpKind.CROSS_ENTROPY_GRAD and nid in node_buf and not node_buf[nid][2] and \
                        gemm_use(nid) and not any(nid in s_ for s_ in multi) and \
                        any(y.kind is OpKind.CROSS_ENTROPY and y.inputs == x.inputs for y in ops.values()):
                    # the fused cross-entropy writes the gradient's bf16 copy ([rows][pitch 8])
                    shp = shapes[nid]
                    self.shadow[nid] = new_buf(shape_size(shp[:-1]) * ((shp[-1] + 7) // 8 * 8) * 2)
                    continue
                if x.kind in (OpKind.GELU, OpKind.GELU_GRAD) and nid in node_buf and not node_buf[nid][2] and \
                        shapes[nid] and shapes[nid][-1] % 8 == 0 and not any(nid in s_ for s_ in multi) and \
                        gemm_use(nid) and os.environ.get("COEX_EW_SHADOW", "1") != "0":
                    # the elementwise pass writes the bf16 copy its GEMM readers use (and skips
                    # the fp32 output when only GEMMs read it, _exec)
                    self.shadow[nid] = new_buf(shape_size(shapes[nid]) * 2)
                    continue
                if x.kind is OpKind.REL_UNSKEW and nid in node_buf and not node_buf[nid][2] and \
                        shapes[nid][-1] % 8 == 0 and not any(nid in s_ for s_ in multi) and \
                        any(c.kind is OpKind.RESHAPE and len(shapes[c.node_id]) == 2 and gemm_use(c.node_id)
                            for c in consumers.get(nid, [])):
                    # C5: the unskewed logits gradient feeds the relative-table GEMMs through a
                    # 2-D reshape; the unskew pass writes their bf16 copy
                    self.shadow[nid] = new_buf(shape_size(shapes[nid]) * 2)
                    continue
                if x.kind not in (OpKind.CAUSAL_SOFTMAX, OpKind.SOFTMAX_GRAD, OpKind.LAYERNORM) or nid not in node_buf:
                    continue
                if node_buf[nid][2] or shapes[nid][-1] % 8 or any(nid in s_ for s_ in multi):
                    continue
                if x.kind is OpKind.LAYERNORM:
                    # layernorm outputs feed the q/k/v, MLP-in and LM-head GEMMs (and their
                    # weight gradients through transposes): written once in bf16 by the producer
                    if gemm_use(nid):
                        self.shadow[nid] = new_buf(shape_size(shapes[nid]) * 2)
                    continue
                if any(c.kind in (OpKind.BMM, OpKind.BMM_TN) and not c.inputs[0].fed and c.inputs[0].cands == (nid,)
                       for c in consumers.get(nid, [])):
                    self.shadow[nid] = new_buf(shape_size(shapes[nid]) * 2)
        for s in list(multi):
            # start pointing at a candidate's buffer (same shape for every candidate): a
            # cancelled pass that skipped every producer still hands its readers valid memory
            init = next((node_buf[c][0] for c in sorted(s) if c in node_buf), -1)
            multi[s] = new_cell(init)
        slot_buf: dict = {}
        slot_cell: dict = {}
        slot_rec: dict = {}
        for slot in sorted(self.sp.feed_slots):
            shp = self.feed_shapes.get(slot)
            if shp is None:
                raise ShapeMiss(f"no shape known for feed slot {slot}")
            slot_buf[slot] = new_buf(shape_size(shp) * self.esize)
            slot_cell[slot] = new_cell(slot_buf[slot])
            slot_rec[slot] = len(slot_rec)
            if slot in self.const_slots:              # speculative constant: prefilled, never fed
                consts.append(float(self.const_slots[slot]))
                fills.append((slot_buf[slot], 1, len(consts) - 1))
        pubs: dict = {}
        for nid in ops:
            pubs[nid] = [vcell[nid]] + [c for s, c in multi.items() if nid in s]
        for a_nid, p_nid in self.folded_assigns.items():
            v = self.var_index[ops[a_nid].attrs["var_name"]]
            pubs[p_nid] = pubs[p_nid] + [-(2000 + v)] + pubs[a_nid]
        for nid, lst in pubs.items():
            if len(lst) > MAX_PUB:
                raise ShapeMiss(f"node {nid} publishes to {len(lst)} cells (max {MAX_PUB})")

        def in_cell(b):
            if b.fed:
                return slot_cell[b.slot]
            if len(b.cands) == 1:
                c = b.cands[0]
                if c in self.elided_reads:
                    return -(1000 + self.var_index[ops[c].attrs["var_name"]])
                return vcell[c]
            return multi[frozenset(b.cands)]

        # variables assigned by the program (committed at pass end)
        assigned: dict = {}
        shape_ids: dict = {}
        for x in walk(self.sp.body):
            if isinstance(x, ExecOp) and x.kind is OpKind.ASSIGN_VAR:
                name = x.attrs["var_name"]
                s = shapes[x.node_id]
                assigned[name] = shape_size(s) * self.esize
                shape_ids.setdefault(s, len(shape_ids))
        self._sids = shape_ids
        late_count = [0]
        n_compute = [0]
        flops = [0]
        w: list = []

        def out_words(nid, late):
            b0, b1, pp = node_buf.get(nid, (-1, -1, False))
            p = pubs[nid]
            if late:
                late_count[0] += 1
            return [b0, b1, int(pp), int(late), len(p)] + p + [0] * (MAX_PUB - len(p))

        def ptr_item(op, nid, cin, var_idx, shape_id):
            return [T_PTR, op, nid, cin, var_idx, shape_id] + out_words(nid, False)

        self.consumers = consumers
        self._copies = {}
        self.n_chains = 0
        self.n_mchains = 0
        self._act_for = {}
        self._ce_loss = {}                       # fused cross-entropy: gradient node -> loss node
        self._skew_add = set()                   # adds fused with their rel_skew operand (kind 104)
        self._skip_f32 = {}                      # gradient node -> (plan word, attr index): 1 = no fp32 reader
        self._skip_cell = {}                     # its output cell -> gradient node
        self.n_attn = 0                          # flash-attention groups (forward + backward)
        self.n_head_fold = 0                     # ... of which read / write the merged head layout
        self.n_ar_buckets = 0                    # asynchronous bucketed all-reduces
        self._bias_for = {}                      # MatMul node -> bias_add fused into its epilogue
        self.n_bias_fused = 0
        self._ar_lists = []                      # instruction lists after bucketing (inspection)
        self._emitted = set()                    # node ids emitted as their own plan items
        self._fa_shadow = {}                     # attention output node -> its bf16 copy buffer
        self.chain_lates = 0
        self._chain_meta = {}

        def feed_item(x):
            if x.slot in self.const_slots:
                return None
            shp = tuple(self.feed_shapes[x.slot])
            return ([T_FEED, slot_code(x.slot), shape_size(shp), len(shp)] + _pad(shp)
                    + [slot_buf[x.slot], slot_cell[x.slot], slot_rec[x.slot],
                       _f64_bits(self.index_slots.get(x.slot, 0.0))])

        def emit(insts) -> list:
            items = []
            saved = self._copies
            self._copies = {}
            try:
                return emit_list(insts, items)
            finally:
                self._copies = saved

        def emit_list(insts, items) -> list:
            act_of = self._bn_act_pairs(insts) if (self.fuse and self.bf16) else {}
            if act_of:
                gone = {a.node_id for a in act_of.values()}
                insts = [y for y in insts if not (isinstance(y, ExecOp) and y.node_id in gone)]
            groups = self._attn_groups(insts, shapes) if (self.fuse and self.bf16) else []
            if groups:                              # flash attention: S, P, dP, dS never stored
                repl, gone = {}, set()
                for g in groups:
                    repl[g["O"].node_id] = _Attn(0, g)
                    repl[g["G"].node_id] = _Attn(1, g)
                    gone |= {g[k].node_id for k in ("S", "P", "dP", "DQ", "DK", "DV")}
                    gone |= g.get("fold_gone", set())
                    self.n_head_fold += 1 if "fold_gone" in g else 0
                    g["lse"] = self.new_buf(g["BH"] * g["T"] * 4)
                    g["delta"] = self.new_buf(g["BH"] * g["T"] * 4)
                    g["tiles"] = self.new_buf(4 * g["BH"] * g["T"] * FA_HEAD * 2)   # bf16 q | k | v | dO tiles
                    # folded outputs read only by GEMMs (through their [B*T, H*hd] reshape): the
                    # attention epilogue also writes the bf16 copy those GEMMs use
                    if "dst" in g and os.environ.get("COEX_FA_SHADOW", "1") != "0":
                        g["shadow"] = {}
                        for name, xnode in g["dst"].items():
                            r4 = [c.node_id for c in self.consumers.get(xnode.node_id, [])]
                            if len(r4) == 1 and self.ops[r4[0]].kind is OpKind.RESHAPE and \
                                    len(shapes[r4[0]]) == 2 and self._gemm_reader(r4[0]):
                                b_ = self.new_buf(shape_size(shapes[r4[0]]) * 2)
                                g["shadow"][name] = b_
                                self._fa_shadow[xnode.node_id] = b_
                    self.n_attn += 1
                insts = [repl.get(y.node_id, y) if isinstance(y, ExecOp) else y for y in insts
                         if not (isinstance(y, ExecOp) and y.node_id in gone)]
            bias_of = self._bias_pairs(insts) if (self.fuse and self.bf16) else {}
            if bias_of:                             # bias_add folded into its GEMM's epilogue
                gone_b = {y.node_id for y in bias_of.values()}
                insts = [y for y in insts if not (isinstance(y, ExecOp) and y.node_id in gone_b)]
                self._bias_for.update(bias_of)
                self.n_bias_fused += len(bias_of)
            skew_of = self._skew_pairs(insts) if (self.fuse and self.esize == 4) else {}
            if skew_of:                             # the skewed relative term is added on the fly
                gone_s = {sk.node_id for _, sk in skew_of.values()}
                insts = [skew_of[y.node_id][0] if isinstance(y, ExecOp) and y.node_id in skew_of else y
                         for y in insts if not (isinstance(y, ExecOp) and y.node_id in gone_s)]
            ce_of = self._ce_pairs(insts) if self.fuse else {}
            if ce_of:                               # the gradient moves up to the loss's position
                grads = {g.node_id for g in ce_of.values()}
                insts = [ce_of.get(y.node_id, y) if isinstance(y, ExecOp) else y for y in insts
                         if not (isinstance(y, ExecOp) and y.node_id in grads)]
            insts = self._bucket_allreduce(insts, node_buf, shapes)
            bn_groups, bn_skip = self._bn_bwd_groups(insts, shapes) if self.fuse else ({}, set())
            if self.fuse:
                segs = self._segments(insts, shapes, folded)
            else:
                segs = [("inst", x) for x in insts]
            for kind_, seg in segs:
                if kind_ == "inst" and isinstance(seg, ExecOp):
                    if seg.node_id in bn_skip:
                        continue
                    if seg.node_id in bn_groups:
                        items.append(self._bn_bwd_word(bn_groups[seg.node_id], shapes, in_cell, out_words, pubs,
                                                       n_compute))
                        continue
                if kind_ == "chain":
                    run, feeds = seg
                    for f in feeds:
                        it = feed_item(f)
                        if it is not None:
                            items.append(it)
                    try:
                        items.append(self._chain_item(run, shapes, in_cell, node_buf, pubs, multi, n_compute))
                    except _TooWide:
                        items.extend(emit(run))
                    self._invalidate([c for r in run for c in pubs[r.node_id]] +
                                     [slot_cell[f.slot] for f in feeds if f.slot in slot_cell])
                    continue
                x = seg
                if isinstance(x, InputFeed):
                    it = feed_item(x)
                    if it is not None:
                        items.append(it)
                    if x.slot in slot_cell:
                        self._invalidate([slot_cell[x.slot]])
                elif isinstance(x, OutputFetch):
                    shp = shapes[x.node_id]
                    items.append([T_FETCH, x.node_id, vcell[x.node_id], shape_size(shp), len(shp)] + _pad(shp))
                elif isinstance(x, _Attn):
                    items.append(self._attn_word(x, in_cell, out_words, pubs, n_compute, flops, shapes))
                elif isinstance(x, ExecOp):
                    items.extend(self._exec(x, shapes, in_cell, out_words, ptr_item, pubs, multi,
                                            folded, n_compute, flops))
                    self._invalidate(pubs[x.node_id])
                    self._register_shadow(x, pubs, shapes)
                    if x.kind is OpKind.ASSIGN_VAR:
                        self._invalidate([-(2000 + self.var_index[x.attrs["var_name"]])])
                elif isinstance(x, SwitchCase):
                    self._invalidate()
                    it = [T_SWITCH, x.branch_id, len(x.cases)]
                    for c in x.cases:
                        it += seq(c)
                    items.append(it)
                elif isinstance(x, While):
                    self._invalidate()
                    items.append([T_WHILE, x.loop_id] + seq(x.body))
                elif isinstance(x, UnrolledLoop):
                    self._invalidate()
                    for b in x.bodies:
                        items.extend(emit(b))
                elif type(x).__name__ == "AllReduce":
                    self._invalidate(pubs[x.node_id])      # only the reduced value changes
                    b0, b1, pp = node_buf.get(x.node_id, (-1, -1, True))
                    if b0 < 0 or pp:
                        raise NeedsReplicated(f"node {x.node_id} has no static buffer to all-reduce")
                    items.append([T_ALLREDUCE, b0, shape_size(shapes[x.node_id]), int(x.avg), 0])
                elif isinstance(x, _NvlsZero):
                    items.append([T_NVLS_ZERO, x.first, x.last])
                elif isinstance(x, _ARBucket):
                    # only the members' values change (shared bf16 operand copies of anything
                    # else stay valid across the collective)
                    self._invalidate([c for m in x.members for c in pubs[m.node_id]])
                    first = node_buf[x.members[0].node_id][0]
                    # span of the adjacent arena buffers (each padded to 256 bytes, csrc plan load)
                    span = 0
                    for i, m in enumerate(x.members):
                        nbytes = shape_size(shapes[m.node_id]) * self.esize
                        span += nbytes if i == len(x.members) - 1 else (max(nbytes, 16) + 255) // 256 * 256
                    tag = T_NVLS_AR if first in self.nvls_set else T_ALLREDUCE
                    items.append([tag, first, span // self.esize, int(x.members[0].avg), 1])
                    self.n_ar_buckets += 1
                elif isinstance(x, _Join):
                    items.append([T_JOIN])
            return self._group_chains(items) if self.fuse else items

        def seq(insts) -> list:
            items = emit(insts)
            self._invalidate()
            out = [T_SEQ, len(items)]
            for it in items:
                out += it
            return out

        body = seq(self.sp.body)
        w += [MAGIC, VERSION, len(bufs)] + bufs
        w += [len(self.nvls_bufs)] + self.nvls_bufs
        w += [len(cell_init)] + cell_init
        w += [len(slot_rec), late_count[0] + self.chain_lates]
        w += [len(fills)]
        for b0, n, ci in fills:
            w += [b0, n, ci]
        w += [len(assigned)]
        for name, nbytes in assigned.items():
            w += [self.var_index[name], nbytes]
        w += [len(shape_ids)]
        for s, sid in shape_ids.items():
            w += [sid, len(s)] + list(s)
        w += body
        sig = (tuple(sorted((k, tuple(v)) for k, v in self.var_shapes.items())),
               tuple(sorted((k, tuple(v)) for k, v in self.feed_shapes.items())))
        plan = Plan(w, consts, sig, n_compute[0], flops[0], shapes, dict(self.feed_shapes), folded, self.n_attn)
        plan.const_slots = dict(self.const_slots)
        plan.nvls_bufs = len(self.nvls_bufs)         # gradient buffers in the NVLS region
        plan.nvls_buckets = sum(1 for lst in self._ar_lists for x in lst if isinstance(x, _ARBucket)
                                and self._node_buf[x.members[0].node_id][0] in self.nvls_set)
        return plan

    def _exec(self, x, shapes, in_cell, out_words, ptr_item, pubs, multi, folded, n_compute, flops) -> list:
        nid = x.node_id
        self._emitted.add(nid)
        k = x.kind
        if k is OpKind.FILL:
            if any(nid in s for s in multi):
                return [ptr_item(PTR_ALIAS, nid, in_cell_const(nid, pubs), -1, -1)]
            return []
        if k is OpKind.RESHAPE:
            return [ptr_item(PTR_ALIAS, nid, in_cell(x.inputs[0]), -1, -1)]
        if k is OpKind.READ_VAR:
            if nid in self.elided_reads:
                return []
            return [ptr_item(PTR_READ_VAR, nid, -1, self.var_index[x.attrs["var_name"]], -1)]
        if k is OpKind.ASSIGN_VAR and nid in self.folded_assigns:
            return []
        if k is OpKind.ASSIGN_VAR:
            s = shapes[nid]
            return [ptr_item(PTR_ASSIGN_VAR, nid, in_cell(x.inputs[0]), self.var_index[x.attrs["var_name"]],
                             self._shape_id(s))]
        if nid in folded:
            return []
        if nid in self.index_nodes:
            return [ptr_item(PTR_ALIAS, nid, in_cell(x.inputs[0]), -1, -1)]
        if k in XOP:
            return [self._xop_word(x, shapes, in_cell, out_words, pubs, n_compute, flops)]
        ins = list(x.inputs)
        trans = [0, 0]
        cells = []
        in_shapes = []
        for i, b in enumerate(ins):
            if k is OpKind.MATMUL and not b.fed and len(b.cands) == 1 and b.cands[0] in folded:
                tnode = self.ops[b.cands[0]]
                cells.append(in_cell(tnode.inputs[0]))
                in_shapes.append(shapes[tnode.inputs[0].cands[0]])
                trans[i] = 1
            else:
                cells.append(in_cell(b))
                in_shapes.append(self._in_shape(b, shapes))
        while len(cells) < 2:
            cells.append(-1)
            in_shapes.append(())
        ba = self._bias_for.get(nid) if k is OpKind.MATMUL else None
        bias_cell = in_cell(ba.inputs[1]) if ba is not None else -1
        out_nid = ba.node_id if ba is not None else nid
        late = _conflicts(cells + ([bias_cell] if ba is not None else []), pubs[out_nid])
        attr_dims = list(x.attrs.get("perm", ()))
        out_shape = shapes[nid]
        n_compute[0] += 1
        if k is OpKind.MATMUL:
            m, kk = (in_shapes[0][1], in_shapes[0][0]) if trans[0] else in_shapes[0]
            nn = in_shapes[1][0] if trans[1] else in_shapes[1][1]
            flops[0] += 2 * m * nn * kk
        word = [T_OP, k.code, nid, cells[0], cells[1]]
        for s in in_shapes:
            word += [len(s)] + _pad(s)
        word += [len(out_shape)] + _pad(out_shape)
        word += [len(attr_dims)] + _pad(attr_dims) + [_f64_bits(0.0), trans[0], trans[1]]
        if k is OpKind.MATMUL and self.bf16:
            # narrow operands (the GEMM's M or N < 64 on an MN-major copy) are converted
            # transposed into a private K-major copy instead (flag 2): MN-major boxes of a
            # 1..63-wide tensor are mostly padding
            if trans[0] and m < 64:
                ca = (self.new_buf(max(m, 1) * ((kk + 7) // 8 * 8) * 2), 2)
            else:
                ca = self._copy(cells[0], in_shapes[0])
            if not trans[1] and nn < 64:
                cb = (self.new_buf(max(nn, 1) * ((kk + 7) // 8 * 8) * 2), 2)
            else:
                cb = self._copy(cells[1], in_shapes[1])
            self._need_f32(cells[0], ca[1])
            self._need_f32(cells[1], cb[1])
            word += [ca[0], cb[0], ca[1], cb[1]]
        elif k is OpKind.MATMUL and self.tf32:
            p4 = (max(kk, 1) + 3) // 4 * 4
            word += [self.new_buf(2 * max(m, 1) * p4 * 4), self.new_buf(2 * max(nn, 1) * p4 * 4), 1, 1]
        else:
            word += [-1, -1, 0, 0]
        sh = self.shadow.get(nid, -1) if k in (OpKind.GELU, OpKind.GELU_GRAD) else -1
        skip = int(sh != -1 and self._gemm_only(nid))
        word += [bias_cell, sh, skip]
        if skip:
            # a GEMM reader that ends up converting the fp32 tensor after all (its copy lookup
            # missed, e.g. after a collective invalidated the copies) re-enables the fp32 write
            self._skip_f32[nid] = (word, len(word) - 1)
            self._skip_cell[pubs[nid][0]] = nid
        word += out_words(out_nid, late)
        self._invalidate(pubs[out_nid])
        if ba is not None:
            self._invalidate(pubs[nid])
        return [word]

    def _bn_act_pairs(self, insts) -> dict:
        """batchnorm -> relu / leaky_relu of its output in the same instruction list: the
        normalisation kernel also writes the activation (one pass over the data instead of
        two, one launch less).  The activation must read the batchnorm output as its only
        candidate and be a plain stored node (not fetched, merged, pinned, folded or
        self-dependent); the fused op publishes both nodes at the batchnorm's position."""
        multi_nodes = {n for s_ in self._multi_sets() for n in s_}
        banned = set(self.sp.fetch_nodes) | multi_nodes | set(self.force_store) | set(self.folded_assigns.values())
        pos = {x.node_id: i for i, x in enumerate(insts) if isinstance(x, ExecOp)}
        out = {}
        taken = set()
        for x in insts:
            if not isinstance(x, ExecOp) or x.kind not in (OpKind.RELU, OpKind.LEAKY_RELU):
                continue
            b = x.inputs[0]
            if b.fed or len(b.cands) != 1 or x.node_id in banned:
                continue
            bn = self.ops.get(b.cands[0])
            if bn is None or bn.kind is not OpKind.BATCHNORM or bn.node_id in banned or bn.node_id in taken:
                continue
            if bn.node_id not in pos or pos[bn.node_id] > pos[x.node_id]:
                continue
            if any((not bb.fed) and x.node_id in bb.cands for bb in x.inputs):
                continue
            out[bn.node_id] = x
            taken.add(bn.node_id)
        self._act_for.update(out)
        return out

    def _attn_groups(self, insts, shapes) -> list:
        """One layer's causal attention, forward and backward, in one instruction list (the
        C4 program's hand-written attention; oracle/kernels.py BMM / CAUSAL_SOFTMAX /
        SOFTMAX_GRAD): S = bmm_nt(q, k) -> P = causal_softmax(S) -> O = bmm(P, v);
        dP = bmm_nt(dO, v) -> dS = softmax_grad(P, dP) -> dQ = bmm(dS, k), dK = bmm_tn(dS, q);
        dV = bmm_tn(P, dO).  S, P, dP and dS must have no other reader (not fetched, merged or
        pinned), the head dim is 64 and T a multiple of 128.  COEX_FLASH=0 disables it."""
        if os.environ.get("COEX_FLASH", "1") == "0":
            return []
        ex = {x.node_id: x for x in insts if isinstance(x, ExecOp)}
        pos = {x.node_id: i for i, x in enumerate(insts) if isinstance(x, ExecOp)}
        multi_nodes = {n for s_ in self._multi_sets() for n in s_}
        banned = set(self.sp.fetch_nodes) | multi_nodes | set(self.force_store) | set(self.folded_assigns.values())

        def single(b):
            return (not b.fed) and len(b.cands) == 1

        def only(nid):
            return [c.node_id for c in self.consumers.get(nid, [])]

        out = []
        for P in insts:
            if not isinstance(P, ExecOp) or P.kind is not OpKind.CAUSAL_SOFTMAX or not single(P.inputs[0]):
                continue
            S = ex.get(P.inputs[0].cands[0])
            if S is None or S.kind is not OpKind.BMM_NT or only(S.node_id) != [P.node_id]:
                continue
            q, k = S.inputs
            pc = self.consumers.get(P.node_id, [])
            O = [c for c in pc if c.kind is OpKind.BMM and single(c.inputs[0]) and c.inputs[0].cands == (P.node_id,)]
            G = [c for c in pc if c.kind is OpKind.SOFTMAX_GRAD and single(c.inputs[0])
                 and c.inputs[0].cands == (P.node_id,)]
            DV = [c for c in pc if c.kind is OpKind.BMM_TN and single(c.inputs[0]) and c.inputs[0].cands == (P.node_id,)]
            if len(pc) != 3 or len(O) != 1 or len(G) != 1 or len(DV) != 1:
                continue
            O, G, DV = O[0], G[0], DV[0]
            v = O.inputs[1]
            if not single(G.inputs[1]):
                continue
            dP = ex.get(G.inputs[1].cands[0])
            if dP is None or dP.kind is not OpKind.BMM_NT or dP.inputs[1] != v or only(dP.node_id) != [G.node_id]:
                continue
            do = dP.inputs[0]
            if DV.inputs[1] != do:
                continue
            gc = self.consumers.get(G.node_id, [])
            DQ = [c for c in gc if c.kind is OpKind.BMM and c.inputs[0].cands == (G.node_id,) and c.inputs[1] == k]
            DK = [c for c in gc if c.kind is OpKind.BMM_TN and c.inputs[0].cands == (G.node_id,) and c.inputs[1] == q]
            if len(gc) != 2 or len(DQ) != 1 or len(DK) != 1:
                continue
            DQ, DK = DQ[0], DK[0]
            nodes = {"S": S, "P": P, "O": O, "dP": dP, "G": G, "DQ": DQ, "DK": DK, "DV": DV}
            if any(n.node_id in banned or n.node_id not in ex for n in nodes.values()):
                continue
            if not all(single(b) for b in (q, k, v, do)):
                continue
            shp = tuple(self._in_shape(q, shapes))
            if len(shp) != 3 or shp[2] != FA_HEAD or shp[1] % FA_BLOCK or shp[1] == 0 or \
                    any(tuple(self._in_shape(b, shapes)) != shp for b in (k, v, do)):
                continue
            if float(P.attrs["value"]) != float(G.attrs["value"]):
                continue
            if any(self._node_buf.get(n.node_id, (-1, -1, True))[2] for n in (O, DQ, DK, DV)):
                continue                            # ping-pong outputs (self-dependent): not here
            if not (pos[S.node_id] < pos[P.node_id] < pos[O.node_id] and pos[dP.node_id] < pos[G.node_id]
                    and min(pos[DQ.node_id], pos[DK.node_id], pos[DV.node_id]) > pos[G.node_id]):
                continue
            g = dict(nodes, q=q, k=k, v=v, do=do, BH=shp[0], T=shp[1], scale=float(P.attrs["value"]))
            members = {n.node_id for n in nodes.values()}
            fold = self._head_fold(g, ex, members, banned, shapes)
            if fold is not None:
                g.update(fold)
            out.append(g)
        return out

    def _head_fold(self, g, ex, members, banned, shapes):
        """Head split / merge folded into the attention kernels (C4's ``heads_of`` / ``merge``):
        every operand q, k, v, dO is reshape(transpose(reshape(src, [B, T, H, hd]), [0, 2, 1, 3]),
        [B*H, T, hd]) of a merged [B*T, H*hd] tensor, and every output O, dQ, dK, dV is consumed
        only by reshape(transpose(reshape(., [B, H, T, hd]), [0, 2, 1, 3])).  The kernels then
        read the merged rows of src directly (row pitch H*hd, head offset h*hd) and write their
        outputs straight into the merge transposes' buffers: the eight [B*T, H*hd] transposes of
        the layer are never launched.  All or nothing (one operand layout per attention word).
        Returns {"H", "rs", "src": {name: binding}, "dst": {name: transpose node}, "fold_gone"}
        or None."""
        if os.environ.get("COEX_HEAD_FOLD", "1") == "0":
            return None
        BH, T = g["BH"], g["T"]
        cons = self.consumers

        def only(nid):
            return [c.node_id for c in cons.get(nid, [])]

        def node_of(b):
            if b.fed or len(b.cands) != 1:
                return None
            return ex.get(b.cands[0])

        def split(b):                                # operand binding -> (src binding, H, nodes)
            r2 = node_of(b)
            if r2 is None or r2.kind is not OpKind.RESHAPE or not set(only(r2.node_id)) <= members:
                return None
            x = node_of(r2.inputs[0])
            if x is None or x.kind is not OpKind.TRANSPOSE or tuple(x.attrs["perm"]) != (0, 2, 1, 3) or \
                    only(x.node_id) != [r2.node_id]:
                return None
            r1 = node_of(x.inputs[0])
            if r1 is None or r1.kind is not OpKind.RESHAPE or only(r1.node_id) != [x.node_id]:
                return None
            b_, t_, h_, d_ = shapes[r1.node_id]
            if t_ != T or d_ != FA_HEAD or b_ * h_ != BH:
                return None
            src = r1.inputs[0]
            if src.fed or len(src.cands) != 1 or shape_size(self._in_shape(src, shapes)) != BH * T * FA_HEAD:
                return None
            return src, h_, {r2.node_id, x.node_id, r1.node_id}

        def merge(o):                                # output node -> (merge transpose, H, nodes)
            r3 = only(o.node_id)
            if len(r3) != 1 or r3[0] not in ex or ex[r3[0]].kind is not OpKind.RESHAPE:
                return None
            r3 = ex[r3[0]]
            x = only(r3.node_id)
            if len(x) != 1 or x[0] not in ex:
                return None
            x = ex[x[0]]
            if x.kind is not OpKind.TRANSPOSE or tuple(x.attrs["perm"]) != (0, 2, 1, 3) or len(shapes[r3.node_id]) != 4:
                return None
            b_, h_, t_, d_ = shapes[r3.node_id]
            if t_ != T or d_ != FA_HEAD or b_ * h_ != BH:
                return None
            if self._node_buf.get(x.node_id, (-1, -1, True))[2] or x.node_id not in self._node_buf:
                return None
            return x, h_, {r3.node_id}

        src, dst, gone, hs = {}, {}, set(), set()
        for name in ("q", "k", "v", "do"):
            r = split(g[name])
            if r is None:
                return None
            src[name], h, nodes = r
            hs.add(h)
            gone |= nodes
        for name in ("O", "DQ", "DK", "DV"):
            r = merge(g[name])
            if r is None:
                return None
            dst[name], h, nodes = r
            hs.add(h)
            gone |= nodes | {dst[name].node_id}
        if len(hs) != 1 or gone & banned:
            return None
        H = hs.pop()
        return {"H": H, "rs": H * FA_HEAD, "src": src, "dst": dst, "fold_gone": gone}

    def _attn_word(self, a, in_cell, out_words, pubs, n_compute, flops, shapes) -> list:
        """[T_ATTN, mode, BH, T, H, row pitch, scale bits, lse buf, delta buf, tiles buf, cells q k v o dO,
        outputs]"""
        g = a.g
        src = g.get("src", {})
        dst = {k: v.node_id for k, v in g.get("dst", {}).items()}
        opnd = {k: in_cell(src.get(k, g[k])) for k in ("q", "k", "v", "do")}
        out_node = {k: dst.get(k, g[k].node_id) for k in ("O", "DQ", "DK", "DV")}
        o_cell = pubs[out_node["O"]][0]
        if a.mode == 0:
            cells = [opnd["q"], opnd["k"], opnd["v"], -1, -1]
            outs = [out_node["O"]]
            members = ("S", "O")
        else:
            cells = [opnd["q"], opnd["k"], opnd["v"], o_cell, opnd["do"]]
            outs = [out_node["DQ"], out_node["DK"], out_node["DV"]]
            members = ("dP", "DQ", "DK", "DV")
        for m in members:
            x = g[m]
            flops[0] += flops_of(x.kind, [tuple(self._in_shape(b, shapes)) for b in x.inputs], x.attrs)
        n_compute[0] += 1
        sh = g.get("shadow", {})
        shw = [sh.get("O", -1), -1, -1] if a.mode == 0 else [sh.get("DQ", -1), sh.get("DK", -1), sh.get("DV", -1)]
        word = [T_ATTN, a.mode, g["BH"], g["T"], g.get("H", 1), g.get("rs", FA_HEAD), _f64_bits(g["scale"]), g["lse"],
                g["delta"], g["tiles"]] + shw + cells
        for nid in outs:
            word += out_words(nid, _conflicts(cells, pubs[nid]))
            self._invalidate(pubs[nid])
        return word

    def _bias_pairs(self, insts) -> dict:
        """bias_add(matmul(a, b), c) in one instruction list (C4 / C5 projections): the GEMM
        epilogue adds the bias (split-K: the slice reduction does) and writes the bias_add's
        output directly -- no separate pass over the [rows, N] product.  Legal when the
        MatMul's only reader is the bias_add, neither node is fetched / merged / pinned /
        self-dependent, and the bias binding is produced before the MatMul (or fed).
        Returns {matmul node: bias_add node}."""
        if os.environ.get("COEX_BIAS_FUSE", "1") == "0":
            return {}
        multi_nodes = {n for s_ in self._multi_sets() for n in s_}
        banned = set(self.sp.fetch_nodes) | multi_nodes | set(self.force_store) | set(self.folded_assigns.values())
        pos = {x.node_id: i for i, x in enumerate(insts) if isinstance(x, ExecOp)}
        out = {}
        for x in insts:
            if not isinstance(x, ExecOp) or x.kind is not OpKind.BIAS_ADD or x.node_id in banned:
                continue
            a, c = x.inputs
            if a.fed or len(a.cands) != 1 or a.cands[0] not in pos:
                continue
            m = self.ops[a.cands[0]]
            if m.kind is not OpKind.MATMUL or m.node_id in banned or m.node_id in out:
                continue
            if [y.node_id for y in self.consumers.get(m.node_id, [])] != [x.node_id]:
                continue
            if self._node_buf.get(x.node_id, (-1, -1, True))[2] or x.node_id not in self._node_buf:
                continue
            if any((not b.fed) and x.node_id in b.cands for b in x.inputs):
                continue
            if not c.fed and any(cc in pos and pos[cc] > pos[m.node_id] and cc not in self.elided_reads
                                 for cc in c.cands):
                continue                            # (an elided variable read has no position)
            if not c.fed and any(cc == m.node_id for cc in c.cands):
                continue
            out[m.node_id] = x
        return out

    def _skew_pairs(self, insts) -> dict:
        """add(a, rel_skew(x)) (C5's attention logits, q.k^T + skew(q.er^T)) where the skew's
        only reader is that add, in one instruction list: ONE row pass computes the sum
        (csrc k_rel_skew_v4<0, true>, plan kind 104), the skewed [BH, T, T] tensor is never
        stored.  The skew must be a plain stored node (not fetched, merged, pinned or
        assigned) and nothing between the two re-produces x.  Returns {add node: (fused
        ExecOp, skew node)}; the fused op sits at the add's position."""
        multi_nodes = {n for s_ in self._multi_sets() for n in s_}
        banned = set(self.sp.fetch_nodes) | multi_nodes | set(self.force_store) | set(self.folded_assigns.values())
        pos = {x.node_id: i for i, x in enumerate(insts) if isinstance(x, ExecOp)}
        out = {}
        for x in insts:
            if not isinstance(x, ExecOp) or x.kind is not OpKind.ADD or x.node_id in banned:
                continue
            for j in (1, 0):
                b, a = x.inputs[j], x.inputs[1 - j]
                if b.fed or len(b.cands) != 1 or b.cands[0] not in pos:
                    continue
                sk = self.ops[b.cands[0]]
                if sk.kind is not OpKind.REL_SKEW or sk.node_id in banned or pos[sk.node_id] > pos[x.node_id]:
                    continue
                if [c.node_id for c in self.consumers.get(sk.node_id, [])] != [x.node_id]:
                    continue
                xb = sk.inputs[0]
                srcs = set(xb.cands) if not xb.fed else set()
                if any(isinstance(y, ExecOp) and y.node_id in srcs for y in insts[pos[sk.node_id] + 1:pos[x.node_id]]):
                    continue
                fused = ExecOp(x.node_id, OpKind.REL_SKEW, {}, [xb, a])
                self._skew_add.add(x.node_id)
                out[x.node_id] = (fused, sk)
                break
        return out

    def _ce_pairs(self, insts) -> dict:
        """cross_entropy(lg, ids) and cross_entropy_grad(lg, ids) over the same bindings in one
        instruction list: one kernel computes both (the logits are read once).  The fused op
        takes the loss's position; legal when nothing in between re-produces an input and
        neither node is merged, pinned or self-dependent.  Returns {loss node: grad node}."""
        multi_nodes = {n for s_ in self._multi_sets() for n in s_}
        banned = multi_nodes | set(self.folded_assigns.values())
        pos = {x.node_id: i for i, x in enumerate(insts) if isinstance(x, ExecOp)}
        out = {}
        for x in insts:
            if not isinstance(x, ExecOp) or x.kind is not OpKind.CROSS_ENTROPY or x.node_id in banned:
                continue
            g = next((y for y in insts if isinstance(y, ExecOp) and y.kind is OpKind.CROSS_ENTROPY_GRAD
                      and y.inputs == x.inputs and y.node_id not in banned and y.node_id not in self.force_store
                      and pos[y.node_id] > pos[x.node_id]), None)
            if g is None or g in out.values():
                continue
            ids = {x.node_id, g.node_id}
            if any((not b.fed) and (set(b.cands) & ids) for b in x.inputs):
                continue
            lo, hi = pos[x.node_id], pos[g.node_id]
            srcs = {c for b in x.inputs if not b.fed for c in b.cands}
            fed = {b.slot for b in x.inputs if b.fed}
            # (data parallel: the loss's all-reduce sits between them -- it reads the loss only)
            if any((isinstance(y, ExecOp) and y.node_id in srcs) or (isinstance(y, InputFeed) and y.slot in fed)
                   or not (isinstance(y, (ExecOp, InputFeed, OutputFetch))
                           or (type(y).__name__ == "AllReduce" and y.node_id not in srcs))
                   for y in insts[lo + 1:hi]):
                continue
            out[x.node_id] = g
            self._ce_loss[g.node_id] = x
        return out

    def _bn_bwd_groups(self, insts, shapes=None):
        """Batch-norm backward triples in one instruction list -- batchnorm_dx(x, g, dy),
        bn_dgamma(x, dy), sum_rows(dy) with identical x / dy bindings -- run as ONE column-
        statistics pass (all three need sum(dy) and sum(dy * xhat)).  The fused op sits at the
        position of the last member; legal when nothing in between consumes an earlier member's
        output or re-produces an input, and no member is fetched / merged / pinned."""
        groups, skip = {}, set()
        pos = {}
        for i, x in enumerate(insts):
            if isinstance(x, ExecOp):
                pos.setdefault(x.node_id, i)
        multi_nodes = {n for s_ in self._multi_sets() for n in s_}
        # batch norm (any precision) and -- fp32 storage, 4 | d <= 1024 -- layernorm
        ln_ok = self.esize == 4 and os.environ.get("COEX_LN_BWD_FUSE", "1") != "0"
        dxs = [x for x in insts if isinstance(x, ExecOp) and
               (x.kind is OpKind.BATCHNORM_DX or (ln_ok and x.kind is OpKind.LAYERNORM_DX))]
        used = set()
        for d in dxs:
            xb, gb, dyb = d.inputs
            if xb.fed or dyb.fed or "rows" in d.attrs:     # synchronised (data parallel): unfused
                continue
            gkind = OpKind.BN_DGAMMA if d.kind is OpKind.BATCHNORM_DX else OpKind.LN_DGAMMA
            if d.kind is OpKind.LAYERNORM_DX:
                dd = self._in_shape(xb, shapes)[-1] if shapes is not None else 0
                if dd % 4 or dd > 1024 or dd == 0:
                    continue
            g = next((y for y in insts if isinstance(y, ExecOp) and y.kind is gkind
                      and y.node_id not in used and y.inputs[0] == xb and y.inputs[1] == dyb), None)
            sr = next((y for y in insts if isinstance(y, ExecOp) and y.kind is OpKind.SUM_ROWS
                       and y.node_id not in used and y.inputs[0] == dyb), None)
            if g is None or sr is None:
                continue
            mem = [d, g, sr]
            ids = {m.node_id for m in mem}
            # all-reduced (pinned) members are fine: the fused op writes every member's own
            # buffer, and a bucket holding a member between the positions forces the first-
            # member placement below (everything is produced before the collective)
            if any(n in self.sp.fetch_nodes or n in multi_nodes for n in ids):
                continue
            lo = min(pos[m.node_id] for m in mem)
            hi = max(pos[m.node_id] for m in mem)
            ok = True
            for i in range(lo, hi + 1):
                y = insts[i]
                if isinstance(y, ExecOp) and y.node_id in ids:
                    continue
                if not isinstance(y, (ExecOp, InputFeed)):
                    ok = False
                    break
                if any((not b.fed) and (set(b.cands) & ids) for b in y.inputs):
                    ok = False                      # consumes a member's output before the fused op
                    break
                # re-producing an input of a member that already ran (e.g. its gamma ReadVar
                # is fine for the last member, which the fused op replaces in place)
                if any(pos[m.node_id] < i and any((not b.fed) and y.node_id in b.cands for b in m.inputs)
                       for m in mem):
                    ok = False
                    break
            at = insts[hi]
            if not ok:
                # alternatively at the FIRST member's position (the layernorm's dx feeds a
                # residual add before ln_dgamma / sum_rows run): every member reads only
                # (x, g, dy), so that is legal when nothing up to the last member re-produces
                # x, dy or the first member's own inputs, and there is no control flow between
                first = insts[lo]
                srcs = {c for m in mem for b in m.inputs if not b.fed for c in b.cands}
                ok = all((isinstance(y, (ExecOp, InputFeed)) or
                          (isinstance(y, _ARBucket) and not any(m.node_id in srcs for m in y.members))
                          or isinstance(y, _Join)) and
                         not (isinstance(y, ExecOp) and y.node_id not in ids and y.node_id in srcs)
                         for y in insts[lo:hi + 1])
                # the members' own inputs must all exist at the first position
                ok = ok and all(not b.fed and all(pos.get(c, -1) < lo or c not in pos for c in b.cands)
                                or b.fed for m in mem for b in m.inputs)
                if not ok:
                    continue
                at = first
            groups[at.node_id] = (d, g, sr)
            skip |= ids - {at.node_id}
            used |= ids
        return groups, skip

    def _bn_bwd_word(self, grp, shapes, in_cell, out_words, pubs, n_compute) -> list:
        d, g, sr = grp
        cells = [in_cell(b) for b in d.inputs]
        in_shapes = [self._in_shape(b, shapes) for b in d.inputs]
        late = _conflicts(cells, pubs[d.node_id] + pubs[g.node_id] + pubs[sr.node_id])
        n_compute[0] += 1
        out_shape = shapes[d.node_id]
        word = [T_XOP, XOP_LN_BWD if d.kind is OpKind.LAYERNORM_DX else XOP_BN_BWD, d.node_id, 3] + cells
        for s_ in in_shapes:
            word += [len(s_)] + _pad(s_)
        word += [len(out_shape)] + _pad(out_shape)
        word += [0] + _pad([]) + [_f64_bits(0.0)]
        word += out_words(d.node_id, late) + out_words(g.node_id, late) + out_words(sr.node_id, late)
        self._invalidate(pubs[d.node_id] + pubs[g.node_id] + pubs[sr.node_id])
        return word + [-1] * (1 + MAX_XIN) + [0] * MAX_XIN

    def _xop_word(self, x, shapes, in_cell, out_words, pubs, n_compute, flops) -> list:
        nid = x.node_id
        cells = [in_cell(b) for b in x.inputs]
        in_shapes = [self._in_shape(b, shapes) for b in x.inputs]
        late = _conflicts(cells, pubs[nid])
        n_compute[0] += 1
        attr = list(x.attrs["conv"]) if x.kind in CONV_ATTR_KINDS else list(x.attrs.get("dims", ()))
        if x.kind in BMM_KINDS and self.bf16:
            tri = self._tri_flag(x)
            attr = [tri] if tri else []
        if x.kind in CONV_KINDS or x.kind in BMM_KINDS:
            flops[0] += flops_of(x.kind, in_shapes, x.attrs)
        out_shape = shapes[nid]
        act = self._act_for.get(nid)
        ce_loss = self._ce_loss.get(nid)
        kind_code = x.kind.code
        if act is not None:                     # batchnorm + activation in one apply pass
            kind_code = XOP_BN_ACT
            attr = [EW_CODE[act.kind]]
        skip = 0
        if nid in self._skew_add:               # add(a, rel_skew(x))
            kind_code = XOP_SKEW_ADD
        if ce_loss is not None:                 # loss + gradient in one pass over the logits
            kind_code = XOP_CE_FUSED
            skip = int(nid in self.shadow and self._gemm_only(nid))
            attr = [skip]
        word = [T_XOP, kind_code, nid, len(cells)] + cells + [-1] * (MAX_XIN - len(cells))
        for s_ in in_shapes + [()] * (MAX_XIN - len(in_shapes)):
            word += [len(s_)] + _pad(s_)
        word += [len(out_shape)] + _pad(out_shape)
        attr_at = len(word) + 1
        word += [len(attr)] + _pad(attr) + [_f64_bits(float(x.attrs.get("value", x.attrs.get("rows", 0.0))))]
        word += out_words(nid, late)
        if act is not None:
            word += out_words(act.node_id, _conflicts(cells, pubs[act.node_id]))
            self._invalidate(pubs[act.node_id])
        if ce_loss is not None:
            word += out_words(ce_loss.node_id, _conflicts(cells, pubs[ce_loss.node_id]))
            self._invalidate(pubs[ce_loss.node_id])
            if skip:                            # cleared if any GEMM has to convert the fp32 tensor
                self._skip_f32[nid] = (word, attr_at)
                self._skip_cell[pubs[nid][0]] = nid
        word += self._shadow_words(x, cells, in_shapes)
        self._invalidate(pubs[nid])
        return word

    def _register_shadow(self, x, pubs, shapes):
        """After x's publication: its bf16 shadow (written by its kernel) is the valid bf16
        copy of its output for later GEMMs of the same list.  A 2-D reshape of an attention
        output with a bf16 copy (written by the attention epilogue) registers that copy."""
        nid = x.node_id
        if x.kind is OpKind.RESHAPE and not x.inputs[0].fed and len(x.inputs[0].cands) == 1 and \
                x.inputs[0].cands[0] in self._fa_shadow and len(shapes[nid]) == 2:
            shp = shapes[nid]
            self._copies[(pubs[nid][0], shp[0], shp[1])] = self._fa_shadow[x.inputs[0].cands[0]]
            return
        if x.kind is OpKind.RESHAPE and not x.inputs[0].fed and len(x.inputs[0].cands) == 1 and \
                len(shapes[nid]) == 2 and self.ops[x.inputs[0].cands[0]].kind is OpKind.REL_UNSKEW and \
                x.inputs[0].cands[0] in self.shadow and x.inputs[0].cands[0] in self._emitted:
            # the unskew kernel's bf16 copy ([rows][T], T % 8 == 0: no padding) under the
            # reshape's cell -- the relative-table GEMMs read it instead of converting
            shp = shapes[nid]
            self._copies[(pubs[nid][0], shp[0], shp[1])] = self.shadow[x.inputs[0].cands[0]]
            return
        if nid in self.shadow and (x.kind is not OpKind.CROSS_ENTROPY_GRAD or nid in self._ce_loss):
            shp = shapes[nid]
            self._copies[(pubs[nid][0], shape_size(shp[:-1]), shp[-1])] = self.shadow[nid]

    def _gemm_reader(self, nid) -> bool:
        """Some reader of nid's output is a MatMul operand (directly or through a folded
        transpose) -- a bf16 copy written by the producer saves that GEMM a conversion."""
        for c in self.consumers.get(nid, []):
            if c.kind is OpKind.MATMUL:
                return True
            if c.kind is OpKind.TRANSPOSE and c.node_id in self.folded:
                return True
        return False

    def _gemm_only(self, nid) -> bool:
        """Every reader of nid's output is a MatMul operand (directly or through a folded
        transpose) and the value is not fetched, merged, pinned or assigned."""
        if nid in self.sp.fetch_nodes or nid in self.force_store or nid in self.folded_assigns.values():
            return False
        if any(nid in s_ for s_ in self._multi_sets()):
            return False
        for c in self.consumers.get(nid, []):
            if c.kind is OpKind.MATMUL:
                continue
            if c.kind is OpKind.TRANSPOSE and c.node_id in self.folded and \
                    all(cc.kind is OpKind.MATMUL for cc in self.consumers.get(c.node_id, [])):
                continue
            return False
        return True

    def _need_f32(self, cell, conv):
        """A GEMM operand read from ``cell`` needs the fp32 tensor (its copy is converted):
        the producer must write it after all."""
        nid = self._skip_cell.get(cell)
        if nid is not None and conv:
            word, at = self._skip_f32[nid]
            word[at] = 0

    def _causal_prob(self, b) -> bool:
        """Binding b is (single-candidate) a causal_softmax output, or a softmax_grad of one --
        both are exactly zero above the diagonal of every [T, T] block."""
        if b.fed or len(b.cands) != 1:
            return False
        n = self.ops.get(b.cands[0])
        if n is None:
            return False
        if n.kind is OpKind.CAUSAL_SOFTMAX:
            return True
        return n.kind is OpKind.SOFTMAX_GRAD and self._causal_prob(n.inputs[0])

    def _tri_flag(self, x) -> int:
        """Causal structure of a batched GEMM (tcgen05 path): 1 = only the lower triangle of
        the output is ever read (QK^T into causal_softmax, dO.V^T into softmax_grad of a causal
        softmax), 2 / 3 = operand A lower- / upper-triangular (P or dS, as stored / transposed)."""
        if x.kind is OpKind.BMM_NT:
            nid = x.node_id
            cons = self.consumers.get(nid, [])
            if not cons or nid in self.sp.fetch_nodes or any(nid in s_ for s_ in self._multi_sets()):
                return 0
            for c in cons:
                if c.kind is OpKind.CAUSAL_SOFTMAX:
                    continue
                if c.kind is OpKind.SOFTMAX_GRAD and c.inputs[1].cands == (nid,) and \
                        c.inputs[0].cands != (nid,) and self._causal_prob(c.inputs[0]):
                    continue
                return 0
            return 1
        if x.kind in (OpKind.BMM, OpKind.BMM_TN) and self._causal_prob(x.inputs[0]):
            return 2 if x.kind is OpKind.BMM else 3
        return 0

    # ------------------------------------------------------------ shared bf16 operand copies
    # Every tcgen05 GEMM operand is a bf16 copy [rows][pitch(cols)] of the stored tensor, a
    # layout that serves K-major and MN-major use alike.  Within one straight-line instruction
    # list the first GEMM that needs a tensor converts it into a shared buffer and later GEMMs
    # reuse it, until something republishes the tensor's cell (or control flow intervenes).
    def _copy(self, cell, shape) -> tuple:
        """(buffer index, convert?) of the bf16 copy of the tensor behind operand cell ``cell``."""
        shape = tuple(shape)
        rows = shape_size(shape[:-1]) if len(shape) > 1 else 1
        cols = shape[-1] if shape else 1
        key = (cell, rows, cols)
        hit = self._copies.get(key)
        if hit is not None:
            return hit, 0
        buf = self.new_buf(max(rows, 1) * ((max(cols, 1) + 7) // 8 * 8) * 2)
        if cell is not None and cell != -1:
            self._copies[key] = buf
        return buf, 1

    def _invalidate(self, pub_codes=None):
        """Drop copies whose source cell is republished (all copies when ``pub_codes`` is None)."""
        if pub_codes is None:
            self._copies.clear()
            return
        dead = set()
        for c in pub_codes:
            dead.add(c)
            if c <= -2000:                      # a variable's overlay slot: its direct reads change
                dead.add(-(1000 + (-2000 - c)))
        for key in [k for k in self._copies if k[0] in dead]:
            del self._copies[key]

    def _shadow_words(self, x, in_cells=None, in_shapes=None) -> list:
        """[own bf16 shadow buffer] + per input [bf16 copy buffer] + per input [convert?] for the
        batched GEMMs (others: no copies)."""
        bufs, conv = [-1] * MAX_XIN, [0] * MAX_XIN
        if x.kind in BMM_KINDS and self.bf16 and in_cells is not None:
            for i in range(2):
                bufs[i], conv[i] = self._copy(in_cells[i], in_shapes[i])
                self._need_f32(in_cells[i], conv[i])
        return [self.shadow.get(x.node_id, -1)] + bufs + conv

    # ------------------------------------------------------------ pointer-op rewrites
    def _pointer_rewrites(self, consumers, multi, folded):
        """ReadVar nodes whose consumers all follow them in the same instruction list with no
        assignment to the variable in between read the variable directly (no pointer kernel);
        an AssignVar that directly follows its producer is folded into the producer's publish
        list (the producer writes the variable's overlay slot)."""
        ops = self.ops
        multi_nodes = {n for s_ in multi for n in s_}
        elided, fold = set(), {}
        lists = list(_lists(self.sp.body))
        for nid, x in ops.items():
            if x.kind is OpKind.READ_VAR and nid not in self.sp.fetch_nodes and nid not in multi_nodes \
                    and nid not in self.force_store:
                var = x.attrs["var_name"]
                cons = consumers.get(nid, [])
                if not cons or any(len(b.cands) != 1 for c in cons for b in c.inputs if not b.fed and nid in b.cands):
                    continue
                cids = {c.node_id for c in cons}
                if all(_reads_local(L, nid, cids, var) for L in lists):
                    elided.add(nid)
        for nid, x in ops.items():
            if x.kind is not OpKind.ASSIGN_VAR or x.inputs[0].fed or len(x.inputs[0].cands) != 1:
                continue
            p = x.inputs[0].cands[0]
            px = ops.get(p)
            if px is None or px.kind not in COMPUTE or p in folded or p in self.force_store:
                continue
            var = x.attrs["var_name"]
            if all(_assign_local(L, p, nid, var) for L in lists):
                fold[nid] = p
        return elided, fold

    # ------------------------------------------------------------ fusion
    def _segments(self, insts, shapes, folded) -> list:
        """Split one instruction list into fused runs and plain instructions.  A run is a
        maximal sequence of same-size elementwise ExecOps (InputFeeds in between are
        hoisted in order), optionally closed by SUM / MEAN of a value computed in the run;
        an OutputFetch or any other instruction ends it."""
        segs: list = []
        run: list = []
        feeds: list = []
        n_run = [None]

        def flush():
            if len(run) >= 2:
                segs.append(("chain", (list(run), list(feeds))))
            else:
                segs.extend(("inst", f) for f in feeds)
                segs.extend(("inst", r) for r in run)
            run.clear()
            feeds.clear()
            n_run[0] = None

        def in_run(nid):
            return any(r.node_id == nid for r in run)

        for x in insts:
            if isinstance(x, InputFeed) and run:
                feeds.append(x)
                continue
            if isinstance(x, ExecOp) and x.kind in EW_CODE and x.node_id not in folded and \
                    x.node_id not in self.index_nodes:
                n = shape_size(shapes[x.node_id])
                if run and n != n_run[0] or len(run) >= CHAIN_OPS:
                    flush()
                if not run:
                    n_run[0] = n
                run.append(x)
                continue
            if (isinstance(x, ExecOp) and x.kind in (OpKind.SUM, OpKind.MEAN) and run
                    and not x.inputs[0].fed and len(x.inputs[0].cands) == 1 and in_run(x.inputs[0].cands[0])
                    and len(run) < CHAIN_OPS):
                run.append(x)
                flush()
                continue
            flush()
            segs.append(("inst", x))
        flush()
        return segs

    def _arm_views(self, consumers, multi, folded, shapes, new_buf, new_view) -> dict:
        """Arm-exclusive node buffers: the cases of a SwitchCase never run in the same pass, so
        a node produced inside one case and read only inside that case (an arm-local
        activation) can live in memory the other cases' arm-local nodes use too.  Per
        SwitchCase one region of max-over-cases bytes; each case lays its local nodes out from
        the region's start (256-byte slots).  Never aliased: fetched, merged (multi-candidate),
        pinned (force_store), variable-published, self-dependent or folded nodes, constants,
        nodes that occur in several cases.  C3 (four SDPoint arms) and C2 (D / G steps).
        COEX_ARM_ALIAS=0 keeps one buffer per node.  Returns {node: view buffer index}."""
        if os.environ.get("COEX_ARM_ALIAS", "1") == "0":
            return {}
        ops = self.ops
        multi_nodes = {n for s_ in multi for n in s_}
        banned = set(self.sp.fetch_nodes) | multi_nodes | set(self.force_store) | \
            set(self.folded_assigns.values()) | set(self.index_nodes)
        out = {}
        self.arm_alias_bytes = [0, 0]          # (bytes without aliasing, region bytes)

        def local_nodes(case, others_count):
            inside = {y.node_id for y in walk(case) if isinstance(y, ExecOp)}
            loc = []
            for nid in sorted(inside):
                x = ops.get(nid)
                if x is None or others_count[nid] > 1 or nid in banned or nid in out:
                    continue
                if x.kind not in COMPUTE or nid in folded:
                    continue
                if any((not b.fed) and nid in b.cands for b in x.inputs):
                    continue
                if not all(c.node_id in inside for c in consumers.get(nid, [])):
                    continue
                loc.append(nid)
            return loc

        def visit(insts):
            for x in insts:
                if isinstance(x, SwitchCase):
                    from collections import Counter
                    cnt = Counter(y.node_id for c in x.cases for y in walk(c) if isinstance(y, ExecOp))
                    layouts, size = [], 0
                    for c in x.cases:
                        off, lay = 0, []
                        for nid in local_nodes(c, cnt):
                            nbytes = max(shape_size(shapes[nid]) * self.esize, 16)
                            lay.append((nid, off))
                            off += (nbytes + 255) // 256 * 256
                            self.arm_alias_bytes[0] += nbytes
                        layouts.append(lay)
                        size = max(size, off)
                    if size > 0 and sum(len(l) for l in layouts) > 0:
                        region = new_buf(size)
                        self.arm_alias_bytes[1] += size
                        for lay in layouts:
                            for nid, off in lay:
                                out[nid] = new_view(region, off)
                    for c in x.cases:                # nested switches: their own regions
                        visit(c)
                elif isinstance(x, While):
                    visit(x.body)
                elif isinstance(x, UnrolledLoop):
                    for b in x.bodies:
                        visit(b)

        visit(self.sp.body)
        return out

    def _bucket_allreduce(self, insts, node_buf, shapes) -> list:
        """Data-parallel gradient all-reduces (dp.py AllReduce items) of one instruction list,
        bucketed and overlapped: consecutive all-reduces whose buffers are adjacent in the
        arena (build() allocates all-reduced nodes in program order) and share sum / average
        form one collective (up to AR_BUCKET_BYTES), issued as a side branch of the graph
        (T_ALLREDUCE async); the compute that follows does not wait.  A _Join goes in front of
        the first instruction that reads a value whose collective is pending or issued
        (typically the parameter updates at the end of the backward pass), in front of any
        control flow, and at the end of the list.  COEX_AR_BUCKET_MB=0 keeps one synchronous
        collective per gradient."""
        if AR_BUCKET_BYTES <= 0 or not any(type(x).__name__ == "AllReduce" for x in insts):
            return insts
        out, pending, issued = [], [], set()
        nbytes = [0]

        def flush():
            if pending:
                out.append(_ARBucket(list(pending)))
                issued.update(m.node_id for m in pending)
                pending.clear()
                nbytes[0] = 0

        def join():
            flush()
            if issued:
                out.append(_Join())
                issued.clear()

        for x in insts:
            if type(x).__name__ == "AllReduce":
                b0 = node_buf.get(x.node_id, (-1, -1, True))
                if b0[0] < 0 or b0[2]:
                    raise NeedsReplicated(f"node {x.node_id} has no static buffer to all-reduce")
                if pending:
                    last = node_buf[pending[-1].node_id][0]
                    if b0[0] != last + 1 or x.avg != pending[-1].avg:
                        flush()
                pending.append(x)
                nbytes[0] += shape_size(shapes[x.node_id]) * self.esize
                if nbytes[0] >= AR_BUCKET_BYTES:
                    flush()
                continue
            waiting = issued | {m.node_id for m in pending}
            if isinstance(x, ExecOp):
                if waiting and any((not b.fed) and any(c in waiting for c in b.cands) for b in x.inputs):
                    join()
            elif isinstance(x, OutputFetch):
                if x.node_id in waiting:
                    join()
            elif not isinstance(x, InputFeed):
                join()                                   # control flow: everything settles first
            out.append(x)
        join()
        # NVLS: the list's bucket buffers are zeroed (every rank) before anything adds into them
        nv = [node_buf[m.node_id][0] for x in out if isinstance(x, _ARBucket) for m in x.members
              if node_buf[m.node_id][0] in self.nvls_set]
        if nv:
            out.insert(0, _NvlsZero(min(nv), max(nv)))
        self._ar_lists.append(out)
        return out

    def _group_chains(self, items: list) -> list:
        """Adjacent elementwise chains that neither read what another one publishes (cells,
        variable overlay slots) nor reduce run as one k_chain_multi launch (T_MCHAIN) -- e.g.
        every parameter update of a step; each keeps its own late-publication counter."""
        out, group = [], []

        def flush():
            if len(group) == 1:
                out.append(group[0])
            elif group:
                w = [T_MCHAIN, len(group)]
                for g in group:
                    w += g
                out.append(w)
                self.n_mchains += 1
            group.clear()

        for it in items:
            meta = self._chain_meta.get(id(it))
            if meta is None or meta[0] is not it or meta[3]:     # (ids of dropped words get reused)
                flush()
                out.append(it)
                continue
            ok = len(group) < MAX_MCHAIN
            for g in group:
                gm = self._chain_meta[id(g)]
                if _conflicts(meta[1], gm[2]) or _conflicts(gm[1], meta[2]):
                    ok = False
                    break
            if not ok:
                flush()
            group.append(it)
        flush()
        return out

    def _chain_item(self, run, shapes, in_cell, node_buf, pubs, multi, n_compute) -> list:
        red = run[-1] if run[-1].kind in (OpKind.SUM, OpKind.MEAN) else None
        ew = run[:-1] if red is not None else run
        n = shape_size(shapes[ew[0].node_id])
        inputs: list = []          # (cell, scalar)
        ops: list = []
        reg_of: dict = {}          # position in run -> register

        def src(pos, b):
            if not b.fed:
                for q in range(pos - 1, -1, -1):
                    if run[q].node_id in b.cands:
                        return reg_of[q]
            cell = in_cell(b)
            scal = 1 if (n > 1 and shape_size(self._in_shape_any(b, shapes)) == 1) else 0
            key = (cell, scal)
            if key not in inputs:
                inputs.append(key)
            return CHAIN_REGS + inputs.index(key)

        for pos, x in enumerate(ew):
            a = src(pos, x.inputs[0])
            b = src(pos, x.inputs[1]) if len(x.inputs) > 1 else 0
            reg_of[pos] = pos
            ops.append((EW_CODE[x.kind], pos, a, b))
        red_reg = src(len(ew), red.inputs[0]) if red is not None else 0
        if len(inputs) > CHAIN_IN:
            raise _TooWide()
        outs: list = []
        for pos, x in enumerate(ew):
            if self._must_store(x.node_id, run, pos):
                p = pubs[x.node_id]
                if len(p) > CHAIN_PUB or len(outs) >= CHAIN_OUT:
                    raise _TooWide()
                outs.append((pos, node_buf[x.node_id][0], p))
        pub_cells = {c for _, _, p in outs for c in p}
        if red is not None:
            pub_cells |= set(pubs[red.node_id])
        late = int(_conflicts([c for c, _ in inputs], pub_cells))
        self.chain_lates += late
        n_compute[0] += 1
        self.n_chains += 1
        w = [T_CHAIN, n]
        if red is not None:
            rp = pubs[red.node_id]
            if len(rp) > CHAIN_PUB:
                raise _TooWide()
            w += [1 if red.kind is OpKind.SUM else 2, red_reg, node_buf[red.node_id][0], len(rp)] + rp + \
                [0] * (CHAIN_PUB - len(rp))
        else:
            w += [0, 0, -1, 0] + [0] * CHAIN_PUB
        w += [late, len(inputs)]
        for cell, scal in inputs + [(-1, 0)] * (CHAIN_IN - len(inputs)):
            w += [cell, scal]
        w += [len(ops)]
        for op in ops + [(0, 0, 0, 0)] * (CHAIN_OPS - len(ops)):
            w += list(op)
        w += [len(outs)]
        for reg, buf, p in outs + [(0, -1, [])] * (CHAIN_OUT - len(outs)):
            w += [reg, buf, len(p)] + list(p) + [0] * (CHAIN_PUB - len(p))
        self._chain_meta[id(w)] = (w, [c for c, _ in inputs], sorted(pub_cells), red is not None)
        return w

    def _must_store(self, nid, run, pos) -> bool:
        """A value computed in a run stays in registers only if every consumer anywhere in the
        program is a later op of this run that reads it as its latest candidate."""
        if nid in self.sp.fetch_nodes or nid in self.force_store or any(nid in s for s in self._multi_sets()):
            return True
        later = {id(x): q for q, x in enumerate(run) if q > pos}
        for c in self.consumers.get(nid, []):
            q = later.get(id(c))
            if q is None:
                return True
            for b in c.inputs:
                if not b.fed and nid in b.cands:
                    last = max((r for r in range(q) if run[r].node_id in b.cands), default=None)
                    if last != pos:
                        return True
        return False

    def _multi_sets(self):
        ms = getattr(self, "_ms", None)
        if ms is None:
            ms = self._ms = [frozenset(b.cands) for x in walk(self.sp.body) if isinstance(x, ExecOp)
                             for b in x.inputs if not b.fed and len(b.cands) > 1]
        return ms

    def _in_shape_any(self, b, shapes):
        if b.fed:
            return tuple(self.feed_shapes[b.slot])
        return shapes[b.cands[0]]

    def _in_shape(self, b, shapes):
        if b.fed:
            return tuple(self.feed_shapes[b.slot])
        return shapes[b.cands[0]]

    def _shape_id(self, s):
        return self._sids[tuple(s)]


def in_cell_const(nid, pubs):
    return pubs[nid][0]


def _mentions(x, nid) -> bool:
    return any(isinstance(y, ExecOp) and y.node_id == nid for y in walk([x]))


def _fold_is_local(insts, tnid: int, producer: int) -> bool:
    """A transpose may be read in place by its MatMul consumer only if, in every
    instruction list holding the transpose, a consuming MatMul follows in the
    same list and nothing in between can re-execute the transpose's producer."""
    ok = True
    found = False

    def scan(lst):
        nonlocal ok, found
        for i, x in enumerate(lst):
            if isinstance(x, ExecOp) and x.node_id == tnid:
                found = True
                j = i + 1
                hit = False
                while j < len(lst):
                    y = lst[j]
                    if isinstance(y, ExecOp) and y.kind is OpKind.MATMUL and \
                            any((not b.fed) and tnid in b.cands for b in y.inputs):
                        hit = True
                        break
                    if _mentions(y, producer) or not isinstance(y, (ExecOp, InputFeed, OutputFetch)):
                        break
                    j += 1
                ok = ok and hit
            elif isinstance(x, SwitchCase):
                for c in x.cases:
                    scan(c)
            elif isinstance(x, While):
                scan(x.body)
            elif isinstance(x, UnrolledLoop):
                for b in x.bodies:
                    scan(b)

    scan(insts)
    return ok and found


class _TooWide(Exception):
    """A fused run needs more inputs / outputs / publish cells than the chain kernel holds."""


class NeedsReplicated(Exception):
    """A sharded plan cannot be lowered (e.g. all-reduce of a pointer-only value)."""


def _conflicts(in_codes, pub_codes) -> bool:
    """A kernel must publish late if it reads a cell it publishes, or reads a variable whose
    overlay slot it publishes (a folded AssignVar of a variable the op itself reads)."""
    pubs = set(pub_codes)
    for c in in_codes:
        if c is None or c == -1:
            continue
        if c >= 0 and c in pubs:
            return True
        if -2000 < c <= -1000 and -(2000 + (-1000 - c)) in pubs:
            return True
    return False


def _lists(insts):
    yield insts
    for x in insts:
        if isinstance(x, SwitchCase):
            for c in x.cases:
                yield from _lists(c)
        elif isinstance(x, While):
            yield from _lists(x.body)
        elif isinstance(x, UnrolledLoop):
            for b in x.bodies:
                yield from _lists(b)


def _touches_var(x, var) -> bool:
    return any(isinstance(y, ExecOp) and y.kind in (OpKind.READ_VAR, OpKind.ASSIGN_VAR)
               and y.attrs.get("var_name") == var for y in walk([x]))


def _assigns_var(x, var) -> bool:
    return any(isinstance(y, ExecOp) and y.kind is OpKind.ASSIGN_VAR and y.attrs.get("var_name") == var
               for y in walk([x]))


def _reads_local(L, rid, cids, var) -> bool:
    """Every consumer instance in list L has an instance of ReadVar ``rid`` earlier in L with
    no assignment to ``var`` in between; consumers nested below L are checked in their lists."""
    last = None
    for j, x in enumerate(L):
        if isinstance(x, ExecOp) and x.node_id == rid:
            last = j
        elif _assigns_var(x, var):
            last = None
        if isinstance(x, ExecOp) and x.node_id in cids:
            if last is None:
                return False
    return True


def _assign_local(L, pid, aid, var) -> bool:
    """In list L every instance of producer ``pid`` is followed by AssignVar ``aid`` and every
    instance of ``aid`` is preceded by ``pid`` with only plain ops (none touching ``var``) between."""
    pending = None
    for j, x in enumerate(L):
        if isinstance(x, ExecOp) and x.node_id == pid:
            if pending is not None:
                return False
            pending = j
            continue
        if isinstance(x, ExecOp) and x.node_id == aid:
            if pending is None:
                return False
            pending = None
            continue
        if pending is not None:
            if not isinstance(x, (ExecOp, InputFeed, OutputFetch)) or _touches_var(x, var):
                return False
        elif any(isinstance(y, ExecOp) and y.node_id in (pid, aid) for y in walk([x])) and \
                not isinstance(x, ExecOp):
            pass                      # nested instances are checked in their own list
    return pending is None
