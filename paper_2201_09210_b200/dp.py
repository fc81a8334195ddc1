"""Data-parallel co-execution: shard a SymProgram over R ranks.

Every rank runs the same host program (skeleton, natives, decisions) on global
shapes; only the device pass is sharded.  Feed slots whose leading dimension is
the global batch are fed row shards; a propagation pass over the SymProgram
tags every value

    R   replicated            (variables, fills, host scalars, all-reduced values)
    S0  rows sharded          (batch inputs and row-wise functions of them)
    S1  columns sharded       (transpose of S0)
    P+  partial sum           (Sum over S0, MatMul contracting the sharded dim)
    P~  partial mean          (Mean over S0 -- equal shards make the mean of
                               local means the global mean)

and inserts ``AllReduce(node, op)`` right after a Partial producer when any
consumer needs a replicated value: AssignVar, OutputFetch, a nonlinear op, or
mixing with R / another Partial kind.  After the all-reduce the node is R for
all consumers, so fetched values -- and hence every rank's decisions -- are
identical.  Anything outside these rules (e.g. fetching a sharded activation,
assigning a sharded value to a variable, slicing a replicated batch tensor)
makes the program run replicated: every rank computes the global batch, no
collective, still correct.

Extension ops (C2): convolutions of a row-sharded NHWC activation with a
replicated weight stay row-sharded (S0); a weight gradient ``conv2d_dw`` of two
row-sharded operands, ``sum_rows`` and ``bn_dgamma`` over row-sharded values are
P+; ``batchnorm`` / ``batchnorm_dx`` / ``bn_dgamma`` of a row-sharded activation
are *synchronised*: the rewrite stamps them with the global row count (attr
``rows``) and the device computes rank-local raw column sums, all-reduces them
(NCCL, inside the op's launch sequence) and normalises with the statistics of
the GLOBAL batch -- the single-device math (SPEC.md:466 sequential-order
equality, up to summation order).  ``batchnorm`` / ``batchnorm_dx`` stay S0;
``bn_dgamma`` is R (already the global sum).

C4 ops: layernorm (rows), bias_add, causal softmax and its gradient, the batched
GEMMs (batch = sequences x heads, sharded with the sequences) and the embedding
gather keep S0; ``embedding_dw`` and ``ln_dgamma`` are P+; ``cross_entropy`` is
P~ (equal row shards); ``cross_entropy_grad`` keeps S0 and is rewritten to divide
by the global row count.  A reshape keeps S0 when its leading target dimension
splits evenly over the ranks (row-major chunks stay contiguous); a transpose keeps
S0 when it leaves axis 0 in place.

Parity: DP results equal the single-device run up to summation order
(tolerance, not bitwise) -- tests/test_dp_gloo.py checks world size 2 on CPU
(distinct row shards, batch norm included).
"""

from __future__ import annotations

import copy
from dataclasses import dataclass, field

from .graph_gen import ExecOp, InputFeed, OutputFetch, SwitchCase, SymProgram, UnrolledLoop, While
from .rng import jump_state
from .tensor import OpKind, Tensor, shape_size

R, S0, S1, PSUM, PAVG = "R", "S0", "S1", "P+", "P~"
PARTIAL = (PSUM, PAVG)
ELEMENTWISE = (OpKind.ADD, OpKind.SUB, OpKind.MUL, OpKind.DIV)
LINEAR_UNARY = (OpKind.NEG,)
NONLINEAR = (OpKind.RELU, OpKind.SIGMOID, OpKind.TANH, OpKind.LEAKY_RELU, OpKind.GELU, OpKind.SQRT)
# extension ops (C2 / C4): row-wise binary nonlinear ops keep the row sharding of their operands
ROW_BINARY = (OpKind.RELU_GRAD, OpKind.LEAKY_RELU_GRAD, OpKind.BCE_TERM, OpKind.GELU_GRAD, OpKind.TO_INDEX)
# C4 ops whose rows (or batch entries) are independent: sharded in, sharded out
ROW_WISE = (OpKind.LAYERNORM, OpKind.LAYERNORM_DX, OpKind.BIAS_ADD, OpKind.CAUSAL_SOFTMAX, OpKind.SOFTMAX_GRAD,
            OpKind.BMM, OpKind.BMM_NT, OpKind.BMM_TN, OpKind.EMBEDDING, OpKind.CROSS_ENTROPY_GRAD,
            OpKind.REL_SKEW, OpKind.REL_UNSKEW,
            # C3: per-image pooling and conv2d's input gradient (weight replicated)
            OpKind.CONV2D_DX, OpKind.MAXPOOL, OpKind.MAXPOOL_GRAD, OpKind.AVGPOOL, OpKind.AVGPOOL_GRAD,
            OpKind.GLOBAL_AVGPOOL, OpKind.GLOBAL_AVGPOOL_GRAD)


@dataclass
class AllReduce:
    """Sum (``avg=False``) or average the node's latest output across ranks, in place."""

    node_id: int
    avg: bool


class Unshardable(Exception):
    pass


@dataclass
class DPPlan:
    sp: SymProgram                  # transformed program (AllReduce inserted, local reshape attrs)
    sharded_slots: set              # feed slots fed row shards
    state: dict                     # node id -> state
    world: int
    replicated: bool = False        # True: program runs unsharded on every rank
    reason: str = ""
    allreduce_nodes: list = field(default_factory=list)


def _iter(insts):
    for x in insts:
        yield x
        if isinstance(x, SwitchCase):
            for c in x.cases:
                yield from _iter(c)
        elif isinstance(x, While):
            yield from _iter(x.body)
        elif isinstance(x, UnrolledLoop):
            for b in x.bodies:
                yield from _iter(b)


class _Prop:
    def __init__(self, sp: SymProgram, feed_shapes: dict, node_shapes: dict, batch: int, world: int):
        self.sp = sp
        self.feed_shapes = feed_shapes
        self.node_shapes = node_shapes
        self.batch = batch
        self.world = world
        self.sharded = {s for s, shp in feed_shapes.items()
                        if len(shp) >= 1 and shp[0] == batch and batch % world == 0}
        self.state: dict = {}
        self.reduce_at: dict = {}       # node id -> avg flag
        self.sync_bn: set = set()       # batch-norm family nodes over row shards (synchronised)
        self.kind: dict = {}
        self.consumers: dict = {}       # node id -> ids of the ops reading it
        for x in _iter(sp.body):
            if isinstance(x, ExecOp):
                self.kind[x.node_id] = x
                for b in x.inputs:
                    if not b.fed:
                        for c in b.cands:
                            self.consumers.setdefault(c, set()).add(x.node_id)

    def bind(self, b):
        if b.fed:
            return S0 if b.slot in self.sharded else R
        sts = {self.eff(c) for c in b.cands if c in self.state}
        if not sts:
            return None
        if len(sts) > 1:
            raise Unshardable(f"candidates {b.cands} disagree on sharding {sorted(sts)}")
        return sts.pop()

    def eff(self, nid):
        """State a consumer sees: all-reduced Partials read as R."""
        st = self.state[nid]
        return R if (st in PARTIAL and nid in self.reduce_at) else st

    def _sole_partial(self, b, st, nid):
        """binding b is one partial producer of kind st read only by node nid"""
        return (not b.fed and len(b.cands) == 1 and self.state.get(b.cands[0]) == st
                and self.consumers.get(b.cands[0], set()) == {nid})

    def need_r(self, nid):
        """A consumer needs node ``nid`` replicated: schedule its all-reduce.  The collective is
        hoisted to the earliest partial producer it can move to -- through a reshape (a view),
        a scaling by a replicated value (the learning-rate product of an update), a negation or
        a sum of partials each read only here -- so the gradient is reduced where the backward
        pass produces it and the planner can overlap it with the rest of the backward
        (planner._bucket_allreduce).  Sums are linear, so the result is the same up to
        summation order."""
        st = self.state.get(nid)
        x = self.kind.get(nid)
        if st in PARTIAL and x is not None and x.kind is OpKind.RESHAPE and not x.inputs[0].fed \
                and len(x.inputs[0].cands) == 1 and self.state.get(x.inputs[0].cands[0]) == st:
            # a reshape is a view with no buffer of its own: reduce its producer in place
            return self.need_r(x.inputs[0].cands[0])
        if st in PARTIAL and x is not None and nid not in self.reduce_at:
            ins = x.inputs
            if x.kind is OpKind.MUL and len(ins) == 2:
                for i in (0, 1):
                    other = ins[1 - i]
                    if self._sole_partial(ins[i], st, nid) and self.bind(other) == R:
                        return self.need_r(ins[i].cands[0])
            if x.kind in LINEAR_UNARY and self._sole_partial(ins[0], st, nid):
                return self.need_r(ins[0].cands[0])
            if x.kind is OpKind.ADD and len(ins) == 2 and all(self._sole_partial(b, st, nid) for b in ins) \
                    and ins[0].cands != ins[1].cands:
                self.need_r(ins[0].cands[0])
                return self.need_r(ins[1].cands[0])
        if st in PARTIAL:
            self.reduce_at[nid] = st == PAVG
            return True
        if st in (S0, S1):
            raise Unshardable(f"node {nid}: a sharded value is needed replicated")
        return False

    def needs_r_binding(self, b):
        if not b.fed:
            for c in b.cands:
                if c in self.state:
                    self.need_r(c)

    def op(self, x: ExecOp):
        k = x.kind
        ins = [self.bind(b) for b in x.inputs]
        if any(s is None for s in ins):
            return None                      # loop-carried input not known yet
        if k in (OpKind.READ_VAR, OpKind.FILL):
            return R
        if k is OpKind.ASSIGN_VAR:
            if ins[0] in PARTIAL:
                self.needs_r_binding(x.inputs[0])
                return R
            if ins[0] != R:
                raise Unshardable("assigning a sharded value to a variable")
            return R
        if k in NONLINEAR:
            if ins[0] in PARTIAL:
                self.needs_r_binding(x.inputs[0])
                return R
            return ins[0]
        if k in LINEAR_UNARY:
            return ins[0]
        if k in (OpKind.CONV2D, OpKind.CONV2D_T, OpKind.CONV2D_DW, OpKind.BATCHNORM, OpKind.BATCHNORM_DX,
                 OpKind.BN_DGAMMA, OpKind.SUM_ROWS, OpKind.EMBEDDING_DW, OpKind.LN_DGAMMA,
                 OpKind.CROSS_ENTROPY) or k in ROW_BINARY or k in ROW_WISE:
            return self._ext(x, ins)
        if k in (OpKind.SLICE, OpKind.CONCAT, OpKind.SUM_AXIS):
            # linear data movement / reduction along one axis: states pass through unless the
            # axis is the sharded one
            ax = x.attrs["dims"][0]
            if any(st == S1 for st in ins) or (ax == 0 and any(st == S0 for st in ins)):
                raise Unshardable(f"node {x.node_id}: {k.value} along the sharded axis")
            if len(set(ins)) > 1:
                raise Unshardable(f"node {x.node_id}: {k.value} of {ins}")
            return ins[0]
        if k is OpKind.DIV and ins[1] in PARTIAL:
            self.needs_r_binding(x.inputs[1])        # a / P is not linear in P
            ins = [ins[0], R]
        if k in ELEMENTWISE:
            a, b = ins
            scalar = [self._rank0(bb) for bb in x.inputs]
            if a == b:
                if a in PARTIAL and k is OpKind.MUL:
                    self.needs_r_binding(x.inputs[0])
                    self.needs_r_binding(x.inputs[1])
                    return R
                return a
            pa, pb = a in PARTIAL, b in PARTIAL
            if pa and pb:                       # P+ with P~
                self.needs_r_binding(x.inputs[0])
                self.needs_r_binding(x.inputs[1])
                return R
            if pa or pb:
                other = b if pa else a
                if k in (OpKind.MUL, OpKind.DIV) and other == R:
                    return a if pa else b       # scaling by a replicated value is linear
                self.needs_r_binding(x.inputs[0 if pa else 1])
                a, b = (R, b) if pa else (a, R)
                if a == b:
                    return R
            # now no partials: combine R with S0/S1
            if a != R and b != R:
                raise Unshardable(f"node {x.node_id}: {a} meets {b}")
            sh = a if a != R else b
            r_side = 1 if a != R else 0
            if not scalar[r_side]:
                raise Unshardable(f"node {x.node_id}: replicated tensor meets a sharded one")
            return sh
        if k in (OpKind.SUM, OpKind.MEAN):
            a = ins[0]
            if a in (S0, S1):
                return PSUM if k is OpKind.SUM else PAVG
            if a in PARTIAL:
                if k is OpKind.MEAN and a == PSUM or k is OpKind.SUM and a == PAVG:
                    return a                    # linear: keeps the partial kind
                return a
            return R
        if k is OpKind.TRANSPOSE:
            a = ins[0]
            perm = tuple(x.attrs["perm"])
            if a == S0 and len(perm) > 2 and perm[0] == 0:
                return S0                            # rows stay on their rank
            if a in (S0, S1):
                if perm != (1, 0):
                    raise Unshardable("transpose of a sharded tensor beyond 2-D")
                return S1 if a == S0 else S0
            return a
        if k is OpKind.RESHAPE:
            a = ins[0]
            if a == S1:
                raise Unshardable("reshape of a column-sharded tensor")
            if a == S0:
                tgt = x.attrs["target_shape"]
                if not tgt or tgt[0] % self.world:
                    raise Unshardable("reshape whose leading dimension does not split over the ranks")
            return a
        if k is OpKind.MATMUL:
            a, b = ins
            if a == S0 and b == R:
                return S0
            if a == S1 and b == S0:
                return PSUM
            if a == R and b == R:
                return R
            if a in PARTIAL and b == R:
                return a
            if a == R and b in PARTIAL:
                return b
            if a in PARTIAL or b in PARTIAL:
                for i, s in enumerate(ins):
                    if s in PARTIAL:
                        self.needs_r_binding(x.inputs[i])
                return self.op(x)
            raise Unshardable(f"matmul of {a} x {b}")
        raise Unshardable(f"no sharding rule for {k.value}")

    def _ext(self, x: ExecOp, ins):
        """Sharding rules of the C2 extension ops (module docstring)."""
        k = x.kind
        for i, st in enumerate(ins):               # every extension op needs complete operands
            if st in PARTIAL:
                self.needs_r_binding(x.inputs[i])
        ins = [R if st in PARTIAL else st for st in ins]
        if k in ROW_BINARY:
            a, b = ins
            if a == b:
                return a
            if S1 in (a, b):
                raise Unshardable(f"node {x.node_id}: column-sharded operand of {k.value}")
            r_side = 1 if a != R else 0
            if not self._rank0(x.inputs[r_side]):
                raise Unshardable(f"node {x.node_id}: replicated tensor meets a sharded one")
            return a if a != R else b
        if k in ROW_WISE:
            # sharded operands: the rows / batch entries; replicated ones: parameters (gamma,
            # beta, bias, embedding table); EMBEDDING's table is operand 0
            sh = [st for st in ins if st != R]
            if not sh:
                return R
            if any(st != S0 for st in sh):
                raise Unshardable(f"node {x.node_id}: {k.value} of {ins}")
            if k in (OpKind.BMM, OpKind.BMM_NT, OpKind.BMM_TN, OpKind.SOFTMAX_GRAD, OpKind.CROSS_ENTROPY_GRAD,
                     OpKind.LAYERNORM_DX, OpKind.CONV2D_DX, OpKind.MAXPOOL_GRAD, OpKind.AVGPOOL_GRAD,
                     OpKind.GLOBAL_AVGPOOL_GRAD) and len(sh) != 2:
                raise Unshardable(f"node {x.node_id}: {k.value} mixes sharded and replicated rows")
            if k is OpKind.EMBEDDING and ins[0] != R:
                raise Unshardable(f"node {x.node_id}: sharded embedding table")
            if k in (OpKind.LAYERNORM, OpKind.BIAS_ADD) and ins[0] != S0:
                raise Unshardable(f"node {x.node_id}: {k.value} of replicated rows with sharded parameters")
            return S0
        if k in (OpKind.EMBEDDING_DW, OpKind.LN_DGAMMA):
            if ins == [S0, S0]:
                return PSUM
            if ins == [R, R]:
                return R
            raise Unshardable(f"node {x.node_id}: {k.value} of {ins}")
        if k is OpKind.CROSS_ENTROPY:
            if ins == [S0, S0]:
                return PAVG
            if ins == [R, R]:
                return R
            raise Unshardable(f"node {x.node_id}: cross_entropy of {ins}")
        if k in (OpKind.CONV2D, OpKind.CONV2D_T):
            xs, w = ins
            if w != R:
                raise Unshardable(f"node {x.node_id}: sharded convolution weight")
            if xs == S1:
                raise Unshardable(f"node {x.node_id}: column-sharded convolution input")
            return xs
        if k is OpKind.CONV2D_DW:
            xs, dy = ins
            if xs == S0 and dy == S0:
                return PSUM
            if xs == R and dy == R:
                return R
            raise Unshardable(f"node {x.node_id}: weight gradient of {xs} x {dy}")
        if k in (OpKind.BATCHNORM, OpKind.BATCHNORM_DX):
            xs = ins[0]
            if ins[1] != R or (k is OpKind.BATCHNORM and ins[2] != R):
                raise Unshardable(f"node {x.node_id}: sharded batch-norm parameters")
            if k is OpKind.BATCHNORM_DX and ins[2] != xs:
                raise Unshardable(f"node {x.node_id}: batch-norm gradient sharded unlike its input")
            if xs == S1:
                raise Unshardable(f"node {x.node_id}: column-sharded batch-norm input")
            if xs == S0:
                self.sync_bn.add(x.node_id)     # synchronised batch statistics
            elif xs in PARTIAL:
                self.needs_r_binding(x.inputs[0])
                return R
            return xs
        # BN_DGAMMA / SUM_ROWS: column sums over the rows
        if any(st == S1 for st in ins):
            raise Unshardable(f"node {x.node_id}: column-sharded operand of {k.value}")
        if all(st == R for st in ins):
            return R
        if any(st == R for st in ins):
            raise Unshardable(f"node {x.node_id}: {k.value} of replicated and sharded operands")
        if k is OpKind.BN_DGAMMA:
            self.sync_bn.add(x.node_id)         # synchronised: the global sum(dy * xhat)
            return R
        return PSUM

    def shape_of(self, b):
        """Global shape of binding b."""
        return self.feed_shapes.get(b.slot) if b.fed else self.node_shapes.get(b.cands[0])

    def _rank0(self, b):
        shp = self.shape_of(b)
        return shp is not None and shape_size(shp) == 1

    def walk(self, insts):
        changed = False
        for x in insts:
            if isinstance(x, ExecOp):
                st = self.op(x)
                if st is not None and self.state.get(x.node_id) != st:
                    self.state[x.node_id] = st
                    changed = True
            elif isinstance(x, OutputFetch):
                if x.node_id in self.state:
                    before = x.node_id in self.reduce_at
                    self.need_r(x.node_id)
                    changed |= (x.node_id in self.reduce_at) != before
            elif isinstance(x, SwitchCase):
                for c in x.cases:
                    changed |= self.walk(c)
            elif isinstance(x, While):
                changed |= self.walk(x.body)
            elif isinstance(x, UnrolledLoop):
                for b in x.bodies:
                    changed |= self.walk(b)
        return changed

    def run(self):
        for _ in range(8):
            before = dict(self.reduce_at)
            self.sync_bn = set()            # recomputed by every walk: the last one is exact
            changed = self.walk(self.sp.body)
            # a node marked for all-reduce on an earlier walk may have become replicated since
            # (its own partial input got reduced in place for another consumer): its mark is
            # stale -- all-reducing a replicated value would multiply it by the world size
            self.reduce_at = {n: v for n, v in self.reduce_at.items() if self.state.get(n) in PARTIAL}
            if not changed and self.reduce_at == before:
                return
        raise Unshardable("sharding states did not converge")


def _rewrite(insts, prop: _Prop) -> list:
    out = []
    for x in insts:
        if isinstance(x, ExecOp):
            y = x
            if x.kind is OpKind.RESHAPE and prop.state.get(x.node_id) == S0:
                tgt = list(x.attrs["target_shape"])
                tgt[0] //= prop.world
                y = ExecOp(x.node_id, x.kind, dict(x.attrs, target_shape=tuple(tgt)), x.inputs)
            if x.kind is OpKind.CROSS_ENTROPY_GRAD and prop.state.get(x.node_id) == S0:
                rows = prop.node_shapes[x.node_id][0]        # divide by the global row count
                y = ExecOp(x.node_id, x.kind, dict(x.attrs, rows=float(rows)), x.inputs)
            if x.node_id in prop.sync_bn:
                shp = prop.shape_of(x.inputs[0])             # normalise over the global rows
                rows = shape_size(shp) // shp[-1]
                y = ExecOp(x.node_id, x.kind, dict(x.attrs, rows=float(rows)), x.inputs)
            out.append(y)
            if x.node_id in prop.reduce_at:
                out.append(AllReduce(x.node_id, prop.reduce_at[x.node_id]))
        elif isinstance(x, SwitchCase):
            out.append(SwitchCase(x.branch_id, [_rewrite(c, prop) for c in x.cases]))
        elif isinstance(x, While):
            out.append(While(x.loop_id, x.node_id, _rewrite(x.body, prop)))
        elif isinstance(x, UnrolledLoop):
            body = _rewrite(x.bodies[0], prop) if x.bodies else []
            out.append(UnrolledLoop(x.loop_id, x.node_id, [body] * len(x.bodies)))
        else:
            out.append(x)
    return out


def shard_program(sp: SymProgram, feed_shapes: dict, node_shapes: dict, batch: int, world: int,
                  force: bool = False) -> DPPlan:
    """Shard ``sp`` for ``world`` ranks with global batch ``batch`` (feeds with dim0 == batch).
    ``node_shapes`` are the global shapes of the specialisation (Planner.infer_shapes)."""
    if world <= 1 and not force:
        return DPPlan(sp, set(), {}, world, replicated=True, reason="world size 1")
    prop = _Prop(sp, feed_shapes, node_shapes, batch, world)
    if not prop.sharded:
        return DPPlan(sp, set(), {}, world, replicated=True, reason="no batch-sized feed")
    try:
        prop.run()
    except Unshardable as e:
        return DPPlan(sp, set(), {}, world, replicated=True, reason=str(e))
    new = copy.copy(sp)
    new.body = _rewrite(sp.body, prop)
    return DPPlan(new, prop.sharded, prop.state, world, False, "", sorted(prop.reduce_at))


def local_feed_shapes(feed_shapes: dict, plan: DPPlan) -> dict:
    out = dict(feed_shapes)
    for s in plan.sharded_slots:
        shp = list(out[s])
        shp[0] //= plan.world
        out[s] = tuple(shp)
    return out


def shard_value(v, rank: int, world: int):
    """Rank ``rank``'s row shard of a fed batch value (host tensor or synthetic descriptor)."""
    from .dataset import SyntheticTensor
    rows = v.shape[0] // world
    if isinstance(v, SyntheticTensor):
        row_elems = shape_size(v.shape[1:])
        st = jump_state(v.state, rank * rows * row_elems)
        return SyntheticTensor(st, (rows,) + tuple(v.shape[1:]))
    data = v.data if hasattr(v, "data") else v
    return Tensor((rows,) + tuple(v.shape[1:]), data[rank * rows:(rank + 1) * rows])


@dataclass
class DPGroup:
    """This process's place in the data-parallel job."""

    rank: int
    world: int
    batch: int                      # global batch: feeds with this leading dim are sharded
    allreduce: object = None        # callable(numpy array, avg) -> numpy array (CPU oracle only)
    force: bool = False             # shard (and all-reduce over NCCL) even at world size 1 (tests)
