"""Interpreter: imperative, traced, skeleton and replay execution of a program.

Specification: SPEC.md:168-264 (the reference ships no implementation).

One tree-walking evaluator serves every mode; what an op call *does* is
delegated to a step context:

* :class:`EagerCtx` -- imperative and traced modes:
  every op runs immediately on the backend (on the B200: ``coex_exec_op``);
  with ``trace`` set it also records TraceEvents.
* :class:`SkeletonCtx` -- co-execution: ops create empty
  handles (shape from ``infer_shape``), the cursor checks the step against the
  TraceGraph, decisions and feeds go to the running pass, materialisation
  blocks on the pass's fetch channel, prints are buffered.

Language semantics fixed here (SPEC leaves them open; DESIGN.md lists them):
host env state does not survive a step: each step starts from
the post-prologue environment; ``step`` is the step index; one-argument
``transpose`` reverses the axes; ``fill`` values are coerced to float; a host
value mixed into an op is lifted to a fed tensor; ``item`` returns a float for
rank-0 tensors and a nested list otherwise.
"""

from __future__ import annotations

import time

from . import lang
from .errors import CoexError, EvalError, ShapeMiss
from .lang import ast
from .natives import eval_native
from .tensor import OpKind, Tensor, canonical_attrs, infer_shape, lift_host_value, shape_size
from .dataset import SyntheticTensor
from .trace_graph import (Diverged, External, Handle, LoopEnter, LoopExit,
                          LoopIterStart, OpEvent, StepEnd)

OP_BY_NAME = {k.value: k for k in OpKind if k not in (OpKind.READ_VAR, OpKind.ASSIGN_VAR)}
CONV_NAMES = frozenset(("conv2d", "conv2d_t", "conv2d_dw", "embedding_dw", "conv2d_dx", "maxpool", "maxpool_grad",
                        "avgpool", "avgpool_grad", "slice", "concat", "sum_axis"))
DIMS_NAMES = frozenset(("embedding_dw", "slice", "concat", "sum_axis"))     # literal -> "dims" attr
SCALE_NAMES = frozenset(("causal_softmax", "softmax_grad"))    # trailing host scale -> "value" attr


class Val:
    """A tensor produced by an op call: ``dev`` is the backend value (None for a
    skeleton's empty handle); ``epoch`` is the step index (-1 = prologue)."""

    __slots__ = ("dev", "hid", "epoch", "shape", "host")

    def __init__(self, dev, hid: int, epoch: int, shape: tuple):
        self.dev = dev
        self.hid = hid
        self.epoch = epoch
        self.shape = shape
        self.host = None

    def rank(self):
        return len(self.shape)


def is_tensor(v) -> bool:
    return isinstance(v, (Val, Tensor, SyntheticTensor))


def fmt_value(v, top: bool = True) -> str:
    """Print formatting: shortest round-trip floats, nested-bracket lists."""
    if isinstance(v, bool):
        return "true" if v else "false"
    if isinstance(v, float):
        return repr(v)
    if isinstance(v, int):
        return str(v)
    if isinstance(v, str):
        return v if top else repr(v)
    if isinstance(v, list):
        return "[" + ", ".join(fmt_value(x, False) for x in v) + "]"
    return str(v)


class StepDiverged(Exception):
    def __init__(self, why: str, pending=None):
        super().__init__(why)
        self.why = why
        self.pending = pending


_KIND_VAL = {k: k.value for k in OpKind}
_IN_KINDS = {k: tuple("h" if b else "e" for b in k)
             for n in range(4) for k in __import__("itertools").product((True, False), repeat=n)}
_SHAPE_CACHE: dict = {}
_LOC_KEYS: dict = {}


def _loc_key(loc) -> tuple:
    k = _LOC_KEYS.get(loc)
    if k is None:
        k = _LOC_KEYS[loc] = (loc.stmt_id, loc.loop_path)
    return k


# ======================================================================= contexts


def _index_input(be, args) -> bool:
    """TO_INDEX of an external host-side input (dataset tensor) by a host scalar."""
    if not hasattr(be, "put_index") or len(args) != 2 or isinstance(args[0], Val):
        return False
    v = args[1]
    if isinstance(v, bool) or not isinstance(v, (int, float)) or not v > 0:
        return False
    return isinstance(args[0], (Tensor, SyntheticTensor))


class EagerCtx:
    """Inline kernel execution on ``backend``; optionally records a trace."""

    skeleton = False

    def __init__(self, backend, epoch: int, trace: list | None = None):
        self.be = backend
        self.epoch = epoch
        self.trace = trace
        self.next_hid = 0
        self.producer: dict = {}     # hid -> index of its OpEvent in trace

    def _arg(self, v, loc, pos, refs, devs):
        if isinstance(v, Val) and v.epoch == self.epoch:
            refs.append(Handle(v.hid))
            devs.append(v.dev)
        else:
            refs.append(External((loc.stmt_id, pos)))
            devs.append(v.dev if isinstance(v, Val) else self.be.put(lift_host_value(v) if not is_tensor(v) else v))

    def _emit(self, kind, attrs, loc, refs, dev, shape, in_shapes=(), in_values=None) -> Val:
        hid = self.next_hid
        self.next_hid += 1
        if self.trace is not None:
            self.producer[hid] = len(self.trace)
            self.trace.append(OpEvent(kind, attrs, loc, refs, [hid], False, tuple(shape), tuple(in_shapes),
                                      in_values))
        return Val(dev, hid, self.epoch, shape)

    def op_site(self, site, args, shapes) -> Val:
        return self.op(site[0], _NOATTRS, args, site[2], shapes)

    def op(self, kind: OpKind, attrs: dict, args: list, loc, shapes: list) -> Val:
        out_shape = infer_shape(kind, attrs, shapes)[0]
        refs, devs = [], []
        if kind is OpKind.TO_INDEX and _index_input(self.be, args):
            # an external input turned into indices: the backend applies TO_INDEX to the f64
            # values while uploading them (same trace refs, no separate op launch)
            refs += [External((loc.stmt_id, 0)), External((loc.stmt_id, 1))]
            dev = self.be.put_index(args[0], float(args[1]))
        else:
            for p, v in enumerate(args):
                self._arg(v, loc, p, refs, devs)
            dev = self.be.exec_op(kind, attrs, devs)
        vals = tuple(float(v) if isinstance(v, (int, float)) else None for v in args) if self.trace is not None \
            else None
        return self._emit(kind, attrs, loc, refs, dev, out_shape, [tuple(s) for s in shapes], vals)

    def read_var(self, name: str, loc) -> Val:
        dev = self.be.var_read(name)
        return self._emit(OpKind.READ_VAR, {"var_name": name}, loc, [], dev, self.be.var_shape(name))

    def assign_var(self, name: str, v, loc, shape) -> Val:
        refs, devs = [], []
        self._arg(v, loc, 0, refs, devs)
        self.be.var_assign(name, devs[0])
        return self._emit(OpKind.ASSIGN_VAR, {"var_name": name}, loc, refs, devs[0], shape, [tuple(shape)])

    def var_shape(self, name: str) -> tuple:
        return self.be.var_shape(name)

    def materialize(self, v) -> Tensor:
        if isinstance(v, Val):
            if v.host is None:
                v.host = self.be.get(v.dev)
            if self.trace is not None and v.epoch == self.epoch:
                self.trace[self.producer[v.hid]].fetch_after = True
            return v.host
        if isinstance(v, SyntheticTensor):
            return v.materialize()
        return v

    def loop_enter(self, lid):
        if self.trace is not None:
            self.trace.append(LoopEnter(lid))

    def loop_iter(self, lid):
        if self.trace is not None:
            self.trace.append(LoopIterStart(lid))

    def loop_exit(self, lid):
        if self.trace is not None:
            self.trace.append(LoopExit(lid))

    def emit_print(self, interp, line: str):
        interp.out.append(line)

    def finish(self):
        if self.trace is not None:
            self.trace.append(StepEnd())


class SkeletonCtx:
    """Skeleton execution against a running pass."""

    skeleton = True

    def __init__(self, backend, epoch: int, cursor, chan, check: bool = False, stats=None):
        self.be = backend
        self.epoch = epoch
        self.cursor = cursor
        self.ch = chan
        self.check = check
        self.stats = stats
        self.next_hid = 0
        self.var_shapes = dict(backend.var_shapes())
        self.prints: list = []
        self.tg_nodes = {}

    def _node(self, nid):
        n = self.tg_nodes.get(nid)
        if n is None:
            n = self.cursor.tg.find(nid)
            self.tg_nodes[nid] = n
        return n

    def _op(self, kind, attrs, loc, args, shape) -> Val:
        epoch = self.epoch
        hids = []
        feeds = None
        for p, v in enumerate(args):
            if type(v) is Val and v.epoch == epoch:
                hids.append(v.hid)
            else:
                hids.append(None)
                if feeds is None:
                    feeds = []
                feeds.append((p, v))
        hid = self.next_hid
        self.next_hid = hid + 1
        in_kinds = _IN_KINDS[tuple(h is not None for h in hids)]
        key = ("op", _KIND_VAL[kind], canonical_attrs(attrs) if attrs else (), _loc_key(loc), in_kinds)
        try:
            nid, _, decisions = self.cursor.advance(key, hids, hid)
        except Diverged as d:
            refs = [Handle(h) if h is not None else External((loc.stmt_id, p)) for p, h in enumerate(hids)]
            raise StepDiverged(d.why, OpEvent(kind, attrs, loc, refs, [hid])) from None
        ch = self.ch
        for d in decisions:
            ch.decide(d)
        if feeds is not None:
            for p, v in feeds:
                if isinstance(v, Val):
                    ch.feed((nid, p), v.dev)
                else:
                    ch.feed((nid, p), v if is_tensor(v) else lift_host_value(v))
        return Val(None, hid, epoch, shape)

    def op_site(self, site, args, shapes) -> Val:
        """Attr-less op from a compiled call site ``(kind, kind value, loc, loc key)``."""
        kind, kval, loc, lkey = site
        ck = (kval, tuple(shapes))
        shape = _SHAPE_CACHE.get(ck)
        if shape is None:
            shape = _SHAPE_CACHE[ck] = infer_shape(kind, _NOATTRS, shapes)[0]
        epoch = self.epoch
        a0 = args[0]
        h0 = a0.hid if (type(a0) is Val and a0.epoch == epoch) else None
        if len(args) == 2:
            a1 = args[1]
            h1 = a1.hid if (type(a1) is Val and a1.epoch == epoch) else None
            hids = [h0, h1]
            in_kinds = ("h" if h0 is not None else "e", "h" if h1 is not None else "e")
        elif len(args) > 2:
            hids = [a.hid if (type(a) is Val and a.epoch == epoch) else None for a in args]
            in_kinds = _IN_KINDS[tuple(h is not None for h in hids)]
        else:
            hids = [h0]
            in_kinds = ("h",) if h0 is not None else ("e",)
        hid = self.next_hid
        self.next_hid = hid + 1
        try:
            nid, _, decisions = self.cursor.advance(("op", kval, (), lkey, in_kinds), hids, hid)
        except Diverged as d:
            refs = [Handle(h) if h is not None else External((loc.stmt_id, p)) for p, h in enumerate(hids)]
            raise StepDiverged(d.why, OpEvent(kind, {}, loc, refs, [hid])) from None
        ch = self.ch
        for d in decisions:
            ch.decide(d)
        for p, h in enumerate(hids):
            if h is None:
                v = args[p]
                if isinstance(v, Val):
                    ch.feed((nid, p), v.dev)
                else:
                    ch.feed((nid, p), v if is_tensor(v) else lift_host_value(v))
        return Val(None, hid, epoch, shape)

    def op(self, kind, attrs, args, loc, shapes) -> Val:
        if attrs:
            shape = infer_shape(kind, attrs, shapes)[0]
        else:
            ck = (kind, tuple(shapes))
            shape = _SHAPE_CACHE.get(ck)
            if shape is None:
                shape = _SHAPE_CACHE[ck] = infer_shape(kind, attrs, shapes)[0]
        return self._op(kind, attrs, loc, args, shape)

    def read_var(self, name, loc) -> Val:
        return self._op(OpKind.READ_VAR, {"var_name": name}, loc, [], self.var_shapes[name])

    def assign_var(self, name, v, loc, shape) -> Val:
        out = self._op(OpKind.ASSIGN_VAR, {"var_name": name}, loc, [v], shape)
        self.var_shapes[name] = shape
        return out

    def var_shape(self, name):
        return self.var_shapes[name]

    def materialize(self, v) -> Tensor:
        if isinstance(v, Val):
            if v.host is not None:
                return v.host
            if v.epoch != self.epoch:
                v.host = self.be.get(v.dev)
                return v.host
            nid, k = self.cursor.producer_of(v.hid)
            if not self._node(nid).fetch:
                raise StepDiverged(f"materialising node {nid}, which the graph does not fetch")
            t0 = time.perf_counter()
            v.host = self.ch.fetch(nid, k)
            if self.stats is not None:
                self.stats.python_stall_s += time.perf_counter() - t0
            if self.check and v.host.shape != v.shape:
                raise CoexError(f"skeleton-check: fetched shape {v.host.shape} != handle shape {v.shape}")
            return v.host
        if isinstance(v, SyntheticTensor):
            return v.materialize()
        return v

    def _loop(self, fn, lid):
        try:
            for d in fn(lid):
                self.ch.decide(d)
        except Diverged as d:
            raise StepDiverged(d.why) from None

    def loop_enter(self, lid):
        self._loop(self.cursor.loop_enter, lid)

    def loop_iter(self, lid):
        self._loop(self.cursor.loop_iter, lid)

    def loop_exit(self, lid):
        self._loop(self.cursor.loop_exit, lid)

    def emit_print(self, interp, line: str):
        self.prints.append(line)

    def finish(self):
        try:
            for d in self.cursor.step_end():
                self.ch.decide(d)
        except Diverged as d:
            raise StepDiverged(d.why) from None


# ======================================================================= interpreter


class Interp:
    """Evaluator over a parsed :class:`~.lang.ast.Program`.

    Each AST node is compiled once into a Python closure ``f(ctx, env)``; a step
    runs the closures of the step body.  Compilation resolves everything that
    does not change between steps (variable vs local names, op kinds, constant
    literals, prologue vs body), so the per-op host cost of the skeleton -- the
    part that overlaps the device pass -- is a few closure calls."""

    def __init__(self, program: ast.Program, dataset, backend, seed: int = 0):
        self.prog = program
        self.ds = dataset
        self.be = backend
        self.seed = seed
        self.var_names = set(program.var_names)
        self.out: list = []            # flushed printed lines
        self.prologue_env: dict = {}
        self.step = -1
        # value-branch margins: every ordered comparison with a float operand
        # -- the conditions a fetched value can drive -- logs (step, line, col, op, a, b);
        # a decision is robust to the precision mode's error when |a-b| / max(|a|,|b|)
        # exceeds that mode's tolerance (Orchestrator.margins())
        self.margin_log: list = []
        self._body = self._c_block(program.body, False)

    # ------------------------------------------------------------------ driver API
    def run_prologue(self):
        self.step = -1
        env: dict = {}
        ctx = EagerCtx(self.be, -1, None)
        for f in self._c_block(self.prog.prologue, True):
            f(ctx, env)
        self.prologue_env = env

    def run_step(self, step: int, ctx) -> None:
        """Run the step body under ``ctx`` (raises StepDiverged in skeleton mode)."""
        self.step = step
        env = dict(self.prologue_env)
        for f in self._body:
            f(ctx, env)
        ctx.finish()

    def _err(self, msg, node) -> EvalError:
        return EvalError(msg, self.step, node.pos.line, node.pos.col)

    # ------------------------------------------------------------------ statements
    def _c_block(self, stmts, prologue) -> list:
        return [self._c_stmt(st, prologue) for st in stmts]

    def _wrap(self, st, body):
        it = self

        def run(ctx, env):
            try:
                body(ctx, env)
            except (EvalError, StepDiverged, ShapeMiss):
                raise
            except CoexError as e:
                raise it._err(str(e), st) from e

        return run

    def _c_cond(self, e, loc, st):
        f = self._c_expr(e, loc)
        it = self

        def cond(ctx, env):
            v = f(ctx, env)
            if v is True or v is False:
                return v
            raise it._err(f"non-boolean condition ({fmt_value(v)})", st)

        return cond

    def _c_stmt(self, st, prologue):
        loc = st.loc()
        be = self.be
        if isinstance(st, ast.VarDecl):
            f = self._c_expr(st.expr, loc)
            name = st.name

            def body(ctx, env):
                v = f(ctx, env)
                be.var_define(name, v.dev if isinstance(v, Val) else (v if is_tensor(v) else lift_host_value(v)))
        elif isinstance(st, (ast.LetDecl, ast.Assign)):
            f = self._c_expr(st.expr, loc)
            name = st.name
            if isinstance(st, ast.Assign) and name in self.var_names:
                if prologue:
                    def body(ctx, env):
                        v = f(ctx, env)
                        if not is_tensor(v):
                            v = lift_host_value(v)
                        be.var_assign(name, v.dev if isinstance(v, Val) else be.put(v))
                else:
                    def body(ctx, env):
                        v = f(ctx, env)
                        if not is_tensor(v):
                            v = lift_host_value(v)
                        ctx.assign_var(name, v, loc, tuple(v.shape))
            else:
                def body(ctx, env):
                    env[name] = f(ctx, env)
        elif isinstance(st, ast.Print):
            f = self._c_expr(st.expr, loc)
            it = self

            def body(ctx, env):
                v = f(ctx, env)
                if is_tensor(v):
                    v = ctx.materialize(v).to_nested()
                ctx.emit_print(it, fmt_value(v))
        elif isinstance(st, ast.If):
            arms = [(self._c_cond(st.cond, loc, st), self._c_block(st.then, prologue))]
            arms += [(self._c_cond(c, loc, st), self._c_block(blk, prologue)) for c, blk in st.elifs]
            orelse = self._c_block(st.orelse, prologue) if st.orelse is not None else None

            def body(ctx, env):
                for cond, blk in arms:
                    if cond(ctx, env):
                        for g in blk:
                            g(ctx, env)
                        return
                if orelse is not None:
                    for g in orelse:
                        g(ctx, env)
        elif isinstance(st, ast.While):
            cond = self._c_cond(st.cond, loc, st)
            blk = self._c_block(st.body, prologue)
            lid = st.loop_id

            def body(ctx, env):
                ctx.loop_enter(lid)
                while cond(ctx, env):
                    ctx.loop_iter(lid)
                    for g in blk:
                        g(ctx, env)
                ctx.loop_exit(lid)
        elif isinstance(st, ast.For):
            cnt = self._c_expr(st.count, loc)
            blk = self._c_block(st.body, prologue)
            lid = st.loop_id
            var = st.var
            it = self

            def body(ctx, env):
                n = cnt(ctx, env)
                if isinstance(n, float) and n.is_integer():
                    n = int(n)
                if isinstance(n, bool) or not isinstance(n, int):
                    raise it._err(f"range() count must be an integer, got {fmt_value(n)}", st)
                ctx.loop_enter(lid)
                for i in range(n):
                    ctx.loop_iter(lid)
                    env[var] = i
                    for g in blk:
                        g(ctx, env)
                ctx.loop_exit(lid)
        else:  # pragma: no cover
            raise self._err(f"unknown statement {type(st).__name__}", st)
        return self._wrap(st, body)

    # ------------------------------------------------------------------ expressions
    def _host_fn(self, f, e):
        it = self

        def g(ctx, env):
            v = f(ctx, env)
            if isinstance(v, (Val, Tensor, SyntheticTensor)):
                raise it._err("tensor value in a host expression; use item()", e)
            return v

        return g

    def _c_expr(self, e, loc):
        it = self
        if isinstance(e, (ast.Num, ast.Str, ast.Bool)):
            c = e.value
            return lambda ctx, env: c
        if isinstance(e, ast.Ident):
            name = e.name
            if name in self.var_names:
                be = self.be

                def var(ctx, env):
                    if it.step < 0:
                        return Val(be.var_read(name), -1, -1, be.var_shape(name))
                    return ctx.read_var(name, loc)
                return var
            if name == "step":
                return lambda ctx, env: max(it.step, 0)

            def ident(ctx, env):
                try:
                    return env[name]
                except KeyError:
                    raise it._err(f"undefined name {name!r}", e) from None
            return ident
        if isinstance(e, ast.OpCall):
            return self._c_opcall(e, loc)
        if isinstance(e, ast.Input):
            shp = None if e.shape is None else self._c_shape(e.shape, loc)
            name = e.name
            ds = self.ds
            if shp is None:
                return lambda ctx, env: ds.next(name, None, it.step)
            return lambda ctx, env: ds.next(name, shp(ctx, env), it.step)
        if isinstance(e, ast.Native):
            fs = [self._c_expr(a, loc) for a in e.args]
            name = e.name

            def native(ctx, env):
                args = []
                for f in fs:
                    v = f(ctx, env)
                    args.append(ctx.materialize(v).to_nested() if is_tensor(v) else v)
                return eval_native(name, args, it.seed, it.step)
            return native
        if isinstance(e, ast.Item):
            f = self._c_expr(e.operand, loc)

            def item(ctx, env):
                v = f(ctx, env)
                return ctx.materialize(v).to_nested() if is_tensor(v) else v
            return item
        if isinstance(e, ast.Not):
            f = self._host_fn(self._c_expr(e.operand, loc), e)

            def not_(ctx, env):
                v = f(ctx, env)
                if not isinstance(v, bool):
                    raise it._err("'not' needs a boolean", e)
                return not v
            return not_
        if isinstance(e, ast.NegOp):
            f = self._host_fn(self._c_expr(e.operand, loc), e)

            def neg(ctx, env):
                v = f(ctx, env)
                if isinstance(v, bool) or not isinstance(v, (int, float)):
                    raise it._err("unary '-' needs a number", e)
                return -v
            return neg
        if isinstance(e, ast.BinOp):
            return self._c_binop(e, loc)
        if isinstance(e, ast.ShapeLit):     # a bracket literal outside a shape position: host list
            fs = [self._host_fn(self._c_expr(d, loc), d) for d in e.dims]
            return lambda ctx, env: [f(ctx, env) for f in fs]
        raise self._err(f"unknown expression {type(e).__name__}", e)

    def _c_binop(self, e, loc):
        it = self
        op = e.op
        fa = self._host_fn(self._c_expr(e.left, loc), e)
        fb = self._host_fn(self._c_expr(e.right, loc), e)
        if op in ("and", "or"):
            want = op == "or"

            def logic(ctx, env):
                a = fa(ctx, env)
                if not isinstance(a, bool):
                    raise it._err(f"'{op}' needs booleans", e)
                if a is want:
                    return a
                b = fb(ctx, env)
                if not isinstance(b, bool):
                    raise it._err(f"'{op}' needs booleans", e)
                return b
            return logic
        if op == "==":
            return lambda ctx, env: fa(ctx, env) == fb(ctx, env)
        if op == "!=":
            return lambda ctx, env: fa(ctx, env) != fb(ctx, env)
        impl = _BINOPS[op]
        ordered = op in ("<", "<=", ">", ">=")
        line, col = e.pos.line, e.pos.col

        def arith(ctx, env):
            a = fa(ctx, env)
            b = fb(ctx, env)
            ta, tb = type(a), type(b)
            if (ta is int or ta is float) and (tb is int or tb is float):
                if op == "/" and b == 0:
                    raise it._err("division by zero", e)
                if ordered and (ta is float or tb is float):
                    it.margin_log.append((it.step, line, col, op, a, b))
                return impl(a, b)
            if ta is str and tb is str and op in ("+", "<", "<=", ">", ">="):
                return impl(a, b)
            raise it._err(f"operator '{op}' needs numbers, got {fmt_value(a)} and {fmt_value(b)}", e)
        return arith

    def _c_shape(self, s: ast.ShapeLit, loc):
        it = self
        fs = [(self._host_fn(self._c_expr(d, loc), d), d) for d in s.dims]

        def shape(ctx, env):
            dims = []
            for f, d in fs:
                v = f(ctx, env)
                if isinstance(v, float) and v.is_integer():
                    v = int(v)
                if isinstance(v, bool) or not isinstance(v, int) or v < 0:
                    raise it._err(f"shape dimension must be a non-negative integer, got {fmt_value(v)}", d)
                dims.append(v)
            return tuple(dims)
        return shape

    @staticmethod
    def _shape_of(v) -> tuple:
        t = type(v)
        if t is Val or t is Tensor or t is SyntheticTensor:
            return v.shape
        if isinstance(v, list):
            return lift_host_value(v).shape
        return ()

    def _c_opcall(self, e: ast.OpCall, loc):
        it = self
        name = e.name
        kind = OP_BY_NAME[name]
        shape_of = self._shape_of
        if name == "fill":
            shp = self._c_shape(e.args[0], loc)
            fv = self._host_fn(self._c_expr(e.args[1], loc), e)

            def fill(ctx, env):
                shape = shp(ctx, env)
                val = fv(ctx, env)
                if isinstance(val, bool) or not isinstance(val, (int, float)):
                    raise it._err("fill value must be a number", e)
                return ctx.op(kind, {"shape": shape, "value": float(val)}, [], loc, [])
            return fill
        fx = self._c_expr(e.args[0], loc)
        if name == "reshape":
            tgt = self._c_shape(e.args[1], loc)

            def reshape(ctx, env):
                x = fx(ctx, env)
                return ctx.op(kind, {"target_shape": tgt(ctx, env)}, [x], loc, [shape_of(x)])
            return reshape
        if name == "transpose":
            perm_f = self._c_shape(e.args[1], loc) if len(e.args) == 2 else None

            def transpose(ctx, env):
                x = fx(ctx, env)
                shp = shape_of(x)
                perm = perm_f(ctx, env) if perm_f is not None else tuple(range(len(shp) - 1, -1, -1))
                return ctx.op(kind, {"perm": tuple(perm)}, [x], loc, [shp])
            return transpose
        if name in CONV_NAMES:
            # extension ops with tensor operands + a trailing shape literal ([k, s, p] / [vocab])
            ftens = [fx] + [self._c_expr(a, loc) for a in e.args[1:-1]]
            geo = self._c_shape(e.args[-1], loc)
            akey = "dims" if name in DIMS_NAMES else "conv"

            def conv(ctx, env):
                xs = [f(ctx, env) for f in ftens]
                if any(isinstance(v, str) for v in xs):
                    raise it._err(f"{name}: string operand", e)
                return ctx.op(kind, {akey: tuple(geo(ctx, env))}, xs, loc, [shape_of(v) for v in xs])
            return conv
        if name in SCALE_NAMES:
            ftens = [fx] + [self._c_expr(a, loc) for a in e.args[1:-1]]
            fsc = self._host_fn(self._c_expr(e.args[-1], loc), e)

            def scaled(ctx, env):
                xs = [f(ctx, env) for f in ftens]
                if any(isinstance(v, str) for v in xs):
                    raise it._err(f"{name}: string operand", e)
                sc = fsc(ctx, env)
                if isinstance(sc, bool) or not isinstance(sc, (int, float)):
                    raise it._err(f"{name}: scale must be a number", e)
                return ctx.op(kind, {"value": float(sc)}, xs, loc, [shape_of(v) for v in xs])
            return scaled
        site = (kind, kind.value, loc, (loc.stmt_id, loc.loop_path))
        if len(e.args) == 3:
            fy = self._c_expr(e.args[1], loc)
            fz = self._c_expr(e.args[2], loc)

            def ternary(ctx, env):
                x, y, z = fx(ctx, env), fy(ctx, env), fz(ctx, env)
                if isinstance(x, str) or isinstance(y, str) or isinstance(z, str):
                    raise it._err(f"{name}: string operand", e)
                return ctx.op_site(site, [x, y, z], [shape_of(x), shape_of(y), shape_of(z)])
            return ternary
        if len(e.args) == 1:
            def unary(ctx, env):
                x = fx(ctx, env)
                if isinstance(x, str):
                    raise it._err(f"{name}: string operand", e)
                return ctx.op_site(site, [x], [shape_of(x)])
            return unary
        fy = self._c_expr(e.args[1], loc)

        def binary(ctx, env):
            x = fx(ctx, env)
            y = fy(ctx, env)
            if isinstance(x, str) or isinstance(y, str):
                raise it._err(f"{name}: string operand", e)
            return ctx.op_site(site, [x, y], [shape_of(x), shape_of(y)])
        return binary


_NOATTRS: dict = {}
_BINOPS = {
    "+": lambda a, b: a + b, "-": lambda a, b: a - b, "*": lambda a, b: a * b, "/": lambda a, b: a / b,
    "<": lambda a, b: a < b, "<=": lambda a, b: a <= b, ">": lambda a, b: a > b, ">=": lambda a, b: a >= b,
}


def run_imperative(program, dataset, backend, config=None) -> "RunResult":
    """The define-by-run oracle: prologue, then each step inline."""
    from .coexec import Mode, run
    res, _ = run(program, dataset, Mode.imperative, config, backend=backend)
    return res


def parse_program(src_or_prog):
    return lang.parse(src_or_prog) if isinstance(src_or_prog, str) else src_or_prog


__all__ = ["Interp", "EagerCtx", "SkeletonCtx", "StepDiverged", "Val", "fmt_value",
           "run_imperative", "shape_size"]
