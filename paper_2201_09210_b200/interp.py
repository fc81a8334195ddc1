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
from .errors import CoexError, EvalError
from .lang import ast
from .natives import eval_native
from .tensor import OpKind, Tensor, infer_shape, lift_host_value, shape_size
from .dataset import SyntheticTensor
from .trace_graph import (Diverged, External, Handle, LoopEnter, LoopExit,
                          LoopIterStart, OpEvent, StepEnd)

OP_BY_NAME = {k.value: k for k in OpKind if k not in (OpKind.READ_VAR, OpKind.ASSIGN_VAR)}


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


# ======================================================================= contexts


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

    def _emit(self, kind, attrs, loc, refs, dev, shape, in_shapes=()) -> Val:
        hid = self.next_hid
        self.next_hid += 1
        if self.trace is not None:
            self.producer[hid] = len(self.trace)
            self.trace.append(OpEvent(kind, attrs, loc, refs, [hid], False, tuple(shape), tuple(in_shapes)))
        return Val(dev, hid, self.epoch, shape)

    def op(self, kind: OpKind, attrs: dict, args: list, loc, shapes: list) -> Val:
        out_shape = infer_shape(kind, attrs, shapes)[0]
        refs, devs = [], []
        for p, v in enumerate(args):
            self._arg(v, loc, p, refs, devs)
        dev = self.be.exec_op(kind, attrs, devs)
        return self._emit(kind, attrs, loc, refs, dev, out_shape, [tuple(s) for s in shapes])

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

    def _advance(self, ev: OpEvent):
        try:
            adv = self.cursor.advance_op(ev)
        except Diverged as d:
            raise StepDiverged(d.why, ev) from None
        for d in adv.decisions:
            self.ch.decide(d)
        return adv

    def _op(self, kind, attrs, loc, args, shape) -> Val:
        refs, feeds = [], []
        for p, v in enumerate(args):
            if isinstance(v, Val) and v.epoch == self.epoch:
                refs.append(Handle(v.hid))
            else:
                refs.append(External((loc.stmt_id, p)))
                feeds.append((p, v))
        hid = self.next_hid
        self.next_hid += 1
        adv = self._advance(OpEvent(kind, attrs, loc, refs, [hid]))
        for p, v in feeds:
            if isinstance(v, Val):
                self.ch.feed((adv.node_id, p), v.dev)
            else:
                self.ch.feed((adv.node_id, p), v if is_tensor(v) else lift_host_value(v))
        return Val(None, hid, self.epoch, shape)

    def op(self, kind, attrs, args, loc, shapes) -> Val:
        return self._op(kind, attrs, loc, args, infer_shape(kind, attrs, shapes)[0])

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
    """Evaluator over a parsed :class:`~.lang.ast.Program`."""

    def __init__(self, program: ast.Program, dataset, backend, seed: int = 0):
        self.prog = program
        self.ds = dataset
        self.be = backend
        self.seed = seed
        self.var_names = set(program.var_names)
        self.out: list = []            # flushed printed lines
        self.prologue_env: dict = {}
        self.step = -1

    # ------------------------------------------------------------------ driver API
    def run_prologue(self):
        self.step = -1
        env: dict = {}
        ctx = EagerCtx(self.be, -1, None)
        self._block(self.prog.prologue, ctx, env, prologue=True)
        self.prologue_env = env

    def run_step(self, step: int, ctx) -> None:
        """Run the step body under ``ctx`` (raises StepDiverged in skeleton mode)."""
        self.step = step
        env = dict(self.prologue_env)
        self._block(self.prog.body, ctx, env, prologue=False)
        ctx.finish()

    # ------------------------------------------------------------------ statements
    def _err(self, msg, node) -> EvalError:
        return EvalError(msg, self.step, node.pos.line, node.pos.col)

    def _block(self, stmts, ctx, env, prologue):
        for st in stmts:
            self._stmt(st, ctx, env, prologue)

    def _stmt(self, st, ctx, env, prologue):
        loc = st.loc()
        try:
            if isinstance(st, ast.VarDecl):
                v = self._expr(st.expr, ctx, env, loc)
                self.be.var_define(st.name, v.dev if isinstance(v, Val) else
                                   (v if is_tensor(v) else lift_host_value(v)))
            elif isinstance(st, (ast.LetDecl, ast.Assign)):
                v = self._expr(st.expr, ctx, env, loc)
                if isinstance(st, ast.Assign) and st.name in self.var_names:
                    if not is_tensor(v):
                        v = lift_host_value(v)
                    if prologue:
                        self.be.var_assign(st.name, v.dev if isinstance(v, Val) else self.be.put(v))
                    else:
                        ctx.assign_var(st.name, v, loc, tuple(v.shape))
                else:
                    env[st.name] = v
            elif isinstance(st, ast.Print):
                v = self._expr(st.expr, ctx, env, loc)
                if is_tensor(v):
                    v = ctx.materialize(v).to_nested()
                ctx.emit_print(self, fmt_value(v))
            elif isinstance(st, ast.If):
                if self._cond(st.cond, ctx, env, loc, st):
                    self._block(st.then, ctx, env, prologue)
                    return
                for c, blk in st.elifs:
                    if self._cond(c, ctx, env, loc, st):
                        self._block(blk, ctx, env, prologue)
                        return
                if st.orelse is not None:
                    self._block(st.orelse, ctx, env, prologue)
            elif isinstance(st, ast.While):
                ctx.loop_enter(st.loop_id)
                while self._cond(st.cond, ctx, env, loc, st):
                    ctx.loop_iter(st.loop_id)
                    self._block(st.body, ctx, env, prologue)
                ctx.loop_exit(st.loop_id)
            elif isinstance(st, ast.For):
                n = self._expr(st.count, ctx, env, loc)
                if isinstance(n, float) and n.is_integer():
                    n = int(n)
                if isinstance(n, bool) or not isinstance(n, int):
                    raise self._err(f"range() count must be an integer, got {fmt_value(n)}", st)
                ctx.loop_enter(st.loop_id)
                for i in range(n):
                    ctx.loop_iter(st.loop_id)
                    env[st.var] = i
                    self._block(st.body, ctx, env, prologue)
                ctx.loop_exit(st.loop_id)
            else:  # pragma: no cover
                raise self._err(f"unknown statement {type(st).__name__}", st)
        except (EvalError, StepDiverged):
            raise
        except CoexError as e:
            raise self._err(str(e), st) from e

    def _cond(self, e, ctx, env, loc, st) -> bool:
        v = self._expr(e, ctx, env, loc)
        if not isinstance(v, bool):
            raise self._err(f"non-boolean condition ({fmt_value(v)})", st)
        return v

    # ------------------------------------------------------------------ expressions
    def _host(self, v, ctx, e):
        if is_tensor(v):
            raise self._err("tensor value in a host expression; use item()", e)
        return v

    def _expr(self, e, ctx, env, loc):
        if isinstance(e, ast.Num):
            return e.value
        if isinstance(e, ast.Str):
            return e.value
        if isinstance(e, ast.Bool):
            return e.value
        if isinstance(e, ast.Ident):
            if e.name in self.var_names:
                if self.step < 0:
                    return Val(self.be.var_read(e.name), -1, -1, self.be.var_shape(e.name))
                return ctx.read_var(e.name, loc)
            if e.name == "step":
                return max(self.step, 0)
            if e.name not in env:
                raise self._err(f"undefined name {e.name!r}", e)
            return env[e.name]
        if isinstance(e, ast.OpCall):
            return self._opcall(e, ctx, env, loc)
        if isinstance(e, ast.Input):
            shape = None if e.shape is None else self._shape(e.shape, ctx, env, loc)
            return self.ds.next(e.name, shape, self.step)
        if isinstance(e, ast.Native):
            args = [self._native_arg(self._expr(a, ctx, env, loc), ctx) for a in e.args]
            return eval_native(e.name, args, self.seed, self.step)
        if isinstance(e, ast.Item):
            v = self._expr(e.operand, ctx, env, loc)
            return ctx.materialize(v).to_nested() if is_tensor(v) else v
        if isinstance(e, ast.Not):
            v = self._host(self._expr(e.operand, ctx, env, loc), ctx, e)
            if not isinstance(v, bool):
                raise self._err("'not' needs a boolean", e)
            return not v
        if isinstance(e, ast.NegOp):
            v = self._host(self._expr(e.operand, ctx, env, loc), ctx, e)
            if isinstance(v, bool) or not isinstance(v, (int, float)):
                raise self._err("unary '-' needs a number", e)
            return -v
        if isinstance(e, ast.BinOp):
            return self._binop(e, ctx, env, loc)
        if isinstance(e, ast.ShapeLit):     # a bracket literal outside a shape position: host list
            return [self._host(self._expr(d, ctx, env, loc), ctx, d) for d in e.dims]
        raise self._err(f"unknown expression {type(e).__name__}", e)

    def _native_arg(self, v, ctx):
        if is_tensor(v):
            return ctx.materialize(v).to_nested()
        return v

    def _binop(self, e, ctx, env, loc):
        op = e.op
        a = self._host(self._expr(e.left, ctx, env, loc), ctx, e)
        if op in ("and", "or"):
            if not isinstance(a, bool):
                raise self._err(f"'{op}' needs booleans", e)
            if (op == "and" and not a) or (op == "or" and a):
                return a
            b = self._host(self._expr(e.right, ctx, env, loc), ctx, e)
            if not isinstance(b, bool):
                raise self._err(f"'{op}' needs booleans", e)
            return b
        b = self._host(self._expr(e.right, ctx, env, loc), ctx, e)
        if op == "==":
            return a == b
        if op == "!=":
            return a != b
        num = (int, float)
        if op == "+" and isinstance(a, str) and isinstance(b, str):
            return a + b
        if isinstance(a, bool) or isinstance(b, bool) or not isinstance(a, num) or not isinstance(b, num):
            if op in ("<", "<=", ">", ">=") and isinstance(a, str) and isinstance(b, str):
                pass
            else:
                raise self._err(f"operator '{op}' needs numbers, got {fmt_value(a)} and {fmt_value(b)}", e)
        if op == "+":
            return a + b
        if op == "-":
            return a - b
        if op == "*":
            return a * b
        if op == "/":
            if b == 0:
                raise self._err("division by zero", e)
            return a / b
        if op == "<":
            return a < b
        if op == "<=":
            return a <= b
        if op == ">":
            return a > b
        if op == ">=":
            return a >= b
        raise self._err(f"unknown operator {op!r}", e)

    def _shape(self, s: ast.ShapeLit, ctx, env, loc) -> tuple:
        dims = []
        for d in s.dims:
            v = self._host(self._expr(d, ctx, env, loc), ctx, d)
            if isinstance(v, float) and v.is_integer():
                v = int(v)
            if isinstance(v, bool) or not isinstance(v, int) or v < 0:
                raise self._err(f"shape dimension must be a non-negative integer, got {fmt_value(v)}", d)
            dims.append(v)
        return tuple(dims)

    @staticmethod
    def _shape_of(v) -> tuple:
        if isinstance(v, (Val, Tensor, SyntheticTensor)):
            return tuple(v.shape)
        if isinstance(v, list):
            return lift_host_value(v).shape
        return ()

    def _opcall(self, e: ast.OpCall, ctx, env, loc):
        name = e.name
        kind = OP_BY_NAME[name]
        if name == "fill":
            shape = self._shape(e.args[0], ctx, env, loc)
            val = self._host(self._expr(e.args[1], ctx, env, loc), ctx, e)
            if isinstance(val, bool) or not isinstance(val, (int, float)):
                raise self._err("fill value must be a number", e)
            return ctx.op(kind, {"shape": shape, "value": float(val)}, [], loc, [])
        x = self._expr(e.args[0], ctx, env, loc)
        if name == "reshape":
            tgt = self._shape(e.args[1], ctx, env, loc)
            return ctx.op(kind, {"target_shape": tgt}, [x], loc, [self._shape_of(x)])
        if name == "transpose":
            shp = self._shape_of(x)
            perm = self._shape(e.args[1], ctx, env, loc) if len(e.args) == 2 else tuple(reversed(range(len(shp))))
            return ctx.op(kind, {"perm": tuple(perm)}, [x], loc, [shp])
        args = [x] + [self._expr(a, ctx, env, loc) for a in e.args[1:]]
        for a in args:
            if isinstance(a, str):
                raise self._err(f"{name}: string operand", e)
        return ctx.op(kind, {}, args, loc, [self._shape_of(a) for a in args])


def run_imperative(program, dataset, backend, config=None) -> "RunResult":
    """The define-by-run oracle: prologue, then each step inline."""
    from .coexec import Mode, run
    res, _ = run(program, dataset, Mode.imperative, config, backend=backend)
    return res


def parse_program(src_or_prog):
    return lang.parse(src_or_prog) if isinstance(src_or_prog, str) else src_or_prog


__all__ = ["Interp", "EagerCtx", "SkeletonCtx", "StepDiverged", "Val", "fmt_value",
           "run_imperative", "shape_size"]
