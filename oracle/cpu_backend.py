"""CPU graph runner + eager backend (TEST INFRASTRUCTURE, see oracle/__init__.py).

Restates the reference's symbolic executor from SPEC.md:420-486:

* ``ChannelSet``: decision FIFO, per-slot feed FIFOs, per-node
  fetch FIFOs, one-shot cancel.  Bounded blocking pushes for decisions/feeds
  (capacity 64, coex/config.py:10), cancel-interruptible blocking pops.  Fetch
  FIFOs are unbounded so an unconsumed fetch can never block the runner
  ("no lost fetches").
* ``run_pass`` walks the SymProgram sequentially on its own
  thread: ExecOp -> ``oracle.kernels.execute_kernel``; ReadVar sees overlay then
  committed; AssignVar writes the overlay; SwitchCase / While pop decisions and
  assert the branch / loop id (DecisionMismatch otherwise); commit at the end,
  Cancelled (overlay kept for rollback) when cancel fires.
* Lazy mode: the same pass, advanced on the caller's thread
  only when the skeleton needs a fetch or waits for StepEnd.

Input resolution follows the value-binding rule of the product's TraceGraph:
an in-graph input is the latest executed of its candidate producers.
"""

from __future__ import annotations

import threading
import time
from collections import defaultdict, deque

from paper_2201_09210_b200.dataset import SyntheticTensor
from paper_2201_09210_b200.errors import (ChannelClosed, DecisionMismatch, InFlightPass,
                                          PassCancelled)
from paper_2201_09210_b200.graph_gen import (ExecOp, InputFeed, OutputFetch, SwitchCase,
                                             UnrolledLoop, While)
from paper_2201_09210_b200.dp import AllReduce, shard_program, shard_value
from paper_2201_09210_b200.runner_api import PassResult
from paper_2201_09210_b200.tensor import OpKind, Tensor
from paper_2201_09210_b200.trace_graph import CaseDecision, LoopDecision

from .kernels import bn_sync, execute_kernel

_NEED = object()
SYNC_BN = (OpKind.BATCHNORM, OpKind.BATCHNORM_DX, OpKind.BN_DGAMMA)


class ChannelSet:
    def __init__(self, capacity: int = 64, lazy: bool = False):
        self.capacity = capacity
        self.lazy = lazy
        self.cv = threading.Condition()
        self.decisions = deque()
        self.feeds = defaultdict(deque)
        self.fetches = defaultdict(deque)
        self.commit = deque()          # commit token: the skeleton reached StepEnd
        self.cancelled = False

    def _push(self, q, item, bounded=True):
        with self.cv:
            while bounded and not self.lazy and len(q) >= self.capacity and not self.cancelled:
                self.cv.wait()
            q.append(item)
            self.cv.notify_all()

    def push_decision(self, d):
        self._push(self.decisions, d)

    def push_feed(self, slot, t):
        self._push(self.feeds[slot], t)

    def push_fetch(self, nid, t):
        self._push(self.fetches[nid], t, bounded=False)

    def cancel(self):
        with self.cv:
            self.cancelled = True
            self.cv.notify_all()


class VariableStore:
    """committed + overlay; reads see overlay first."""

    def __init__(self):
        self.committed: dict = {}
        self.overlay: dict = {}
        self.in_flight = False

    def read(self, name):
        v = self.overlay.get(name)
        return self.committed[name] if v is None else v

    def commit(self):
        self.committed.update(self.overlay)
        self.overlay.clear()

    def rollback(self):
        self.overlay.clear()

    def snapshot(self) -> dict:
        if self.in_flight:
            raise InFlightPass("snapshot_vars during an in-flight pass")
        return dict(self.committed)


def _host(v) -> Tensor:
    return v.materialize() if isinstance(v, SyntheticTensor) else v


class _Runner:
    """One pass over a SymProgram as a generator: yields _NEED when it must block."""

    def __init__(self, sp, ch: ChannelSet, vs: VariableStore, dp=None):
        self.sp = sp
        self.ch = ch
        self.vs = vs
        self.dp = dp
        self.vals: dict = {}       # node id -> (tick, Tensor)
        self.fed: dict = {}        # slot -> Tensor
        self.tick = 0
        self.ops = 0
        self.fetches = 0
        self.exec_s = 0.0
        self.stall_s = 0.0

    def _pop(self, q):
        t0 = None
        while True:
            with self.ch.cv:
                if self.ch.cancelled:
                    raise PassCancelled()
                if q:
                    item = q.popleft()
                    self.ch.cv.notify_all()
                    if t0 is not None:
                        self.stall_s += time.perf_counter() - t0
                    return item
            if t0 is None:
                t0 = time.perf_counter()
            yield _NEED

    def _resolve(self, b):
        if b.fed:
            return self.fed[b.slot]
        best = None
        for c in b.cands:
            v = self.vals.get(c)
            if v is not None and (best is None or v[0] > best[0]):
                best = v
        if best is None:
            raise ChannelClosed(f"no executed producer among {b.cands}")
        return best[1]

    def _exec(self, x: ExecOp):
        t0 = time.perf_counter()
        if x.kind is OpKind.READ_VAR:
            out = self.vs.read(x.attrs["var_name"])
        else:
            ins = [self._resolve(b) for b in x.inputs]
            if self.dp is not None and "rows" in x.attrs and x.kind in SYNC_BN:
                # synchronised batch norm of a row shard (dp.py marks it with the global rows)
                out = Tensor._wrap(bn_sync(x.kind, [t.data for t in ins], x.attrs["rows"], self.dp.allreduce))
            else:
                out = execute_kernel(x.kind, x.attrs, ins)[0]
            if x.kind is OpKind.ASSIGN_VAR:
                self.vs.overlay[x.attrs["var_name"]] = out
        self.tick += 1
        self.vals[x.node_id] = (self.tick, out)
        self.ops += 1
        self.exec_s += time.perf_counter() - t0

    def run(self, insts):
        for x in insts:
            if self.ch.cancelled:
                raise PassCancelled()
            if isinstance(x, ExecOp):
                self._exec(x)
            elif isinstance(x, InputFeed):
                self.fed[x.slot] = _host((yield from self._pop(self.ch.feeds[x.slot])))
            elif isinstance(x, OutputFetch):
                self.ch.push_fetch(x.node_id, self.vals[x.node_id][1])
                self.fetches += 1
            elif isinstance(x, AllReduce):
                tick, t = self.vals[x.node_id]
                self.vals[x.node_id] = (tick, Tensor(t.shape, self.dp.allreduce(t.data, x.avg)))
            elif isinstance(x, SwitchCase):
                d = yield from self._pop(self.ch.decisions)
                if not isinstance(d, CaseDecision) or d.branch_id != x.branch_id:
                    raise DecisionMismatch(f"switch {x.branch_id} popped {d}")
                yield from self.run(x.cases[d.case_index])
            elif isinstance(x, While):
                while True:
                    d = yield from self._pop(self.ch.decisions)
                    if not isinstance(d, LoopDecision) or d.loop_id != x.loop_id:
                        raise DecisionMismatch(f"while loop {x.loop_id} popped {d}")
                    if not d.cont:
                        break
                    yield from self.run(x.body)
            elif isinstance(x, UnrolledLoop):
                for body in x.bodies:
                    yield from self.run(body)

    def whole(self):
        yield from self.run(self.sp.body)
        # never commit before the skeleton confirms StepEnd: a pass that ran to
        # its end ahead of a late divergence must still be cancellable
        yield from self._pop(self.ch.commit)


def run_pass(sp, ch: ChannelSet, vs: VariableStore, dp=None) -> PassResult:
    """Blocking structured execution of ``sp``."""
    r = _Runner(sp, ch, vs, dp)
    gen = r.whole()
    vs.in_flight = True
    try:
        for _ in gen:
            with ch.cv:
                ch.cv.wait(timeout=0.05)
    except PassCancelled:
        return PassResult(False, r.exec_s * 1e3, r.stall_s * 1e3, r.ops, r.fetches)
    finally:
        vs.in_flight = False
    vs.commit()
    return PassResult(True, r.exec_s * 1e3, r.stall_s * 1e3, r.ops, r.fetches)


def rollback(vs: VariableStore):
    vs.rollback()


def snapshot_vars(vs: VariableStore) -> dict:
    return vs.snapshot()


class CpuPass:
    """The skeleton-facing side of one pass (threaded, or lazy on the caller's thread)."""

    def __init__(self, sp, vs: VariableStore, capacity: int, lazy: bool, dp=None, sharded=()):
        self.dp = dp
        self.sharded = set(sharded)
        self.ch = ChannelSet(capacity, lazy)
        self.vs = vs
        self.lazy = lazy
        self.result = None
        self.error = None
        self.done = False
        self.consumed: dict = {}    # node id -> fetch entries already taken
        if lazy:
            self.runner = _Runner(sp, self.ch, vs, dp)
            self.gen = self.runner.whole()
            vs.in_flight = True
        else:
            self.thread = threading.Thread(target=self._thread_main, args=(sp,), daemon=True)
            self.thread.start()

    def _thread_main(self, sp):
        try:
            self.result = run_pass(sp, self.ch, self.vs, self.dp)
        except BaseException as e:  # surfaced as ChannelClosed to the skeleton
            self.error = e
            self.ch.cancel()
        finally:
            self.done = True
            with self.ch.cv:
                self.ch.cv.notify_all()

    def _finish(self, committed: bool):
        self.done = True
        self.vs.in_flight = False
        if committed:
            self.vs.commit()
        r = self.runner
        self.result = PassResult(committed, r.exec_s * 1e3, r.stall_s * 1e3, r.ops, r.fetches)

    def _advance(self, ready):
        """Lazy mode: run the pass on this thread until ``ready()`` or the pass ends.
        Everything the pass consumes before a sync point has already been published,
        so a pass that blocks first is starved (an orchestrator bug)."""
        while not self.done and not ready():
            try:
                r = next(self.gen)
            except StopIteration:
                self._finish(True)
            except PassCancelled:
                self._finish(False)
            except BaseException as e:
                self.error = e
                self._finish(False)
            else:
                if r is _NEED and not ready():
                    raise ChannelClosed("lazy pass starved: input not published before a sync point")

    def decide(self, d):
        self.ch.push_decision(d)

    def feed(self, slot, v):
        if slot in self.sharded:
            v = shard_value(_host(v) if not hasattr(v, "state") else v, self.dp.rank, self.dp.world)
        self.ch.push_feed(slot, v)

    def _take(self, nid: int, k: int):
        q = self.ch.fetches[nid]
        while q and self.consumed.get(nid, 0) < k:
            q.popleft()
            self.consumed[nid] = self.consumed.get(nid, 0) + 1
        if q and self.consumed.get(nid, 0) == k:
            self.consumed[nid] = k + 1
            return q.popleft()
        return None

    def fetch(self, nid: int, k: int) -> Tensor:
        if self.lazy:
            q = self.ch.fetches[nid]
            self._advance(lambda: len(q) > k - self.consumed.get(nid, 0))
        while True:
            with self.ch.cv:
                t = self._take(nid, k)
                if t is not None:
                    return t
                if self.done or self.error is not None:
                    raise ChannelClosed(f"pass ended without a fetch for node {nid}#{k}: {self.error}")
                self.ch.cv.wait(timeout=0.05)

    def cancel(self):
        self.ch.cancel()

    def wait(self) -> PassResult:
        if not self.ch.cancelled:
            self.ch._push(self.ch.commit, True, bounded=False)
        if self.lazy:
            if not self.done and self.ch.cancelled:
                self._finish(False)
            self._advance(lambda: False)
        else:
            self.thread.join()
        if self.error is not None and not self.ch.cancelled:
            return PassResult(False, error=repr(self.error))
        if self.result is None:             # cancelled pass whose runner raised before returning
            return PassResult(False, error=repr(self.error))
        return self.result


class CpuBackend:
    """Oracle backend: numpy kernels, dict variable store, thread-based passes."""

    name = "cpu-oracle"
    precision = "f64"

    def __init__(self, capacity: int = 64, dp=None):
        self.vs = VariableStore()
        self.capacity = capacity
        self.dp = dp
        self.dp_plans: list = []

    # ---- eager
    def put(self, t):
        return _host(t)

    def get(self, v) -> Tensor:
        return _host(v)

    def exec_op(self, kind, attrs, values):
        return execute_kernel(kind, attrs, [_host(v) for v in values])[0]

    def var_define(self, name, value):
        self.vs.committed[name] = _host(value)

    def var_read(self, name):
        return self.vs.read(name)

    def var_assign(self, name, value):
        self.vs.committed[name] = _host(value)

    def var_shape(self, name):
        return self.vs.read(name).shape

    def var_shapes(self) -> dict:
        return {k: v.shape for k, v in self.vs.committed.items()}

    def snapshot_vars(self) -> dict:
        return self.vs.snapshot()

    def rollback(self):
        self.vs.rollback()

    # ---- symbolic
    def compile(self, sp, tg):
        if self.dp is None or self.dp.world <= 1:
            return (sp, ())
        from paper_2201_09210_b200.planner import Planner
        feed_shapes = {(n.id, p): tuple(s) for n in tg.all_nodes() if n.typ == "op" for p, s in n.feed_shapes.items()}
        node_shapes = Planner(sp, tg, {}, self.var_shapes(), feed_shapes, 8).infer_shapes()
        plan = shard_program(sp, feed_shapes, node_shapes, self.dp.batch, self.dp.world)
        self.dp_plans.append(plan)
        return (plan.sp, plan.sharded_slots)

    def begin_pass(self, prog, lazy: bool = False) -> CpuPass:
        sp, sharded = prog
        return CpuPass(sp, self.vs, self.capacity, lazy, self.dp, sharded)
