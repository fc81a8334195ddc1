"""Orchestrator: the Tracing <-> CoExec phase machine, lazy mode and Stats.

Specification: SPEC.md:488-565 (the reference ships no implementation).

``run(program, dataset, mode, config, backend)``:

* ``imperative`` -- every step inline on the backend (the oracle).
* ``coexec`` -- start in Tracing; merge each traced step; when a trace is
  covered, generate the SymProgram (``graph_regens``) and switch to CoExec.  A
  CoExec step launches one pass and runs the skeleton against it; on
  divergence the pass is cancelled, variables rolled back, prints discarded,
  dataset cursors restored and the step replayed traced, after which the
  machine is back in Tracing (``steps_replayed``, ``phase_transitions``).
* ``lazy`` -- same machine, but the pass only advances when the skeleton needs
  a fetch or reaches StepEnd.
* ``skeleton-check`` -- coexec with extra per-event assertions.

``backend`` executes all tensor work.  This package ships exactly one: the B200
backend (:class:`paper_2201_09210_b200.b200.B200Backend`), used when
``backend`` is None.  There is no CPU fallback here; the CPU restatement used as
the parity oracle lives in the repo's ``oracle/`` test infrastructure.
"""

from __future__ import annotations

import enum
import time
from dataclasses import dataclass, field

from .config import RunConfig
from .errors import BudgetExceeded, EvalError, ShapeMiss
from .graph_gen import GenConfig, structure
from .interp import EagerCtx, Interp, SkeletonCtx, StepDiverged
from .lang import ast
from .trace_graph import Cursor, TraceGraph, merge_trace


class Phase(enum.Enum):
    Tracing = "tracing"
    CoExec = "coexec"
    ImperativeOnly = "imperative_only"


class Mode(enum.Enum):
    imperative = "imperative"
    coexec = "coexec"
    lazy = "lazy"
    skeleton_check = "skeleton-check"


@dataclass
class Stats:
    """Fig. 5 categories + Appendix F counters."""

    python_exec_ms: float = 0.0
    python_stall_ms: float = 0.0
    graph_exec_ms: float = 0.0
    graph_stall_ms: float = 0.0
    phase_transitions: int = 0
    traces_collected: int = 0
    graph_regens: int = 0
    steps_replayed: int = 0
    throughput: float = 0.0
    steps: int = 0
    shape_replays: int = 0          # B200 only: graph specialisation misses (not divergences)
    per_step: list = field(default_factory=list)
    decision_log: list = field(default_factory=list)   # per co-exec step: tuple of decisions
    python_stall_s: float = 0.0     # scratch accumulator used by the skeleton

    def to_json(self) -> dict:
        keys = ("python_exec_ms", "python_stall_ms", "graph_exec_ms", "graph_stall_ms",
                "phase_transitions", "traces_collected", "graph_regens", "steps_replayed",
                "throughput", "steps", "shape_replays")
        d = {k: getattr(self, k) for k in keys}
        d["per_step"] = self.per_step
        return d

    def counters(self) -> tuple:
        """The counters that must be identical across backends (bit-exact parity)."""
        return (self.phase_transitions, self.traces_collected, self.graph_regens, self.steps_replayed)


@dataclass
class RunResult:
    lines: list
    vars: dict
    step_times: list


class _DecisionRecorder:
    """Wraps a pass channel to log decisions for parity comparisons."""

    def __init__(self, ch):
        self.ch = ch
        self.log: list = []

    def decide(self, d):
        self.log.append(d)
        self.ch.decide(d)

    def feed(self, slot, v):
        self.ch.feed(slot, v)

    def fetch(self, nid, k):
        return self.ch.fetch(nid, k)


class Orchestrator:
    def __init__(self, program, dataset, mode: Mode, config: RunConfig, backend):
        self.prog = program
        self.ds = dataset
        self.mode = mode
        self.cfg = config
        self.be = backend
        self.it = Interp(program, dataset, backend, config.seed)
        self.stats = Stats()
        self.tg = TraceGraph()
        self.sp = None
        self.compiled = None
        self.phase = Phase.Tracing
        self.step_times: list = []

    # ---- phases --------------------------------------------------------------
    def _imperative_step(self, step):
        self.it.run_step(step, EagerCtx(self.be, step))

    def _traced_step(self, step) -> list:
        trace: list = []
        self.it.run_step(step, EagerCtx(self.be, step, trace))
        self.stats.traces_collected += 1
        return trace

    def _regenerate(self):
        try:
            self.sp, _ = structure(self.tg, GenConfig(self.cfg.max_ops))
        except BudgetExceeded:
            self.phase = Phase.ImperativeOnly
            self.sp = None
            self.compiled = None
            return
        self.stats.graph_regens += 1
        self.compiled = self.be.compile(self.sp, self.tg)
        self.phase = Phase.CoExec
        self.stats.phase_transitions += 1

    def step_tracing(self, step):
        """SPEC.md:516-524."""
        trace = self._traced_step(step)
        rep = merge_trace(self.tg, trace)
        if rep.covered:
            self._regenerate()
        return rep

    def step_coexec(self, step, lazy: bool):
        """SPEC.md:525-533 (and the lazy variant)."""
        snap = self.ds.snapshot()
        lines_before = len(self.it.out)
        try:
            ch = self.be.begin_pass(self.compiled, lazy=lazy)
        except ShapeMiss:
            # no graph for this shape signature yet and no hint to build one: run inline
            self.stats.shape_replays += 1
            self._imperative_step(step)
            return
        rec = _DecisionRecorder(ch)
        cursor = Cursor(self.tg, self.sp.unrolled)
        ctx = SkeletonCtx(self.be, step, cursor, rec, check=self.mode is Mode.skeleton_check, stats=self.stats)
        t0 = time.perf_counter()
        self.stats.python_stall_s = 0.0
        try:
            self.it.run_step(step, ctx)
        except (StepDiverged, ShapeMiss) as d:
            ch.cancel()
            res = ch.wait()
            self._account_pass(res)
            self.be.rollback()
            del self.it.out[lines_before:]
            self.ds.restore(snap)
            if isinstance(d, ShapeMiss):
                # graph specialisation miss: replay inline, stay in CoExec (not a divergence)
                self.stats.shape_replays += 1
                self._imperative_step(step)
                return
            trace = self._traced_step(step)
            merge_trace(self.tg, trace)
            self.stats.steps_replayed += 1
            self.stats.phase_transitions += 1
            self.phase = Phase.Tracing
            return
        except BaseException:
            ch.cancel()
            try:
                ch.wait()
            finally:
                self.be.rollback()
            raise
        t_wait = time.perf_counter()
        res = ch.wait()
        t1 = time.perf_counter()
        if not res.committed:
            raise EvalError(f"graph pass failed: {res.error}", step)
        self.stats.python_stall_s += t1 - t_wait
        self.stats.python_stall_ms += self.stats.python_stall_s * 1e3
        self.stats.python_exec_ms += (t1 - t0 - self.stats.python_stall_s) * 1e3
        self._account_pass(res)
        self.stats.decision_log.append(tuple(rec.log))
        self.it.out.extend(ctx.prints)

    def _account_pass(self, res):
        self.stats.graph_exec_ms += res.exec_ms
        self.stats.graph_stall_ms += res.stall_ms

    # ---- main loop -----------------------------------------------------------
    def start(self):
        """Run the prologue imperatively."""
        self.it.run_prologue()
        self.next_step = 0

    def step(self) -> Phase:
        """Run the next step in the current phase; returns the phase it ran in."""
        step = self.next_step
        self.next_step += 1
        t0 = time.perf_counter()
        phase = self.phase
        if self.mode is Mode.imperative or phase is Phase.ImperativeOnly:
            self._imperative_step(step)
            self.stats.python_exec_ms += (time.perf_counter() - t0) * 1e3
        elif phase is Phase.Tracing:
            self.step_tracing(step)
            self.stats.python_exec_ms += (time.perf_counter() - t0) * 1e3
        else:
            self.step_coexec(step, lazy=self.mode is Mode.lazy)
        dt = time.perf_counter() - t0
        self.step_times.append(dt)
        self.stats.per_step.append({"step": step, "phase": phase.value, "ms": dt * 1e3})
        return phase

    def margins(self) -> list:
        """Value-driven comparisons evaluated so far (the latest evaluation per step and
        source position): {"step", "line", "col", "op", "a", "b", "rel_margin"} with
        rel_margin = |a - b| / max(|a|, |b|).  A decision whose margin is below the precision
        mode's tolerance may legitimately differ from the f64 oracle's."""
        last = {}
        for st, ln, col, op, a, b in self.it.margin_log:
            last[(st, ln, col)] = (op, a, b)
        out = []
        for (st, ln, col), (op, a, b) in sorted(last.items()):
            den = max(abs(a), abs(b))
            out.append({"step": st, "line": ln, "col": col, "op": op, "a": a, "b": b,
                        "rel_margin": abs(a - b) / den if den > 0 else 0.0})
        return out

    def result(self) -> RunResult:
        return RunResult(list(self.it.out), self.be.snapshot_vars(), self.step_times)

    def run(self):
        self.start()
        t_run = time.perf_counter()
        while self.next_step < self.prog.step_count:
            self.step()
        total = time.perf_counter() - t_run
        self.stats.steps = self.prog.step_count
        self.stats.throughput = self.prog.step_count / total if total > 0 else 0.0
        return self.result(), self.stats


def default_backend():
    """The B200 backend; fails loudly when the CUDA extension or GPU is missing."""
    from .b200 import B200Backend
    return B200Backend()


def run(program, dataset, mode=Mode.coexec, config: RunConfig | None = None, backend=None):
    """Run ``program`` in ``mode``. Returns (RunResult, Stats)."""
    from . import lang
    if isinstance(program, str):
        program = lang.parse(program)
    if isinstance(mode, str):
        mode = Mode(mode)
    cfg = config or RunConfig()
    be = backend if backend is not None else default_backend()
    return Orchestrator(program, dataset, mode, cfg, be).run()


__all__ = ["Phase", "Mode", "Stats", "RunResult", "run", "Orchestrator", "ast"]
