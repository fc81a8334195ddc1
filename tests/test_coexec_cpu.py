"""Orchestrator acceptance on the CPU oracle (SPEC.md:628-637 criteria 1, 5, 6)
and the graph_runner examples."""

import time

import pytest

from oracle.cpu_backend import ChannelSet, CpuBackend, VariableStore, rollback, run_pass, snapshot_vars
from paper_2201_09210_b200 import coexec, lang
from paper_2201_09210_b200.dataset import SyntheticDataset
from paper_2201_09210_b200.errors import InFlightPass
from paper_2201_09210_b200.graph_gen import ExecOp, structure
from paper_2201_09210_b200.tensor import OpKind, Tensor
from paper_2201_09210_b200.trace_graph import CaseDecision, LoopDecision, TraceGraph, merge_trace
from programs import CORPUS, fuzz_program
from test_trace_graph import fig3_traces

MODES = ["imperative", "coexec", "lazy", "skeleton-check"]


def run(src, mode):
    return coexec.run(lang.parse(src), SyntheticDataset(0), mode, backend=CpuBackend())


def canon(res):
    return res.lines, {k: v.data.tobytes() for k, v in res.vars.items()}


def test_oracle_equivalence_corpus_and_fuzz():
    t0 = time.time()
    for src in list(CORPUS.values()) + [fuzz_program(i) for i in range(200)]:
        ref = canon(run(src, "imperative")[0])
        for m in MODES[1:]:
            assert canon(run(src, m)[0]) == ref
    assert time.time() - t0 < 120


def test_single_path_transitions_after_step2():
    _, st = run(CORPUS["straight"], "coexec")
    assert st.phase_transitions == 1 and st.graph_regens == 1 and st.traces_collected == 2


DEOPT = """
var w = fill([2], 1.0)
steps 100 {
  if step == 50 { w = mul(w, 0.5) } else { w = add(w, fill([2], 0.01)) }
  print(sum(w))
}
"""


def test_deoptimisation_new_path_at_step_50():
    res, st = run(DEOPT, "coexec")
    assert (st.phase_transitions, st.steps_replayed) == (3, 1)
    assert canon(res) == canon(run(DEOPT, "imperative")[0])


UNROLL_CONST = """
var w = fill([2], 1.0)
steps 6 {
  for i in range(3) { w = add(w, fill([2], 1.0)) }
  print(sum(w))
}
"""
UNROLL_VAR = UNROLL_CONST.replace("range(3)", "range(2 + native choice(2, 0))")
UNROLL_FORCED = UNROLL_CONST.replace("range(3)", "range(3 + native mod(step / 5, 1) * 0 + (step == 4) * 1)")


def _sp(src, steps):
    o = coexec.Orchestrator(lang.parse(src), SyntheticDataset(0), coexec.Mode.coexec, coexec.RunConfig(), CpuBackend())
    r, st = o.run()
    return o, st


def test_unrolling_rules():
    from paper_2201_09210_b200.graph_gen import UnrolledLoop, While, count_kind
    o, _ = _sp(UNROLL_CONST, 6)
    assert count_kind(o.sp, While) == 0 and count_kind(o.sp, UnrolledLoop) == 1
    o, _ = _sp(UNROLL_VAR, 6)
    assert count_kind(o.sp, While) == 1


FORCED = """
var w = fill([2], 1.0)
steps 8 {
  let n = 3
  if step == 5 { n = 4 }
  for i in range(n) { w = add(w, fill([2], 1.0)) }
  print(sum(w))
}
"""


def test_unrolled_new_trip_count_diverges_once():
    res, st = run(FORCED, "coexec")
    assert st.steps_replayed == 1
    assert canon(res) == canon(run(FORCED, "imperative")[0])


def test_budget_exceeded_goes_imperative():
    src = "var w = fill([1], 0.0)\nsteps 6 {\n" + "".join(
        f"  if native coin({k}) {{ w = add(w, fill([1], {k}.0)) }} else {{ w = sub(w, fill([1], {k}.0)) }}\n"
        for k in range(6)) + "  print(w)\n}\n"
    o = coexec.Orchestrator(lang.parse(src), SyntheticDataset(0), coexec.Mode.coexec,
                            coexec.RunConfig(max_ops=4), CpuBackend())
    res, st = o.run()
    assert canon(res) == canon(run(src, "imperative")[0])


def _fig4():
    tg = TraceGraph()
    t1, t2 = fig3_traces()
    merge_trace(tg, t1)
    merge_trace(tg, t2)
    sp, _ = structure(tg)
    return tg, sp


def test_run_pass_fig4_driven_by_trace2():
    tg, sp = _fig4()
    vs = VariableStore()
    ch = ChannelSet()
    op2p = [n for n in tg.nodes.values() if n.typ == "op" and n.loc.stmt_id == 9][0]
    ch.push_decision(CaseDecision(tg.start, tg.succ[tg.start].index(op2p.id)))
    ch.push_feed((op2p.id, 0), Tensor.scalar(2.0))
    ch.push_decision(LoopDecision(0, True))
    ch.push_decision(LoopDecision(0, False))
    ch.commit.append(True)
    res = run_pass(sp, ch, vs)
    assert res.committed and res.ops == 3                 # Op2', Op3, one Op4
    op3 = [n for n in tg.nodes.values() if n.typ == "op" and n.loc.stmt_id == 10][0]
    assert len(ch.fetches[op3.id]) == 1


def test_run_pass_linear_and_cancel():
    tg = TraceGraph()
    from test_trace_graph import TB
    t = TB()
    a = t.op(0, kind=OpKind.FILL)
    t.ev[-1].attrs = {"shape": (2,), "value": 1.0}
    b = t.op(1, a)
    t.op(2, b)
    merge_trace(tg, t.end())
    sp, _ = structure(tg)
    ch = ChannelSet()
    ch.commit.append(True)
    res = run_pass(sp, ch, VariableStore())
    assert res.committed and res.ops == 3 and res.stall_ms == 0.0
    # cancel while blocked on a CaseDecision
    tg2, sp2 = _fig4()
    ch2 = ChannelSet()
    ch2.cancel()
    vs = VariableStore()
    vs.overlay["w"] = Tensor.scalar(1.0)
    res = run_pass(sp2, ch2, vs)
    assert not res.committed
    rollback(vs)
    assert vs.overlay == {}


def test_variable_store_snapshot_rollback():
    vs = VariableStore()
    vs.committed["w"] = Tensor((2,), [0.0, 0.0])
    assert snapshot_vars(vs)["w"].to_nested() == [0.0, 0.0]
    vs.overlay["w"] = Tensor((2,), [1.0, 1.0])
    rollback(vs)
    rollback(vs)
    assert vs.read("w").to_nested() == [0.0, 0.0]
    vs.in_flight = True
    with pytest.raises(InFlightPass):
        snapshot_vars(vs)


def test_imperative_examples():
    res, _ = run("var w = fill([2], 0.0)\nsteps 2 { w = add(w, fill([2], 1.0)) }\n", "imperative")
    assert res.vars["w"].to_nested() == [2.0, 2.0]
    res, _ = run("steps 1 { print(1) }", "coexec")
    assert res.lines == ["1"]


def test_lazy_and_coexec_stats_shape():
    _, st = run(CORPUS["heavy_fetch"], "lazy")
    d = st.to_json()
    for k in ("python_exec_ms", "python_stall_ms", "graph_exec_ms", "graph_stall_ms", "phase_transitions",
              "traces_collected", "graph_regens", "steps_replayed", "throughput"):
        assert k in d


def test_dcgan_reaches_steady_coexec():
    """C2 alternates D / G steps through one SwitchCase: after both paths are traced
    every step runs co-executed (no divergence, no replay) -- ternary extension ops
    (batchnorm) must key identically in traced and skeleton steps."""
    from paper_2201_09210_b200.workloads import C2_SMALL, dcgan_program
    o = coexec.Orchestrator(lang.parse(dcgan_program(steps=12, **C2_SMALL)), SyntheticDataset(0),
                            coexec.Mode.coexec, coexec.RunConfig(), CpuBackend())
    o.run()
    assert o.stats.counters() == (1, 3, 1, 0)
