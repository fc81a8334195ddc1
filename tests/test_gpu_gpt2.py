"""Config C4 (GPT-2, BASELINE.json configs[3]) end to end on the B200 at a reduced parity
size (2 layers, d=64, 4 heads, T=32, vocab 97): embeddings, pre-LN causal attention
blocks, tied LM head, cross-entropy, the hand-written backward pass, and a data-dependent
``while`` over the fetched loss.  Against the CPU oracle (f64): TraceGraph JSON, decision
log and Stats counters bit-exact; printed losses within tolerance; final variables within
tolerance norm-wise over all parameters together (the key-projection bias gradient is
exactly zero in exact arithmetic -- softmax is shift-invariant per row -- so that variable
holds only rounding noise and has no meaningful relative error of its own)."""

import math

import numpy as np
import pytest

from oracle.cpu_backend import CpuBackend
from paper_2201_09210_b200.trace_graph import to_json_text
from paper_2201_09210_b200.workloads import C4_SMALL, gpt2_program
from test_gpu_coexec import run

pytestmark = pytest.mark.gpu

SRC = gpt2_program(steps=5, **C4_SMALL)
SRC_ADAM = gpt2_program(steps=5, optimizer="adam", **C4_SMALL)


@pytest.fixture(scope="module")
def oracle_run():
    return run(SRC, "coexec", CpuBackend())


@pytest.mark.parametrize("prec,tol", [("f64", 1e-10), ("fp32", 1e-4), ("bf16", 3e-2)])
def test_gpt2_parity(b200_factory, oracle_run, prec, tol):
    ref, ref_st, ref_o = oracle_run
    be = b200_factory(prec, fresh=True)
    try:
        got, st, o = run(SRC, "coexec", be)
    finally:
        be.close()
    assert st.counters() == ref_st.counters()
    assert st.decision_log == ref_st.decision_log
    assert to_json_text(o.tg) == to_json_text(ref_o.tg)
    assert len(ref.lines) == len(got.lines)
    for a, b in zip(ref.lines, got.lines):
        assert math.isclose(float(a), float(b), rel_tol=tol), (a, b)
    keys = sorted(ref.vars)
    w = np.concatenate([ref.vars[k].data.ravel() for k in keys])
    g = np.concatenate([got.vars[k].data.ravel() for k in keys])
    assert np.linalg.norm(g - w) / np.linalg.norm(w) <= min(tol, 2e-2)


@pytest.mark.parametrize("prec,tol", [("f64", 1e-10), ("bf16", 3e-2)])
def test_gpt2_adam_parity(b200_factory, prec, tol):
    """The Adam rewrite (sqrt / div elementwise, fused into chains) against the oracle."""
    ref, ref_st, _ = run(SRC_ADAM, "coexec", CpuBackend())
    be = b200_factory(prec, fresh=True)
    try:
        got, st, _ = run(SRC_ADAM, "coexec", be)
    finally:
        be.close()
    assert st.counters() == ref_st.counters()
    for a, b in zip(ref.lines, got.lines):
        assert math.isclose(float(a), float(b), rel_tol=tol), (a, b)
    keys = sorted(ref.vars)
    w = np.concatenate([ref.vars[k].data.ravel() for k in keys])
    g = np.concatenate([got.vars[k].data.ravel() for k in keys])
    assert np.linalg.norm(g - w) / np.linalg.norm(w) <= min(tol, 2e-2)
