"""Config C5 (Music Transformer, BASELINE.json configs[4]) end to end on the B200 at a
reduced parity size (2 layers, d=32, 2 heads, T=16, vocab 29): relative attention with the
skew (rel_skew / rel_unskew), an untied output head, and the config's generator and
try/except control flow simulated with natives (a host-drawn ``while`` trip count and a
``native coin`` SwitchCase whose arms differ in which variables they assign).  Against the
CPU oracle (f64): TraceGraph JSON, decision log and Stats counters bit-exact; printed
losses within tolerance; final variables within tolerance norm-wise over all parameters
together (see test_gpu_gpt2.py for why not per variable)."""

import math

import numpy as np
import pytest

from oracle.cpu_backend import CpuBackend
from paper_2201_09210_b200.trace_graph import to_json_text
from paper_2201_09210_b200.workloads import C5_SMALL, music_transformer_program
from test_gpu_coexec import run

pytestmark = pytest.mark.gpu

SRC = music_transformer_program(steps=6, **C5_SMALL)


@pytest.fixture(scope="module")
def oracle_run():
    return run(SRC, "coexec", CpuBackend())


@pytest.mark.parametrize("prec,tol", [("f64", 1e-10), ("fp32", 1e-4), ("bf16", 3e-2)])
@pytest.mark.parametrize("mode", ["coexec", "lazy"])
def test_music_transformer_parity(b200_factory, oracle_run, prec, tol, mode):
    ref, ref_st, ref_o = oracle_run
    be = b200_factory(prec, fresh=True)
    try:
        got, st, o = run(SRC, mode, be)
    finally:
        be.close()
    if mode == "coexec":
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
