"""End-to-end parity on the B200: every corpus program and 200 fuzzed programs run
in imperative / coexec / lazy / skeleton-check modes on the device and must equal
the CPU oracle's imperative run: printed lines and final variables bit-exact
(f64 parity mode, programs without sigmoid), or within the stated tolerance;
TraceGraph and Stats counters identical."""

import math

import numpy as np
import pytest

from oracle.cpu_backend import CpuBackend
from paper_2201_09210_b200 import coexec, lang
from paper_2201_09210_b200.dataset import SyntheticDataset
from paper_2201_09210_b200.trace_graph import to_json_text
from programs import CORPUS, fuzz_program

pytestmark = pytest.mark.gpu

MODES = ["imperative", "coexec", "lazy", "skeleton-check"]


def run(src, mode, be):
    orch = coexec.Orchestrator(lang.parse(src), SyntheticDataset(0), coexec.Mode(mode), coexec.RunConfig(), be)
    res, st = orch.run()
    return res, st, orch


def _nums(line):
    return [float(t) for t in line.replace("[", " ").replace("]", " ").replace(",", " ").split()
            if t not in ("true", "false")]


def assert_close(ref, got, rtol, exact):
    assert len(ref.lines) == len(got.lines)
    for a, b in zip(ref.lines, got.lines):
        if exact:
            assert a == b
        else:
            x, y = _nums(a), _nums(b)
            assert len(x) == len(y)
            for u, v in zip(x, y):
                assert math.isclose(u, v, rel_tol=rtol, abs_tol=rtol), (a, b)
    for k, t in ref.vars.items():
        g = got.vars[k]
        assert g.shape == t.shape
        if exact:
            assert g.data.tobytes() == t.data.tobytes(), k
        else:
            err = np.linalg.norm(g.data - t.data) / max(np.linalg.norm(t.data), 1e-30)
            assert err <= rtol, (k, err)


@pytest.mark.parametrize("name", sorted(CORPUS))
@pytest.mark.parametrize("mode", MODES)
def test_corpus_f64(b200_factory, name, mode):
    src = CORPUS[name]
    ref, ref_st, ref_o = run(src, "coexec" if mode != "imperative" else "imperative", CpuBackend())
    be = b200_factory("f64", fresh=True)
    try:
        got, st, o = run(src, mode, be)
    finally:
        be.close()
    exact = "sigmoid" not in src
    assert_close(ref, got, 1e-12, exact)
    if mode != "imperative":
        assert st.counters() == ref_st.counters()
        assert to_json_text(o.tg) == to_json_text(ref_o.tg)
        assert st.decision_log == ref_st.decision_log


@pytest.mark.parametrize("name", ["fig3", "straight", "branchy", "c1_small", "var_trip"])
def test_corpus_fp32(b200_factory, name):
    src = CORPUS[name]
    ref, ref_st, _ = run(src, "coexec", CpuBackend())
    be = b200_factory("fp32", fresh=True)
    try:
        got, st, _ = run(src, "coexec", be)
    finally:
        be.close()
    assert_close(ref, got, 1e-5, False)
    assert st.counters() == ref_st.counters()


def test_fuzz_200_coexec(b200_factory):
    be = b200_factory("f64", fresh=True)
    bad = []
    try:
        for seed in range(200):
            src = fuzz_program(seed)
            ref, ref_st, _ = run(src, "imperative", CpuBackend())
            be2 = b200_factory("f64", fresh=True)
            try:
                got, st, _ = run(src, "coexec", be2)
            finally:
                be2.close()
            try:
                assert_close(ref, got, 1e-12, "sigmoid" not in src)
            except AssertionError as e:
                bad.append((seed, str(e)[:200]))
    finally:
        be.close()
    assert not bad, bad[:5]


@pytest.mark.parametrize("prec", ["f64", "bf16"])
def test_pinned_host_feeds_read_in_place(b200_factory, prec):
    """Host-resident inputs registered with B200Backend.pin are fed with
    coex_pass_feed_mapped (the feed kernel reads them across the bus, no staging copy):
    the run equals the staged-copy run bit for bit."""
    from paper_2201_09210_b200.tensor import Tensor
    from paper_2201_09210_b200.workloads import InMemoryDataset, c1_program
    src = c1_program(steps=8, batch=8, hidden=16, din=12, dout=3)
    r = np.random.default_rng(3)
    recs = {"x": [Tensor((8, 12), r.uniform(-1, 1, (8, 12))) for _ in range(3)],
            "y": [Tensor((8, 3), r.uniform(-1, 1, (8, 3))) for _ in range(3)],
            "w1_init": [Tensor((12, 16), r.uniform(-1, 1, (12, 16)))],
            "w2_init": [Tensor((16, 3), r.uniform(-1, 1, (16, 3)))]}
    outs = []
    for pinned in (False, True):
        be = b200_factory(prec, fresh=True)
        try:
            if pinned:
                for k in ("x", "y"):
                    for t in recs[k]:
                        be.pin(t.data)
                assert be.is_pinned(recs["x"][0].data)
            orch = coexec.Orchestrator(lang.parse(src), InMemoryDataset(recs), coexec.Mode.coexec,
                                       coexec.RunConfig(), be)
            res, st = orch.run()
            outs.append((res.lines, {k: v.data.tobytes() for k, v in res.vars.items()}, st.counters()))
        finally:
            be.close()
    assert outs[0] == outs[1]
    assert outs[1][2][1] >= 1                                 # graph passes ran
