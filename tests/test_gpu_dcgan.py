"""Config C2 (DCGAN, BASELINE.json configs[1]) end to end on the B200 at a reduced
parity size: the discriminator/generator alternation is a SwitchCase on
``native mod(step, 2)`` whose two bodies are the two backward passes.  Against the
CPU oracle (oracle/, f64): TraceGraph JSON, decision log and Stats counters
bit-exact; printed losses within the precision's tolerance; final variables within
it norm-wise (f64 / fp32: per variable; bf16: over all variables together -- the
batch-norm offsets are sums of near-cancelling gradients whose own relative error
is not meaningful at bf16 operand precision)."""

import math

import numpy as np
import pytest

from oracle.cpu_backend import CpuBackend
from paper_2201_09210_b200.trace_graph import to_json_text
from paper_2201_09210_b200.workloads import C2_SMALL, dcgan_program
from test_gpu_coexec import assert_close, run

pytestmark = pytest.mark.gpu

SRC = dcgan_program(steps=6, **C2_SMALL)
# a second shape: 32x32 images (3 up / 3 down layers), odd batch
SRC32 = dcgan_program(steps=4, batch=3, nz=5, ngf=4, ndf=4, img=32)


@pytest.fixture(scope="module")
def oracle_runs():
    return {k: run(src, mode, CpuBackend()) for k, src in (("16", SRC), ("32", SRC32))
            for mode in ("coexec",)}


@pytest.mark.parametrize("prec,tol", [("f64", 1e-10), ("fp32", 1e-4), ("bf16", 3e-2)])
@pytest.mark.parametrize("which", ["16", "32"])
@pytest.mark.parametrize("mode", ["coexec", "lazy"])
def test_dcgan_parity(b200_factory, oracle_runs, prec, tol, which, mode):
    ref, ref_st, ref_o = oracle_runs[which]
    be = b200_factory(prec, fresh=True)
    try:
        got, st, o = run(SRC if which == "16" else SRC32, mode, be)
        launched = be.kernel_count()
    finally:
        be.close()
    assert launched > 0
    assert st.counters() == ref_st.counters()
    assert st.decision_log == ref_st.decision_log
    assert to_json_text(o.tg) == to_json_text(ref_o.tg)
    if prec != "bf16":
        assert_close(ref, got, tol, False)
        return
    assert len(ref.lines) == len(got.lines)
    for a, b in zip(ref.lines, got.lines):
        assert math.isclose(float(a), float(b), rel_tol=tol), (a, b)
    keys = sorted(ref.vars)
    w = np.concatenate([ref.vars[k].data.ravel() for k in keys])
    g = np.concatenate([got.vars[k].data.ravel() for k in keys])
    assert np.linalg.norm(g - w) / np.linalg.norm(w) <= 2e-2


def test_dcgan_imperative_f64(b200_factory):
    ref, _, _ = run(SRC, "imperative", CpuBackend())
    be = b200_factory("f64", fresh=True)
    try:
        got, _, _ = run(SRC, "imperative", be)
    finally:
        be.close()
    assert_close(ref, got, 1e-10, False)
