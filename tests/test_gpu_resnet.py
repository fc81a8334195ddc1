"""Config C3 (ResNet-50 with SDPoint, BASELINE.json configs[2]) end to end on the B200 at
a reduced parity size (batch 8, 64x64 images, width 4, one bottleneck per stage, 10
classes): strided / 1x1 / 7x7 convolutions and their input gradients (conv2d_dx), max
pooling, projection shortcuts, global average pooling, and the SDPoint SwitchCase after
which the network runs at a path-dependent spatial size.  Against the CPU oracle (f64):
TraceGraph JSON, decision log and Stats counters bit-exact; printed losses within
tolerance; final variables norm-wise over all parameters together (the batch-norm offsets
are sums of near-cancelling gradients, see test_gpu_dcgan.py)."""

import math

import numpy as np
import pytest

from oracle.cpu_backend import CpuBackend
from paper_2201_09210_b200.trace_graph import to_json_text
from paper_2201_09210_b200.workloads import C3_SMALL, resnet_program
from test_gpu_coexec import run

pytestmark = pytest.mark.gpu

# lr 1e-3: the tiny network's training amplifies rounding differences ~10x per step at
# larger rates (tests/test_dp_gloo.py); f64 parity is stated at 1e-8 and fp32 at 1e-3 for
# the same reason (batch-norm over 8-32-row batches at 1x1 / 2x2 spatial size in the last
# stages amplifies operand rounding)
SRC = resnet_program(steps=14, lr=1e-3, **C3_SMALL)


@pytest.fixture(scope="module")
def oracle_run():
    return run(SRC, "coexec", CpuBackend())


@pytest.mark.parametrize("prec,tol", [("f64", 1e-8), ("fp32", 1e-3), ("bf16", 3e-2)])
@pytest.mark.parametrize("mode", ["coexec", "lazy"])
def test_resnet_sdpoint_parity(b200_factory, oracle_run, prec, tol, mode):
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
