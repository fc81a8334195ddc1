"""Transformer extension op set (config C4, GPT-2 small; SURVEY §2.4 / §8(a) row a*)
through the C-ABI against the f64 restatement in oracle/kernels.py.

Tolerances: f64 <= 1e-12 relative norm-wise (parallel row / column reductions, CUDA
transcendental functions; the batched MatMuls use the sequential-k parity kernel and are
bit-exact); fp32 <= 1e-5; bf16 mode: batched GEMMs on tcgen05 with bf16 operands <= 2e-2,
everything else runs in fp32 (<= 1e-5)."""

import numpy as np
import pytest

from oracle.kernels import execute_kernel
from paper_2201_09210_b200.tensor import OpKind, Tensor

pytestmark = pytest.mark.gpu

RNG = np.random.default_rng(2026)


def rt(*shape, scale=1.0):
    return Tensor(shape, RNG.standard_normal(shape) * scale)


def ids(shape, v):
    return Tensor(shape, RNG.integers(0, v, shape).astype(np.float64))


BMM = [
    (OpKind.BMM, {}, [rt(3, 17, 9), rt(3, 9, 5)]),
    (OpKind.BMM_NT, {}, [rt(3, 17, 9), rt(3, 5, 9)]),
    (OpKind.BMM_TN, {}, [rt(3, 9, 17), rt(3, 9, 5)]),
    (OpKind.BMM_NT, {}, [rt(8, 256, 64), rt(8, 256, 64)]),
    (OpKind.BMM, {}, [rt(8, 256, 256), rt(8, 256, 64)]),
    (OpKind.BMM_TN, {}, [rt(8, 256, 256), rt(8, 256, 64)]),
    (OpKind.BMM_TN, {}, [rt(4, 128, 200), rt(4, 128, 72)]),
]

ROWS = [
    (OpKind.EMBEDDING, {}, [rt(50, 24), ids((4, 7), 50)]),
    (OpKind.EMBEDDING_DW, {"dims": (50,)}, [ids((4, 7), 50), rt(4, 7, 24)]),
    (OpKind.EMBEDDING_DW, {"dims": (11,)}, [ids((300,), 11), rt(300, 64)]),
    (OpKind.LAYERNORM, {}, [rt(33, 70, scale=2.0), rt(70), rt(70)]),
    (OpKind.LAYERNORM, {}, [Tensor((16, 768), RNG.standard_normal((16, 768)) + 3.0), rt(768), rt(768)]),
    (OpKind.LAYERNORM_DX, {}, [rt(33, 70), rt(70), rt(33, 70)]),
    (OpKind.LN_DGAMMA, {}, [rt(33, 70), rt(33, 70)]),
    (OpKind.LN_DGAMMA, {}, [rt(2000, 768), rt(2000, 768)]),
    (OpKind.BIAS_ADD, {}, [rt(6, 5, 12), rt(12)]),
    (OpKind.BIAS_ADD, {}, [rt(9, 7), rt(7)]),
    (OpKind.CAUSAL_SOFTMAX, {"value": 0.125}, [rt(2, 3, 40, 40, scale=4.0)]),
    (OpKind.CAUSAL_SOFTMAX, {"value": 1.0}, [rt(1, 1, 1)]),
    (OpKind.SOFTMAX_GRAD, {"value": 0.125}, [rt(4, 40, 40), rt(4, 40, 40)]),
    (OpKind.CROSS_ENTROPY, {}, [rt(37, 101, scale=3.0), ids((37,), 101)]),
    (OpKind.CROSS_ENTROPY_GRAD, {}, [rt(37, 101, scale=3.0), ids((37,), 101)]),
    (OpKind.CROSS_ENTROPY, {}, [rt(4, 5000), ids((4,), 5000)]),
    (OpKind.GELU, {}, [rt(1000, scale=3.0)]),
    (OpKind.GELU_GRAD, {}, [rt(50, 3), rt(50, 3)]),
    (OpKind.TO_INDEX, {}, [Tensor((6,), [-1.0, -0.5, 0.0, 0.3, 0.999999, 1.5]), Tensor((), 97.0)]),
    # relative attention (C5): shifted copies, bit-exact in every precision
    (OpKind.REL_SKEW, {}, [rt(3, 37, 37)]),
    (OpKind.REL_SKEW, {}, [rt(1, 1)]),
    (OpKind.REL_UNSKEW, {}, [rt(2, 2, 64, 64)]),
    (OpKind.REL_UNSKEW, {}, [rt(4, 100, 100)]),
    # general axis ops: bit-exact in every precision except sum_axis (fp32 accumulation)
    (OpKind.SLICE, {"dims": (1, 3, 17)}, [rt(4, 30, 7)]),
    (OpKind.SLICE, {"dims": (0, 2, 3)}, [rt(9, 5)]),
    (OpKind.CONCAT, {"dims": (1,)}, [rt(4, 30, 7), rt(4, 2, 7)]),
    (OpKind.CONCAT, {"dims": (2,)}, [rt(3, 5, 64), rt(3, 5, 64)]),
    (OpKind.SUM_AXIS, {"dims": (1,)}, [rt(6, 300, 33)]),
    (OpKind.SUM_AXIS, {"dims": (0,)}, [rt(1000, 17)]),
]


def nrel(got, want):
    g, w = got.data.ravel(), want.data.ravel()
    den = np.linalg.norm(w)
    return np.linalg.norm(g - w) / (den if den > 0 else 1.0)


def run(be, kind, attrs, ins):
    want = execute_kernel(kind, attrs, ins)[0]
    got = be.get(be.exec_op(kind, attrs, ins))
    assert got.shape == want.shape, (got.shape, want.shape)
    return got, want


@pytest.mark.parametrize("i", range(len(BMM)))
def test_bmm_f64_bitwise(b200_factory, i):
    got, want = run(b200_factory("f64"), *BMM[i])
    assert got.data.tobytes() == want.data.tobytes()


@pytest.mark.parametrize("prec,tol", [("fp32", 1e-5), ("bf16", 2e-2)])
@pytest.mark.parametrize("i", range(len(BMM)))
def test_bmm_tolerance(b200_factory, prec, tol, i):
    got, want = run(b200_factory(prec), *BMM[i])
    assert nrel(got, want) <= tol


@pytest.mark.parametrize("prec,tol", [("f64", 1e-12), ("fp32", 1e-5), ("bf16", 1e-5)])
@pytest.mark.parametrize("i", range(len(ROWS)))
def test_row_ops(b200_factory, prec, tol, i):
    kind, attrs, ins = ROWS[i]
    got, want = run(b200_factory(prec), kind, attrs, ins)
    if kind is OpKind.TO_INDEX or (kind in (OpKind.EMBEDDING, OpKind.REL_SKEW, OpKind.REL_UNSKEW, OpKind.SLICE,
                                            OpKind.CONCAT, OpKind.SUM_AXIS) and prec == "f64"):
        assert got.data.tobytes() == want.data.tobytes()
    else:
        assert nrel(got, want) <= tol
