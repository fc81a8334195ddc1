"""Extension op set (configs C2-C5, SURVEY §2.4 / §8(a) row a*) through the C-ABI
against the builder's f64 restatement in oracle/kernels.py.

Tolerances (stated per precision; parity for these ops is unpinned by the reference):
* f64: convolutions and the piecewise-linear ops bit-exact (im2col + the sequential-k
  parity GEMM + ordered col2im); tanh / bce_term <= 4 ulp-ish (1e-14 relative);
  batch-norm family 1e-12 relative (parallel column reductions).
* fp32: 1e-5 relative, norm-wise.
* bf16: convolutions on tcgen05 with bf16 operands 2e-2 relative, norm-wise; the other
  ops run in fp32 (1e-5).
"""

import numpy as np
import pytest

from oracle.kernels import execute_kernel
from paper_2201_09210_b200.tensor import OpKind, Tensor

pytestmark = pytest.mark.gpu

RNG = np.random.default_rng(2201)


def rt(*shape, scale=1.0):
    return Tensor(shape, RNG.standard_normal(shape) * scale)


CONV = [
    (OpKind.CONV2D, {"conv": (4, 2, 1)}, [rt(2, 8, 8, 3), rt(48, 5)]),
    (OpKind.CONV2D, {"conv": (3, 1, 1)}, [rt(3, 5, 5, 7), rt(63, 16)]),
    (OpKind.CONV2D, {"conv": (3, 2, 0)}, [rt(2, 7, 7, 4), rt(36, 3)]),
    (OpKind.CONV2D, {"conv": (4, 2, 1)}, [rt(8, 16, 16, 64), rt(1024, 128)]),
    (OpKind.CONV2D, {"conv": (4, 2, 1)}, [rt(4, 8, 8, 256), rt(4096, 512)]),
    (OpKind.CONV2D_T, {"conv": (4, 2, 1)}, [rt(2, 4, 4, 8), rt(48, 8)]),
    (OpKind.CONV2D_T, {"conv": (3, 1, 1)}, [rt(2, 5, 5, 6), rt(36, 6)]),
    (OpKind.CONV2D_T, {"conv": (4, 2, 1)}, [rt(4, 8, 8, 64), rt(512, 64)]),
    (OpKind.CONV2D_T, {"conv": (4, 2, 1)}, [rt(8, 16, 16, 128), rt(48, 128)]),
    (OpKind.CONV2D_DW, {"conv": (4, 2, 1)}, [rt(2, 8, 8, 3), rt(2, 4, 4, 5)]),
    (OpKind.CONV2D_DW, {"conv": (3, 1, 1)}, [rt(3, 5, 5, 7), rt(3, 5, 5, 16)]),
    (OpKind.CONV2D_DW, {"conv": (4, 2, 1)}, [rt(8, 16, 16, 64), rt(8, 8, 8, 128)]),
    (OpKind.CONV2D_DW, {"conv": (4, 2, 1)}, [rt(16, 32, 32, 3), rt(16, 16, 16, 64)]),
    (OpKind.CONV2D_DW, {"conv": (4, 2, 1)}, [rt(2, 6, 6, 4), rt(2, 3, 3, 12)]),
    (OpKind.CONV2D, {"conv": (4, 2, 1)}, [rt(2, 6, 6, 4), rt(64, 12)]),
    (OpKind.CONV2D_T, {"conv": (4, 2, 1)}, [rt(2, 3, 3, 12), rt(64, 12)]),
    # implicit-GEMM paths (C % 64 == 0): pixel blocks spanning rows / images, padding taps
    (OpKind.CONV2D, {"conv": (4, 2, 1)}, [rt(16, 8, 8, 64), rt(1024, 32)]),
    (OpKind.CONV2D, {"conv": (3, 1, 1)}, [rt(2, 16, 16, 128), rt(1152, 64)]),
    (OpKind.CONV2D, {"conv": (4, 2, 1)}, [rt(2, 6, 6, 64), rt(1024, 16)]),
    (OpKind.CONV2D_T, {"conv": (4, 2, 1)}, [rt(16, 4, 4, 128), rt(1024, 128)]),
    (OpKind.CONV2D_T, {"conv": (4, 2, 1)}, [rt(2, 32, 32, 64), rt(48, 64)]),
    (OpKind.CONV2D_DW, {"conv": (4, 2, 1)}, [rt(16, 8, 8, 64), rt(16, 4, 4, 32)]),
    (OpKind.CONV2D_DW, {"conv": (3, 1, 1)}, [rt(2, 16, 16, 128), rt(2, 16, 16, 64)]),
]
# C3: conv2d's input gradient onto the forward geometry (strided shapes whose forward
# rounding leaves rows without a window: conv2d_t's size would differ) -- (dy, w, x)
def _dx_case(n, h, c, f, k, s, p):
    ho = (h + 2 * p - k) // s + 1
    return (OpKind.CONV2D_DX, {"conv": (k, s, p)}, [rt(n, ho, ho, f), rt(k * k * c, f), rt(n, h, h, c)])


CONV += [
    _dx_case(2, 8, 3, 5, 3, 2, 1),       # even input, 3x3/2: one row past conv2d_t's size
    _dx_case(2, 7, 4, 6, 3, 2, 1),       # odd input: exact conv2d_t geometry
    _dx_case(2, 8, 4, 6, 1, 2, 0),       # 1x1/2 projection shortcut
    _dx_case(2, 9, 3, 8, 7, 2, 3),       # 7x7/2 stem
    _dx_case(2, 8, 64, 64, 3, 1, 1),     # 3x3/1: sub-pixel implicit path (bf16)
    _dx_case(4, 14, 128, 64, 3, 2, 1),   # strided, explicit path
    _dx_case(2, 16, 64, 256, 1, 1, 0),   # 1x1/1 expansion
]
MATMUL_SPLIT = [  # bf16 MatMuls whose tile grid is too small: split-K slices
    (OpKind.MATMUL, {}, [rt(128, 8192), rt(8192, 1)]),
    (OpKind.MATMUL, {}, [rt(8192, 128), rt(128, 1)]),
    (OpKind.MATMUL, {}, [rt(100, 128), rt(128, 8192)]),
    (OpKind.MATMUL, {}, [rt(256, 4096), rt(4096, 96)]),
]

BN = [
    (OpKind.BATCHNORM, {}, [rt(4, 4, 4, 8, scale=3.0), rt(8), rt(8)]),
    (OpKind.BATCHNORM, {}, [rt(64, 300), rt(300), rt(300)]),
    (OpKind.BATCHNORM, {}, [rt(1000, 7), rt(7), rt(7)]),
    (OpKind.BATCHNORM, {}, [Tensor((2, 3, 3, 512), RNG.standard_normal((2, 3, 3, 512)) + 5.0), rt(512), rt(512)]),
    (OpKind.BATCHNORM_DX, {}, [rt(4, 4, 4, 8), rt(8), rt(4, 4, 4, 8)]),
    (OpKind.BATCHNORM_DX, {}, [rt(64, 300), rt(300), rt(64, 300)]),
    (OpKind.BATCHNORM_DX, {}, [rt(128, 16, 16, 64), rt(64), rt(128, 16, 16, 64)]),
    (OpKind.BN_DGAMMA, {}, [rt(4, 4, 4, 8), rt(4, 4, 4, 8)]),
    (OpKind.BN_DGAMMA, {}, [rt(1000, 7), rt(1000, 7)]),
    (OpKind.SUM_ROWS, {}, [rt(4, 4, 4, 8)]),
    (OpKind.SUM_ROWS, {}, [rt(3000, 513)]),
    (OpKind.SUM_ROWS, {}, [rt(5)]),
    (OpKind.SUM_ROWS, {}, [rt(8, 5000)]),        # wide rows: column-parallel kernel
    (OpKind.SUM_ROWS, {}, [rt(4096, 3072)]),     # wide rows, row chunks + fp64 atomics
]

POOL = [
    (OpKind.MAXPOOL, {"conv": (3, 2, 1)}, [rt(2, 9, 9, 5)]),
    (OpKind.MAXPOOL, {"conv": (3, 2, 1)}, [rt(4, 16, 16, 64)]),
    (OpKind.MAXPOOL, {"conv": (2, 2, 0)}, [Tensor((1, 4, 4, 2), np.repeat(np.arange(16.0), 2).reshape(1, 4, 4, 2) % 3)]),
    (OpKind.MAXPOOL_GRAD, {"conv": (3, 2, 1)}, [rt(2, 9, 9, 5), rt(2, 5, 5, 5)]),
    (OpKind.MAXPOOL_GRAD, {"conv": (3, 2, 1)}, [rt(4, 16, 16, 64), rt(4, 8, 8, 64)]),
    (OpKind.MAXPOOL_GRAD, {"conv": (2, 2, 0)},   # ties: the first maximum takes the gradient
     [Tensor((1, 4, 4, 2), np.repeat(np.arange(16.0), 2).reshape(1, 4, 4, 2) % 3), rt(1, 2, 2, 2)]),
    (OpKind.AVGPOOL, {"conv": (2, 2, 0)}, [rt(2, 7, 7, 6)]),
    (OpKind.AVGPOOL, {"conv": (3, 1, 1)}, [rt(2, 5, 5, 3)]),
    (OpKind.AVGPOOL_GRAD, {"conv": (2, 2, 0)}, [rt(2, 7, 7, 6), rt(2, 3, 3, 6)]),
    (OpKind.AVGPOOL_GRAD, {"conv": (3, 1, 1)}, [rt(2, 5, 5, 3), rt(2, 5, 5, 3)]),
    (OpKind.GLOBAL_AVGPOOL, {}, [rt(3, 7, 7, 33)]),
    (OpKind.GLOBAL_AVGPOOL_GRAD, {}, [rt(3, 7, 7, 33), rt(3, 33)]),
]

EDGE = np.array([-800.0, -30.0, -1.0, -0.0, 0.0, 1e-30, 0.5, 30.0, 800.0, np.nan])
EW = [
    (OpKind.TANH, {}, [Tensor(EDGE.shape, EDGE)]),
    (OpKind.TANH, {}, [rt(37, 41, scale=3.0)]),
    (OpKind.LEAKY_RELU, {}, [Tensor(EDGE.shape, EDGE)]),
    (OpKind.LEAKY_RELU, {}, [rt(1000)]),
    (OpKind.RELU_GRAD, {}, [Tensor(EDGE.shape, EDGE), rt(10)]),
    (OpKind.RELU_GRAD, {}, [rt(7, 9), rt()]),
    (OpKind.LEAKY_RELU_GRAD, {}, [Tensor(EDGE.shape, EDGE), rt(10)]),
    (OpKind.BCE_TERM, {}, [Tensor(EDGE.shape, EDGE), Tensor((), 1.0)]),
    (OpKind.BCE_TERM, {}, [rt(64, 1, scale=4.0), Tensor((), 0.0)]),
    (OpKind.SQRT, {}, [Tensor(EDGE.shape, EDGE)]),
    (OpKind.SQRT, {}, [Tensor((300,), np.abs(RNG.standard_normal(300)))]),
    (OpKind.DIV, {}, [Tensor(EDGE.shape, EDGE), Tensor((), 3.0)]),
    (OpKind.DIV, {}, [rt(37, 41), rt(37, 41)]),
]


def nrel(got, want):
    g, w = got.data.ravel(), want.data.ravel()
    ok = ~np.isnan(w)
    assert np.array_equal(np.isnan(g), np.isnan(w))
    den = np.linalg.norm(w[ok])
    return np.linalg.norm(g[ok] - w[ok]) / (den if den > 0 else 1.0)


def run(be, kind, attrs, ins):
    want = execute_kernel(kind, attrs, ins)[0]
    got = be.get(be.exec_op(kind, attrs, ins))
    assert got.shape == want.shape, (got.shape, want.shape)
    return got, want


@pytest.mark.parametrize("i", range(len(CONV)))
def test_conv_f64_bitwise(b200_factory, i):
    got, want = run(b200_factory("f64"), *CONV[i])
    assert got.data.tobytes() == want.data.tobytes(), np.max(np.abs(got.data - want.data))


@pytest.mark.parametrize("prec,tol", [("fp32", 1e-5), ("bf16", 2e-2)])
@pytest.mark.parametrize("i", range(len(CONV)))
def test_conv_tolerance(b200_factory, prec, tol, i):
    got, want = run(b200_factory(prec), *CONV[i])
    assert nrel(got, want) <= tol


@pytest.mark.parametrize("i", range(len(MATMUL_SPLIT)))
def test_matmul_bf16_split(b200_factory, i):
    got, want = run(b200_factory("bf16"), *MATMUL_SPLIT[i])
    assert nrel(got, want) <= 2e-2


@pytest.mark.parametrize("prec,tol", [("f64", 1e-12), ("fp32", 1e-5), ("bf16", 1e-5)])
@pytest.mark.parametrize("i", range(len(BN)))
def test_batchnorm_family(b200_factory, prec, tol, i):
    got, want = run(b200_factory(prec), *BN[i])
    assert nrel(got, want) <= tol


@pytest.mark.parametrize("prec,tol", [("f64", 1e-14), ("fp32", 1e-6), ("bf16", 1e-6)])
@pytest.mark.parametrize("i", range(len(EW)))
def test_elementwise_ext(b200_factory, prec, tol, i):
    kind, attrs, ins = EW[i]
    got, want = run(b200_factory(prec), kind, attrs, ins)
    if prec == "f64" and kind in (OpKind.LEAKY_RELU, OpKind.RELU_GRAD, OpKind.LEAKY_RELU_GRAD, OpKind.SQRT, OpKind.DIV):
        assert got.data.tobytes() == want.data.tobytes()
    else:
        assert nrel(got, want) <= tol


@pytest.mark.parametrize("prec,tol", [("f64", 0.0), ("fp32", 1e-6), ("bf16", 1e-6)])
@pytest.mark.parametrize("i", range(len(POOL)))
def test_pooling(b200_factory, prec, tol, i):
    """Pooling (C3): f64 bit-exact (same tap / window order as the oracle); fp32 storage
    (the bf16 mode stores activations in fp32) within 1e-6."""
    got, want = run(b200_factory(prec), *POOL[i])
    if prec == "f64":
        assert got.data.tobytes() == want.data.tobytes()
    else:
        assert nrel(got, want) <= tol


def test_bn_gradient_consistency(b200_factory):
    """batchnorm_dx / bn_dgamma / sum_rows are the gradients of sum(batchnorm(x,g,b) * dy)."""
    be = b200_factory("f64")
    x, g, b, dy = rt(6, 5, 4), rt(4), rt(4), rt(6, 5, 4)
    dx = be.get(be.exec_op(OpKind.BATCHNORM_DX, {}, [x, g, dy])).data
    dg = be.get(be.exec_op(OpKind.BN_DGAMMA, {}, [x, dy])).data
    db = be.get(be.exec_op(OpKind.SUM_ROWS, {}, [dy])).data

    def f(xx, gg, bb):
        y = be.get(be.exec_op(OpKind.BATCHNORM, {}, [Tensor(xx.shape, xx), Tensor(gg.shape, gg),
                                                     Tensor(bb.shape, bb)])).data
        return float(np.sum(y * dy.data))

    h = 1e-6
    for (arr, grad, which) in ((x.data, dx, 0), (g.data, dg, 1), (b.data, db, 2)):
        flat = arr.ravel()
        for j in (0, flat.size // 2, flat.size - 1):
            p, m = [x.data.copy(), g.data.copy(), b.data.copy()], [x.data.copy(), g.data.copy(), b.data.copy()]
            p[which].ravel()[j] += h
            m[which].ravel()[j] -= h
            num = (f(*p) - f(*m)) / (2 * h)
            assert abs(num - grad.ravel()[j]) <= 1e-6 * max(1.0, abs(num)), (which, j, num, grad.ravel()[j])
