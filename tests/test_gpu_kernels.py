"""Kernel parity through the C-ABI (coex_exec_op) against the CPU oracle
(oracle/kernels.py, itself pinned to the reference by tests/golden)."""

import numpy as np
import pytest

from oracle.kernels import execute_kernel
from paper_2201_09210_b200.dataset import SyntheticTensor, synth_values
from paper_2201_09210_b200.tensor import OpKind, Tensor

pytestmark = pytest.mark.gpu

RNG = np.random.default_rng(1234)


def rt(*shape, scale=1.0):
    return Tensor(shape, RNG.standard_normal(shape) * scale)


CASES = [
    (OpKind.ADD, {}, [rt(5, 7), rt(5, 7)]),
    (OpKind.ADD, {}, [rt(5, 7), rt()]),
    (OpKind.ADD, {}, [rt(), rt(4)]),
    (OpKind.SUB, {}, [rt(3, 1000), rt(3, 1000)]),
    (OpKind.MUL, {}, [rt(257), rt()]),
    (OpKind.NEG, {}, [rt(9, 9)]),
    (OpKind.RELU, {}, [Tensor((6,), [-1.0, -0.0, 0.0, 2.5, float("nan"), -3.0])]),
    (OpKind.SUM, {}, [rt(64, 10)]),
    (OpKind.SUM, {}, [rt(1000, 1000)]),
    (OpKind.SUM, {}, [rt(2048, 2049)]),          # tolerance modes: multi-block k_reduce_multi
    (OpKind.MEAN, {}, [rt(3, 1 << 20)]),
    (OpKind.SUM, {}, [Tensor((3,), [-0.0, -0.0, -0.0])]),
    (OpKind.SUM, {}, [Tensor((0,), [])]),
    (OpKind.MEAN, {}, [rt(33, 17)]),
    (OpKind.MATMUL, {}, [rt(2, 2), Tensor((2, 2), [[1.0, 0.0], [0.0, 1.0]])]),
    (OpKind.MATMUL, {}, [rt(64, 784), rt(784, 128)]),
    (OpKind.MATMUL, {}, [rt(128, 64), rt(64, 10)]),
    (OpKind.MATMUL, {}, [rt(513, 300), rt(300, 1025)]),
    (OpKind.MATMUL, {}, [rt(3, 0), rt(0, 4)]),
    (OpKind.MATMUL, {}, [Tensor((1, 2), [[-0.0, 1.0]]), Tensor((2, 1), [[5.0], [-0.0]])]),
    (OpKind.TRANSPOSE, {"perm": (1, 0)}, [rt(64, 784)]),
    (OpKind.TRANSPOSE, {"perm": (2, 0, 1)}, [rt(3, 4, 5)]),
    (OpKind.TRANSPOSE, {"perm": ()}, [rt()]),
    (OpKind.RESHAPE, {"target_shape": (10, 3)}, [rt(5, 6)]),
    (OpKind.FILL, {"shape": (4, 5), "value": 0.05}, []),
    (OpKind.FILL, {"shape": (), "value": -2.0}, []),
]


@pytest.mark.parametrize("i", range(len(CASES)))
def test_f64_bitwise(b200_factory, i):
    be = b200_factory("f64")
    kind, attrs, ins = CASES[i]
    want = execute_kernel(kind, attrs, ins)[0]
    got = be.get(be.exec_op(kind, attrs, ins))
    assert got.shape == want.shape
    assert got.data.tobytes() == want.data.tobytes(), (kind, np.max(np.abs(got.data - want.data)))


def test_sigmoid_f64_ulps(b200_factory):
    be = b200_factory("f64")
    x = Tensor((4096,), np.concatenate([RNG.standard_normal(4000) * 10, [800.0, -800.0, 0.0, -0.0],
                                         np.linspace(-40, 40, 92)]))
    want = execute_kernel(OpKind.SIGMOID, {}, [x])[0].data
    got = be.get(be.exec_op(OpKind.SIGMOID, {}, [x])).data
    ulp = np.abs(got.view(np.int64) - want.view(np.int64))
    assert ulp.max() <= 4, ulp.max()


@pytest.mark.parametrize("i", range(len(CASES)))
def test_fp32_tolerance(b200_factory, i):
    be = b200_factory("fp32")
    kind, attrs, ins = CASES[i]
    want = execute_kernel(kind, attrs, ins)[0].data
    got = be.get(be.exec_op(kind, attrs, ins)).data
    assert got.shape == want.shape
    if want.size == 0:
        return
    nan = np.isnan(want)
    assert np.array_equal(nan, np.isnan(got))
    err = np.linalg.norm(got[~nan] - want[~nan]) / max(np.linalg.norm(want[~nan]), 1e-30)
    assert err <= 1e-5, err


@pytest.mark.parametrize("shape", [(4,), (64, 784), (3, 5, 7), (100003,)])
def test_device_synthetic_dataset_bitwise(b200_factory, shape):
    be = b200_factory("f64")
    st = SyntheticTensor(0x1234_5678_9ABC_DEF1, shape)
    got = be.get(be.put(st)).data
    want = synth_values(st.state, st.size()).reshape(shape)
    assert got.tobytes() == want.tobytes()


def test_var_store_roundtrip(b200_factory):
    be = b200_factory("f64", fresh=True)
    be.var_define("w", Tensor((2,), [0.0, 0.0]))
    one = be.put(Tensor((2,), [1.0, 1.0]))
    for _ in range(2):
        be.var_assign("w", be.exec_op(OpKind.ADD, {}, [be.var_read("w"), one]))
    assert be.snapshot_vars()["w"].to_nested() == [2.0, 2.0]
    be.close()
