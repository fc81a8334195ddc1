"""tcgen05 bf16 GEMM (bf16 precision mode) against the float64 oracle.

Contract (BASELINE.json north_star): any bf16 tensor-core path agrees within 2e-2
relative.  A tighter check against the product of the bf16-rounded operands
(1e-3) catches layout / descriptor bugs that a loose tolerance could hide."""

import numpy as np
import pytest

from oracle.kernels import execute_kernel
from paper_2201_09210_b200.tensor import OpKind, Tensor

pytestmark = pytest.mark.gpu


def bf16_round(x):
    b = np.asarray(x, dtype=np.float32).view(np.uint32).astype(np.uint64)
    r = ((b + 0x7FFF + ((b >> 16) & 1)) >> 16) << 16
    return r.astype(np.uint32).view(np.float32).astype(np.float64)


@pytest.mark.parametrize("m,k,n", [(128, 64, 128), (64, 784, 128), (1, 1, 1), (130, 70, 250),
                                   (1000, 300, 700), (256, 4096, 384), (784, 64, 128), (3, 0, 5)])
def test_bf16_gemm(b200_factory, m, k, n):
    be = b200_factory("bf16")
    r = np.random.default_rng(m * 7 + k * 13 + n)
    a = Tensor((m, k), r.uniform(-1, 1, (m, k)))
    b = Tensor((k, n), r.uniform(-1, 1, (k, n)))
    got = be.get(be.exec_op(OpKind.MATMUL, {}, [a, b])).data
    want = execute_kernel(OpKind.MATMUL, {}, [a, b])[0].data
    assert got.shape == (m, n)
    if k == 0:
        assert not got.any()
        return
    tight = bf16_round(a.data) @ bf16_round(b.data)
    err_tight = np.linalg.norm(got - tight) / max(np.linalg.norm(tight), 1e-30)
    err = np.linalg.norm(got - want) / max(np.linalg.norm(want), 1e-30)
    assert err_tight <= 1e-3, err_tight
    assert err <= 2e-2, err


def test_bf16_gemm_transposed_operands(b200_factory):
    from paper_2201_09210_b200 import coexec, lang
    from paper_2201_09210_b200.dataset import SyntheticDataset
    from oracle.cpu_backend import CpuBackend
    src = """
var w = input("w", [96, 40])
steps 5 {
  let x = input("x", [200, 96])
  let h = matmul(x, w)
  let g = matmul(transpose(x), h)
  let z = matmul(h, transpose(w))
  w = sub(w, mul(g, 0.0001))
  print(mean(mul(h, h)))
  print(mean(mul(z, z)))
}
"""
    res = {}
    for name, be in (("ref", CpuBackend()), ("bf16", b200_factory("bf16", fresh=True))):
        res[name] = coexec.run(lang.parse(src), SyntheticDataset(0), "coexec", backend=be)[0]
    for a, b in zip(res["ref"].lines, res["bf16"].lines):
        assert abs(float(a) - float(b)) <= 2e-2 * abs(float(a)), (a, b)
    w0, w1 = res["ref"].vars["w"].data, res["bf16"].vars["w"].data
    assert np.linalg.norm(w1 - w0) / np.linalg.norm(w0) <= 2e-2
