"""fp32-mode MatMul as 3xTF32 on the tcgen05 tensor cores (csrc/gemm_tf32.cuh, COEX_TF32=1)
against the float64 oracle (oracle.kernels.execute_kernel <- tensor.py:228-236).

A single TF32 product would miss the fp32 bar (~5e-4); the hi / lo split brings a single op
to the tensor core's fp32-accumulation floor (~2e-6, measured), checked here per op against
1e-5 (norm-wise and element-wise against the operand scale) over aligned and ragged shapes,
split-K launches, folded transposes and a co-executed program.  The fp32 mode's default stays
the SIMT kernel: end to end, that floor exceeds the contract's 1e-5 gradient bar."""

import numpy as np
import pytest

from oracle.kernels import execute_kernel
from paper_2201_09210_b200.tensor import OpKind, Tensor

pytestmark = pytest.mark.gpu


@pytest.fixture(autouse=True)
def _tf32(monkeypatch):
    monkeypatch.setenv("COEX_TF32", "1")


@pytest.mark.parametrize("m,k,n", [(128, 64, 128), (64, 784, 128), (1, 1, 1), (130, 70, 250), (1000, 300, 700),
                                   (256, 4096, 384), (784, 64, 128), (3, 0, 5), (8192, 768, 64), (33, 5000, 65)])
def test_tf32x3_gemm(b200_factory, m, k, n):
    be = b200_factory("fp32")
    r = np.random.default_rng(m * 7 + k * 13 + n)
    a = Tensor((m, k), r.uniform(-1, 1, (m, k)))
    b = Tensor((k, n), r.uniform(-1, 1, (k, n)))
    got = be.get(be.exec_op(OpKind.MATMUL, {}, [a, b])).data
    want = execute_kernel(OpKind.MATMUL, {}, [a, b])[0].data
    assert got.shape == (m, n)
    if k == 0:
        assert not got.any()
        return
    err = np.linalg.norm(got - want) / max(np.linalg.norm(want), 1e-30)
    # element-wise against the dot products' own scale (|a| . |b|): a wrong tile shows here
    scale = np.abs(a.data) @ np.abs(b.data)
    elem = float(np.max(np.abs(got - want) / np.maximum(scale, 1e-30)))
    assert err <= 1e-5, err
    assert elem <= 1e-5, elem


def test_tf32x3_kernels_launched(b200_factory):
    """the fp32 MatMul is the tensor-core path (hi / lo split + k_gemm_tf32), not SIMT"""
    be = b200_factory("fp32", fresh=True)
    r = np.random.default_rng(3)
    a = Tensor((256, 512), r.uniform(-1, 1, (256, 512)))
    b = Tensor((512, 256), r.uniform(-1, 1, (512, 256)))
    prof = be.profile_op(OpKind.MATMUL, {}, [a, b], reps=2)
    names = [n for n, _ in prof]
    assert any("k_cvt_tf32" in n for n in names) and any("k_gemm_tf32" in n for n in names), names


def test_tf32x3_transposed_operands(b200_factory):
    """folded transposes (A stored [K][M], B stored [N][K]) through a co-executed program"""
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
    for name, be in (("ref", CpuBackend()), ("fp32", b200_factory("fp32", fresh=True))):
        res[name] = coexec.run(lang.parse(src), SyntheticDataset(0), "coexec", backend=be)[0]
    for a, b in zip(res["ref"].lines, res["fp32"].lines):
        assert abs(float(a) - float(b)) <= 1e-5 * abs(float(a)), (a, b)
    w0, w1 = res["ref"].vars["w"].data, res["fp32"].vars["w"].data
    assert np.linalg.norm(w1 - w0) / np.linalg.norm(w0) <= 1e-5
