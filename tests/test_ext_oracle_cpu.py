"""CPU checks of the builder-defined extension ops (SURVEY §8(a) row a*, parity unpinned
by the reference) that the GPU parity tests rely on: the f64 restatements in
oracle/kernels.py against torch autograd, and config C5 (Music Transformer) through the
co-execution engine on the CPU backend."""

import numpy as np
import pytest
import torch

from oracle.cpu_backend import CpuBackend
from oracle.kernels import execute_kernel
from paper_2201_09210_b200.tensor import OpKind, Tensor
from paper_2201_09210_b200.workloads import (C3_SMALL, C4_SMALL, C5_SMALL, gpt2_program, music_transformer_program,
                                             resnet_program)
from test_gpu_coexec import run

RNG = np.random.default_rng(5)


def k(kind, *xs, **attrs):
    return execute_kernel(kind, attrs, [Tensor(x.shape, x) for x in xs])[0].data


def t_skew(x):
    t = x.shape[-1]
    i = torch.arange(t).view(t, 1)
    j = torch.arange(t).view(1, t)
    idx = (t - 1 - i + j).clamp(max=t - 1).expand(*x.shape)
    return torch.where(j <= i, torch.gather(x, -1, idx), torch.zeros((), dtype=x.dtype))


@pytest.mark.parametrize("t", [1, 2, 7, 33])
def test_rel_skew_matches_definition_and_adjoint(t):
    x = RNG.standard_normal((3, t, t))
    dy = RNG.standard_normal((3, t, t))
    y = k(OpKind.REL_SKEW, x)
    assert np.array_equal(y, t_skew(torch.from_numpy(x)).numpy())
    for i in range(t):                       # column j of row i holds relative distance j - i
        for j in range(t):
            assert y[1, i, j] == (x[1, i, t - 1 - i + j] if j <= i else 0.0)
    dx = k(OpKind.REL_UNSKEW, dy)
    assert abs(np.sum(y * dy) - np.sum(x * dx)) <= 1e-12 * np.sum(np.abs(x * dx))


def test_relative_attention_backward_formulas():
    """The C5 program's hand-written attention backward (workloads._decoder_program, music)
    equals torch autograd of softmax(sc * (q.k^T + skew(q.er^T))) . v."""
    bh, t, hd = 3, 9, 4
    sc = 0.5
    q, kk, v = (RNG.standard_normal((bh, t, hd)) for _ in range(3))
    er = RNG.standard_normal((t, hd))
    g = RNG.standard_normal((bh, t, hd))
    # oracle restatement, in the program's order
    qe = k(OpKind.MATMUL, q.reshape(bh * t, hd), er.T.copy()).reshape(bh, t, t)
    s = k(OpKind.ADD, k(OpKind.BMM_NT, q, kk), k(OpKind.REL_SKEW, qe))
    p = k(OpKind.CAUSAL_SOFTMAX, s, value=sc)
    ds = k(OpKind.SOFTMAX_GRAD, p, k(OpKind.BMM_NT, g, v), value=sc)
    dqe = k(OpKind.REL_UNSKEW, ds).reshape(bh * t, t)
    der = k(OpKind.MATMUL, dqe.T.copy(), q.reshape(bh * t, hd))
    dq = k(OpKind.BMM, ds, kk) + k(OpKind.MATMUL, dqe, er).reshape(bh, t, hd)
    dk = k(OpKind.BMM_TN, ds, q)
    # torch autograd
    tq, tk, tv, te = (torch.tensor(a, requires_grad=True) for a in (q, kk, v, er))
    ts = tq @ tk.transpose(1, 2) + t_skew(tq @ te.T)
    mask = torch.ones(t, t, dtype=torch.bool).tril()
    tp = torch.softmax((sc * ts).masked_fill(~mask, -torch.inf), -1)
    (tp @ tv * torch.from_numpy(g)).sum().backward()
    np.testing.assert_allclose(p, tp.detach().numpy(), rtol=1e-12, atol=1e-14)
    np.testing.assert_allclose(dq, tq.grad.numpy(), rtol=1e-10, atol=1e-12)
    np.testing.assert_allclose(dk, tk.grad.numpy(), rtol=1e-10, atol=1e-12)
    np.testing.assert_allclose(der, te.grad.numpy(), rtol=1e-10, atol=1e-12)


def test_music_transformer_coexec_equals_imperative():
    """C5 at its parity size: co-execution (graph + skeleton, natives driving the
    generator loop and the try/except arm) prints and stores exactly what the imperative
    run does, and the relative-attention program reaches the co-execution path."""
    src = music_transformer_program(steps=6, **C5_SMALL)
    ref, _, _ = run(src, "imperative", CpuBackend())
    got, st, _ = run(src, "coexec", CpuBackend())
    assert ref.lines == got.lines
    for name in ref.vars:
        assert np.array_equal(ref.vars[name].data, got.vars[name].data), name
    assert st.counters()[1] > 0                      # passes run as graphs
    kinds = {type(dc).__name__ for step in st.decision_log for dc in step}
    assert kinds == {"CaseDecision", "LoopDecision"}


def _nchw(x):
    return x.permute(0, 3, 1, 2)


def _nhwc(x):
    return x.permute(0, 2, 3, 1)


@pytest.mark.parametrize("k,s,p", [(3, 2, 1), (2, 2, 0), (3, 1, 1), (1, 2, 0), (7, 2, 3)])
def test_pooling_and_conv_dx_match_torch(k, s, p):
    """C3 ops against torch autograd: maxpool / avgpool (count_include_pad) and their
    gradients, conv2d_dx as conv2d's input gradient (including strides whose forward
    rounding leaves input rows without a window), global average pooling."""
    h = 8 if k < 7 else 9
    x = RNG.standard_normal((2, h, h, 3))
    tx = torch.tensor(x, requires_grad=True)
    tm = _nhwc(torch.nn.functional.max_pool2d(_nchw(tx), k, s, p)) if p <= k // 2 else None
    if tm is not None:
        m = k_(OpKind.MAXPOOL, x, conv=(k, s, p))
        dy = RNG.standard_normal(m.shape)
        (tm * torch.from_numpy(dy)).sum().backward()
        np.testing.assert_array_equal(m, tm.detach().numpy())
        np.testing.assert_array_equal(k_(OpKind.MAXPOOL_GRAD, x, dy, conv=(k, s, p)), tx.grad.numpy())
        tx = torch.tensor(x, requires_grad=True)
        ta = _nhwc(torch.nn.functional.avg_pool2d(_nchw(tx), k, s, p, count_include_pad=True))
        (ta * torch.from_numpy(dy)).sum().backward()
        np.testing.assert_allclose(k_(OpKind.AVGPOOL, x, conv=(k, s, p)), ta.detach().numpy(), rtol=1e-14)
        np.testing.assert_allclose(k_(OpKind.AVGPOOL_GRAD, x, dy, conv=(k, s, p)), tx.grad.numpy(), rtol=1e-13, atol=1e-16)
    w = RNG.standard_normal((k * k * 3, 4))
    tx = torch.tensor(x, requires_grad=True)
    ty = _nhwc(torch.nn.functional.conv2d(_nchw(tx), torch.tensor(w).reshape(k, k, 3, 4).permute(3, 2, 0, 1),
                                          stride=s, padding=p))
    y = k_(OpKind.CONV2D, x, w, conv=(k, s, p))
    dy = RNG.standard_normal(y.shape)
    (ty * torch.from_numpy(dy)).sum().backward()
    np.testing.assert_allclose(y, ty.detach().numpy(), rtol=1e-12, atol=1e-12)
    np.testing.assert_allclose(k_(OpKind.CONV2D_DX, dy, w, x, conv=(k, s, p)), tx.grad.numpy(),
                               rtol=1e-12, atol=1e-12)
    tx = torch.tensor(x, requires_grad=True)
    g = RNG.standard_normal((2, 3))
    (tx.mean((1, 2)) * torch.from_numpy(g)).sum().backward()
    np.testing.assert_allclose(k_(OpKind.GLOBAL_AVGPOOL, x), x.mean((1, 2)), rtol=1e-14)
    np.testing.assert_allclose(k_(OpKind.GLOBAL_AVGPOOL_GRAD, x, g), tx.grad.numpy(), rtol=1e-13, atol=1e-16)


def k_(kind, *xs, **attrs):
    return execute_kernel(kind, attrs, [Tensor(x.shape, x) for x in xs])[0].data


def test_resnet_sdpoint_coexec_equals_imperative():
    """C3 at its parity size: the 4-way SDPoint SwitchCase (static shapes per arm) runs as
    graphs once its paths are traced; co-execution prints and stores exactly what the
    imperative run does."""
    src = resnet_program(steps=12, lr=1e-3, **C3_SMALL)
    ref, _, _ = run(src, "imperative", CpuBackend())
    got, st, _ = run(src, "coexec", CpuBackend())
    assert ref.lines == got.lines
    for name in ref.vars:
        assert np.array_equal(ref.vars[name].data, got.vars[name].data), name
    assert st.counters()[1] > 1 and st.shape_replays == 0
    assert len({dc.case_index for step in st.decision_log for dc in step}) >= 2


def test_axis_ops_and_adam_elementwise():
    """slice / concat / sum_axis against numpy (sum_axis bit-exact to a sequential loop),
    sqrt / div IEEE (NaN / inf cases)."""
    x = RNG.standard_normal((3, 5, 4))
    y = RNG.standard_normal((3, 2, 4))
    np.testing.assert_array_equal(k_(OpKind.SLICE, x, dims=(1, 1, 3)), x[:, 1:4, :])
    np.testing.assert_array_equal(k_(OpKind.SLICE, x, dims=(2, 0, 0)), x[:, :, :0])
    np.testing.assert_array_equal(k_(OpKind.CONCAT, x, y, dims=(1,)), np.concatenate([x, y], 1))
    seq = x[:, 0, :] + 0.0
    for j in range(1, 5):
        seq = seq + x[:, j, :]
    np.testing.assert_array_equal(k_(OpKind.SUM_AXIS, x, dims=(1,)), seq)
    np.testing.assert_allclose(k_(OpKind.SUM_AXIS, x, dims=(0,)), x.sum(0), rtol=1e-14)
    v = np.array([4.0, 0.0, -0.0, -1.0, np.inf, 2.0])
    got = k_(OpKind.SQRT, v)
    assert got[0] == 2.0 and got[1] == 0.0 and np.signbit(got[2]) and np.isnan(got[3]) and got[4] == np.inf
    d = k_(OpKind.DIV, v, np.array(0.0))
    assert d[0] == np.inf and np.isnan(d[1]) and d[3] == -np.inf
    with pytest.raises(Exception):
        k_(OpKind.SLICE, x, dims=(1, 3, 3))
    with pytest.raises(Exception):
        k_(OpKind.CONCAT, x, RNG.standard_normal((3, 2, 5)), dims=(1,))


def test_adam_program_coexec_equals_imperative():
    """GPT-2 at its parity size with the Adam rewrite (workloads.adam_program): co-execution
    equals the imperative run bit for bit; the update differs from SGD's."""
    src = gpt2_program(steps=6, optimizer="adam", **C4_SMALL)
    assert "sqrt(div(v_wte, adam_c2))" in src
    ref, _, _ = run(src, "imperative", CpuBackend())
    got, st, _ = run(src, "coexec", CpuBackend())
    assert ref.lines == got.lines and st.counters()[1] > 0
    for name in ref.vars:
        assert np.array_equal(ref.vars[name].data, got.vars[name].data), name
    sgd, _, _ = run(gpt2_program(steps=6, **C4_SMALL), "imperative", CpuBackend())
    assert sgd.lines[0] == ref.lines[0] and sgd.lines[1:] != ref.lines[1:]


def test_fast_matmul_matches_sequential():
    """oracle.kernels.FAST_MATMUL (BLAS f64, used only by the tolerance-mode contract tests
    at full model width) agrees with the sequential-k restatement to f64 rounding."""
    from oracle import kernels as K
    r = np.random.default_rng(3)
    for m, k, n in ((64, 784, 128), (128, 3072, 96), (33, 50257 // 16, 17)):
        a, b = r.uniform(-1, 1, (m, k)), r.uniform(-1, 1, (k, n))
        ref = K.matmul_seq(a, b)
        K.FAST_MATMUL = True
        try:
            fast = K.matmul_seq(a, b)
        finally:
            K.FAST_MATMUL = False
        assert np.linalg.norm(fast - ref) / np.linalg.norm(ref) <= k * 2.0 ** -52


def test_threaded_matmul_bitwise():
    """oracle.kernels.THREADS > 1 (bench.py's CPU reference arm) tiles the output across
    host threads; each element keeps the reference's sequential-k order: bit-identical."""
    from oracle import kernels as K
    r = np.random.default_rng(4)
    for m, k, n in ((130, 300, 2500), (64, 784, 128), (1, 4096, 5000)):
        a, b = r.uniform(-1, 1, (m, k)), r.uniform(-1, 1, (k, n))
        a[0, 0] = -0.0
        ref = K.matmul_seq(a, b)
        K.THREADS = 4
        try:
            par = K.matmul_seq(a, b)
        finally:
            K.THREADS = 1
        assert par.tobytes() == ref.tobytes()
