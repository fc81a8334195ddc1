"""Flash attention on the B200 (csrc/attn_tc.cuh, planner._attn_groups): a GPT-2 step whose
heads are 64 wide and whose sequence is a multiple of 128 runs every layer's attention
forward / backward as tcgen05 flash-attention kernels.  One co-executed grad-probe step
(contract.grad_probe: every gradient lands in a variable) must agree with the f64 oracle per
tensor within the bf16 bar (2e-2), like the unfused bf16 path (COEX_FLASH=0) does; TraceGraph,
decisions and counters bit-exact."""

import numpy as np
import pytest

from contract import compare, grad_probe
from oracle import kernels as OK
from oracle.cpu_backend import CpuBackend
from paper_2201_09210_b200.trace_graph import to_json_text
from paper_2201_09210_b200.workloads import gpt2_program
from test_gpu_coexec import run

pytestmark = pytest.mark.gpu

CFG = dict(batch=2, seq=256, d=128, heads=2, layers=2, vocab=97)


@pytest.fixture(scope="module")
def oracle_run():
    src, grads = grad_probe(gpt2_program(steps=5, **CFG))
    OK.FAST_MATMUL = True
    try:
        ref, ref_st, ref_o = run(src, "coexec", CpuBackend())
    finally:
        OK.FAST_MATMUL = False
    return src, grads, ref, ref_st, ref_o


@pytest.mark.parametrize("flash", ["1", "0"])
def test_flash_attention_gradients(b200_factory, oracle_run, monkeypatch, flash):
    monkeypatch.setenv("COEX_FLASH", flash)
    src, grads, ref, ref_st, ref_o = oracle_run
    be = b200_factory("bf16", fresh=True)
    try:
        got, st, o = run(src, "coexec", be)
        plan = o.compiled.last_plan
    finally:
        be.close()
    assert plan.n_attn == (CFG["layers"] if flash == "1" else 0)
    assert st.counters() == ref_st.counters()
    assert st.decision_log == ref_st.decision_log
    assert to_json_text(o.tg) == to_json_text(ref_o.tg)
    # the key-projection bias gradient is exactly zero in exact arithmetic (softmax is
    # shift-invariant per row): bounded by the query-bias gradient of the same layer
    errs, bad = compare(ref, got, 2e-2, grads, {f"ck_{l}": f"cq_{l}" for l in range(CFG["layers"])})
    print("flash" if flash == "1" else "unfused", sorted(errs.items(), key=lambda kv: -kv[1])[:4])
    assert not bad, bad


# ---------------------------------------------------------------- kernel level (coex_flash_attn)
def _attn_ref(q, k, v, do, scale):
    """f64 causal attention forward / backward (the unfused composition bmm_nt ->
    causal_softmax -> bmm of oracle/kernels.py and its hand-written backward)."""
    T = q.shape[1]
    s = np.einsum("bte,bse->bts", q, k) * scale
    s = np.where(np.tril(np.ones((T, T), bool)), s, -np.inf)
    p = np.exp(s - s.max(-1, keepdims=True))
    p /= p.sum(-1, keepdims=True)
    o = np.einsum("bts,bse->bte", p, v)
    dp = np.einsum("bte,bse->bts", do, v)
    ds = p * (dp - (dp * p).sum(-1, keepdims=True)) * scale
    return o, np.einsum("bts,bse->bte", ds, k), np.einsum("bts,bte->bse", ds, q), np.einsum("bts,bte->bse", p, do)


def _rel(a, b):
    return float(np.linalg.norm(a - b) / np.linalg.norm(b))


@pytest.mark.parametrize("BH,T", [(3, 128), (4, 512), (2, 1024)])
def test_flash_kernels_vs_f64(b200_factory, BH, T):
    """Each k_fa_* kernel against f64 causal attention: bf16 operands, fp32 accumulation --
    within the bf16 bar (2e-2 relative, norm-wise per output tensor)."""
    from paper_2201_09210_b200.tensor import Tensor
    r = np.random.default_rng(BH * T)
    q, k, v, do = (r.standard_normal((BH, T, 64)) for _ in range(4))
    scale = 0.125
    o_ref, dq_ref, dk_ref, dv_ref = _attn_ref(q, k, v, do, scale)
    be = b200_factory("bf16", fresh=True)
    try:
        dq_, dk_, dv_ = (be.put(Tensor(x.shape, x)) for x in (q, k, v))
        o, lse = be.flash_attention([dq_, dk_, dv_], scale)
        o_np = be.get(o).data.reshape(BH, T, 64)
        dq, dk, dv = be.flash_attention([dq_, dk_, dv_, o, be.put(Tensor(do.shape, do)), lse], scale, backward=True)
        got = [be.get(t).data.reshape(BH, T, 64) for t in (dq, dk, dv)]
    finally:
        be.close()
    errs = {"O": _rel(o_np, o_ref), "dQ": _rel(got[0], dq_ref), "dK": _rel(got[1], dk_ref),
            "dV": _rel(got[2], dv_ref)}
    print(BH, T, errs)
    assert all(e <= 2e-2 for e in errs.values()), errs
