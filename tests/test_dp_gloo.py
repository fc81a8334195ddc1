"""Data-parallel co-execution with world size 2 on CPU (gloo), against the single
process run at the global batch: sharded feeds + Partial/AllReduce insertion must
reproduce the global-batch results within tolerance, with identical decisions,
TraceGraph and Stats counters on every rank."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle.cpu_backend import CpuBackend
from paper_2201_09210_b200 import coexec, lang
from paper_2201_09210_b200.dataset import SyntheticDataset
from paper_2201_09210_b200.dp import DPGroup
from paper_2201_09210_b200.tensor import Tensor
from paper_2201_09210_b200.workloads import (c1_program, dcgan_program, gpt2_program, music_transformer_program,
                                             resnet_program)

SMALL_C1 = c1_program(steps=12, batch=8, hidden=16, din=12, dout=3)
BATCH = 8
SMALL_C2 = dcgan_program(steps=6, batch=8, nz=6, ngf=4, ndf=4, img=16)
SMALL_C4 = gpt2_program(steps=4, batch=BATCH, seq=8, d=16, heads=2, layers=2, vocab=23)
SMALL_C3 = resnet_program(steps=14, batch=BATCH, img=32, width=2, blocks=(1, 1, 1, 1), classes=5, lr=1e-3)
SMALL_C4_ADAM = gpt2_program(steps=4, batch=BATCH, seq=8, d=16, heads=2, layers=2, vocab=23, optimizer="adam")
SMALL_C5 = music_transformer_program(steps=8, batch=BATCH, seq=8, d=16, heads=2, layers=2, vocab=23)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, src, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)

    def allreduce(arr, avg):
        t = torch.from_numpy(np.array(arr, dtype=np.float64))
        dist.all_reduce(t)
        if avg:
            t /= world
        return t.numpy()

    be = CpuBackend(dp=DPGroup(rank, world, BATCH, allreduce))
    ds = SyntheticDataset(0)
    o = coexec.Orchestrator(lang.parse(src), ds, coexec.Mode.coexec, coexec.RunConfig(), be)
    res, st = o.run()
    plans = [(p.replicated, p.reason, p.allreduce_nodes, sorted(p.sharded_slots)) for p in be.dp_plans]
    out[rank] = (res.lines, {k: v.data for k, v in res.vars.items()}, st.counters(), st.decision_log, plans)
    dist.destroy_process_group()


def run_dp(src, world=2):
    ctx = mp.get_context("spawn")
    mgr = ctx.Manager()
    out = mgr.dict()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, src, out)) for r in range(world)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(120)
        assert p.exitcode == 0
    return dict(out)


@pytest.mark.parametrize("src", [SMALL_C1], ids=["c1_small"])
def test_dp2_matches_global_batch(src):
    ref, ref_st = coexec.run(lang.parse(src), SyntheticDataset(0), "coexec", backend=CpuBackend())
    out = run_dp(src)
    r0, r1 = out[0], out[1]
    # every rank made the same decisions and printed the same lines
    assert r0[0] == r1[0] and r0[3] == r1[3] and r0[2] == r1[2]
    assert r0[2] == ref_st.counters()
    plans = r0[4]
    assert plans and not plans[-1][0], plans          # sharded, not replicated
    assert len(plans[-1][2]) >= 3                     # loss + two gradients all-reduced
    for a, b in zip(ref.lines, r0[0]):
        assert abs(float(a) - float(b)) <= 1e-12 * max(1.0, abs(float(a)))
    for k, t in ref.vars.items():
        np.testing.assert_allclose(r0[1][k], t.data, rtol=1e-10, atol=1e-13)
        np.testing.assert_array_equal(r0[1][k], r1[1][k])


def test_unshardable_program_runs_replicated():
    src = """
var w = fill([4, 3], 0.5)
steps 6 {
  let x = input("x", [8, 4])
  let h = matmul(x, w)
  print(h)
  w = add(w, fill([4, 3], 0.01))
}
"""
    ref, _ = coexec.run(lang.parse(src), SyntheticDataset(0), "coexec", backend=CpuBackend())
    out = run_dp(src)
    assert out[0][4][-1][0] is True                   # fetching a sharded activation -> replicated
    assert out[0][0] == ref.lines == out[1][0]


@pytest.mark.parametrize("src,tol", [(SMALL_C2, 1e-9), (SMALL_C3, 1e-8)], ids=["dcgan", "resnet_sdpoint"])
def test_dp2_dcgan_matches_global_batch(src, tol):
    """C2 (DCGAN) / C3 (ResNet-50 + SDPoint) data parallel at world size 2 on distinct row
    shards: activations row-sharded through the convolutions, pooling and (C3) the
    path-dependent SDPoint tail; batch norm SYNCHRONISED (rank-local raw column sums
    all-reduced, statistics of the global batch); weight / beta gradients all-reduced (P+),
    gamma gradients already global, the loss averaged (P~).  Equal to the single-process
    global-batch run up to summation order (C3 within 1e-8: the tiny network's training
    dynamics amplify f64 rounding-order differences ~10x per step)."""
    ref, ref_st = coexec.run(lang.parse(src), SyntheticDataset(0), "coexec", backend=CpuBackend())
    out = run_dp(src)
    r0, r1 = out[0], out[1]
    assert r0[0] == r1[0] and r0[3] == r1[3] and r0[2] == r1[2]
    assert r0[2] == ref_st.counters()
    plans = r0[4]
    assert plans and not any(p[0] for p in plans), plans   # every specialisation sharded
    assert max(len(p[2]) for p in plans) >= 6               # weight, BN-shift and loss reductions
    for a, b in zip(ref.lines, r0[0]):
        assert abs(float(a) - float(b)) <= tol * max(1.0, abs(float(a))), (a, b)
    for k, t in ref.vars.items():
        np.testing.assert_allclose(r0[1][k], t.data, rtol=tol * 10, atol=tol * 1e-2)
        np.testing.assert_array_equal(r0[1][k], r1[1][k])


@pytest.mark.parametrize("src", [SMALL_C4, SMALL_C4_ADAM, SMALL_C5], ids=["gpt2", "gpt2_adam", "music_transformer"])
def test_dp2_gpt2_matches_global_batch(src):
    """C4 (GPT-2) / C5 (Music Transformer) data parallel at world size 2: sequences sharded
    through embeddings, layernorms, attention (batch = sequences x heads; C5's relative
    logits q.er^T and their skew row-wise) and the MLP; weight, bias, layernorm, embedding
    and relative-table gradients all-reduced (P+), the loss averaged (P~), the
    cross-entropy gradient divided by the global row count -- equal to the global-batch
    run."""
    ref, ref_st = coexec.run(lang.parse(src), SyntheticDataset(0), "coexec", backend=CpuBackend())
    out = run_dp(src)
    r0, r1 = out[0], out[1]
    assert r0[0] == r1[0] and r0[3] == r1[3] and r0[2] == r1[2]
    assert r0[2] == ref_st.counters()
    plans = r0[4]
    assert plans and not any(p[0] for p in plans), plans
    assert max(len(p[2]) for p in plans) >= 20
    for a, b in zip(ref.lines, r0[0]):
        assert abs(float(a) - float(b)) <= 1e-9 * max(1.0, abs(float(a))), (a, b)
    keys = sorted(ref.vars)
    w = np.concatenate([ref.vars[k].data.ravel() for k in keys])
    g0 = np.concatenate([r0[1][k].ravel() for k in keys])
    g1 = np.concatenate([r1[1][k].ravel() for k in keys])
    assert np.linalg.norm(g0 - w) <= 1e-9 * np.linalg.norm(w)
    np.testing.assert_array_equal(g0, g1)


class _FakeNvlsLib:
    """Stands in for libcoexb200.so's gradient-region entry points (no GPU here): records
    the calls, fails the ones listed in `fail` on this rank."""

    def __init__(self, rank, fail):
        self.rank, self.fail, self.calls = rank, set(fail), []

    def _rc(self, name):
        self.calls.append(name)
        return 8 if name in self.fail else 0

    def coex_nvls_create(self, ctx, nbytes, world, info):
        info[0], info[1], info[2] = 4242, 17, nbytes
        return self._rc("create")

    def coex_nvls_attach(self, ctx, pid, fd, nbytes, world):
        assert (pid, fd, nbytes) == (4242, 17, 1 << 20)     # rank 0's export reached every rank
        return self._rc("attach")

    def coex_nvls_bind(self, ctx):
        return self._rc("bind")

    def coex_p2p_create(self, ctx, nbytes, h):
        h.raw = bytes([self.rank]) * 64
        return self._rc("p2p_create")

    def coex_p2p_open(self, ctx, allh, world):
        assert allh.raw[:64] == bytes([0]) * 64 and allh.raw[64:128] == bytes([1]) * 64
        return self._rc("p2p_open")

    def coex_nvls_info(self, ctx, out):
        mode = 2 if "p2p_open" in self.calls else 1
        out[0], out[1], out[2] = 1 << 20, 2, mode
        return 0

    def coex_last_error(self):
        return b"fake"


def _nvls_worker(rank, world, port, mode, fail, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    if mode is None:
        os.environ.pop("COEX_NVLS", None)
    else:
        os.environ["COEX_NVLS"] = mode
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2201_09210_b200.b200 import B200Backend
    be = object.__new__(B200Backend)            # host logic only: no context, no device
    be.ctx, be.dp = None, DPGroup(rank, world, BATCH)
    be.lib = _FakeNvlsLib(rank, fail.get(rank, ()))
    be.nvls_bytes, be.nvls_mode = 0, "none"
    be._init_nvls(1 << 20)
    out[rank] = (be.nvls_bytes, be.nvls_mode, list(be.lib.calls))
    dist.destroy_process_group()


@pytest.mark.parametrize("mode,fail,want", [
    (None, {}, ("multicast", [["create", "attach", "bind"], ["attach", "bind"]])),
    # a rank that cannot import the multicast fd sends the whole group back to NCCL
    (None, {1: ("attach",)}, ("none", [["create", "attach"], ["attach"]])),
    # ... or, with COEX_NVLS=1, to the P2P transport
    ("1", {1: ("attach",)}, ("p2p", [["create", "attach", "p2p_create", "p2p_open"],
                                     ["attach", "p2p_create", "p2p_open"]])),
    # no multicast object at all (the one-GPU boxes): NCCL by default
    (None, {0: ("create",)}, ("none", [["create"], []])),
    ("p2p", {}, ("p2p", [["p2p_create", "p2p_open"], ["p2p_create", "p2p_open"]])),
], ids=["multicast", "attach_fails_nccl", "attach_fails_p2p", "no_multicast", "forced_p2p"])
def test_dp2_gradient_region_setup(mode, fail, want):
    """World-2 host logic of the GEMM -> all-reduce fusion set-up (B200Backend._init_nvls):
    rank 0's multicast export is broadcast, every rank's attach verdict is agreed on before
    anyone binds, and every rank ends in the same transport."""
    ctx = mp.get_context("spawn")
    mgr = ctx.Manager()
    out = mgr.dict()
    port = _free_port()
    procs = [ctx.Process(target=_nvls_worker, args=(r, 2, port, mode, fail, out)) for r in range(2)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(120)
        assert p.exitcode == 0
    res = dict(out)
    tr, calls = want
    for r in range(2):
        nbytes, got_mode, got_calls = res[r]
        assert got_mode == tr and got_calls == calls[r], (r, res[r])
        assert (nbytes > 0) == (tr != "none")
