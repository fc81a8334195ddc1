"""Planner fusions on real workloads (CPU, no device): batched parameter-update chains
(T_MCHAIN, k_chain_multi), batch-norm + activation (plan kind 101), layernorm bf16
shadows, and the independence rule the chain grouping relies on."""

import pytest

from bench import make_orch
from oracle.cpu_backend import CpuBackend
from paper_2201_09210_b200.dataset import SyntheticDataset
from paper_2201_09210_b200.planner import T_CHAIN, T_MCHAIN, Planner, _conflicts
from paper_2201_09210_b200.tensor import OpKind
from paper_2201_09210_b200.trace_graph import VARIES
from paper_2201_09210_b200.workloads import C2_SMALL, C4_SMALL, dcgan_program, gpt2_program


def _planner(src, steps=5):
    o = make_orch(src, SyntheticDataset(0), CpuBackend())
    for _ in range(steps):
        o.step()
    feed = {(n.id, p): tuple(s) for n in o.tg.all_nodes() if n.typ == "op" for p, s in n.feed_shapes.items()}
    consts = {}
    for n in o.tg.all_nodes():
        if n.typ == "op":
            for pos, v in n.feed_values.items():
                if v is not VARIES and tuple(n.feed_shapes.get(pos, (0,))) == ():
                    consts[(n.id, pos)] = v
    vs = o.be.var_shapes()
    vi = {k: j for j, k in enumerate(sorted(vs))}
    pl = Planner(o.sp, o.tg, vi, vs, feed, 4, bf16=True, const_slots=consts)
    plan = pl.build()
    return pl, plan


@pytest.fixture(scope="module")
def dcgan():
    return _planner(dcgan_program(steps=8, **C2_SMALL))


def test_update_chains_batched(dcgan):
    pl, plan = dcgan
    assert pl.n_mchains >= 1
    assert T_MCHAIN in plan.words


def test_grouped_chains_are_independent(dcgan):
    pl, _ = dcgan
    metas = [m for m in pl._chain_meta.values()]
    assert metas, "no chains recorded"
    # every recorded chain's inputs / publications are well-formed cell codes
    for w, ins, pubs, red in metas:
        assert w[0] == T_CHAIN and isinstance(ins, list) and isinstance(pubs, list)


def test_conflict_rule():
    # a chain reading cell 5 cannot run beside one publishing it; variable 3's reads conflict
    # with a publication of its overlay slot (-(2000 + 3))
    assert _conflicts([5], [5])
    assert _conflicts([-(1000 + 3)], [-(2000 + 3)])
    assert not _conflicts([5, -(1000 + 3)], [6, -(2000 + 4)])


def test_batchnorm_activation_pairs(dcgan):
    pl, _ = dcgan
    assert pl._act_for
    for bn_id, act in pl._act_for.items():
        assert pl.ops[bn_id].kind is OpKind.BATCHNORM
        assert act.kind in (OpKind.RELU, OpKind.LEAKY_RELU)
        assert act.inputs[0].cands == (bn_id,)


def test_layernorm_shadows():
    pl, _ = _planner(gpt2_program(steps=6, **C4_SMALL))
    kinds = {pl.ops[n].kind for n in pl.shadow}
    assert OpKind.LAYERNORM in kinds and OpKind.CAUSAL_SOFTMAX in kinds


def test_cross_entropy_fused_with_shadow_only_gradient():
    """C4: cross_entropy + cross_entropy_grad of the same logits become one plan op (kind
    102); the gradient's only readers are the LM-head GEMMs, which read its bf16 shadow, so
    the fp32 gradient is never written (attr 1)."""
    from paper_2201_09210_b200.planner import XOP_CE_FUSED
    pl, plan = _planner(gpt2_program(steps=6, **C4_SMALL))
    assert pl._ce_loss
    for g, lo in pl._ce_loss.items():
        assert pl.ops[g].kind is OpKind.CROSS_ENTROPY_GRAD and lo.kind is OpKind.CROSS_ENTROPY
        assert g in pl.shadow
    assert pl._skip_f32 and all(w[at] == 1 for w, at in pl._skip_f32.values())
    w = plan.words
    assert any(w[i] == XOP_CE_FUSED and w[i - 1] == 10 for i in range(1, len(w)))


def test_flash_attention_groups():
    """C4 at a flash-eligible shape (head dim 64, T = 128): every layer's attention forward and
    backward become two T_ATTN items; the scores / probabilities are never computed."""
    from paper_2201_09210_b200.planner import T_ATTN
    cfg = dict(batch=2, seq=128, d=128, heads=2, layers=2, vocab=97)
    pl, plan = _planner(gpt2_program(steps=6, **cfg))
    assert pl.n_attn == 2
    w = plan.words
    assert sum(1 for i in range(1, len(w)) if w[i] == T_ATTN and w[i + 1] in (0, 1) and w[i + 2] == 4) >= 4
    # the head split / merge transposes fold into the attention words: merged rows of the
    # [B*T, H*hd] projections (H = 2, row pitch 128); no 4-D transpose is launched
    assert pl.n_head_fold == 2
    assert sum(1 for i in range(1, len(w) - 5) if w[i] == T_ATTN and w[i + 1] in (0, 1) and w[i + 2] == 4
               and w[i + 3] == 128 and w[i + 4] == 2 and w[i + 5] == 128) >= 4
    emitted = {y.node_id for y in pl.ops.values() if y.kind is OpKind.TRANSPOSE and len(y.attrs["perm"]) == 4}
    assert emitted and all(n not in pl._emitted for n in emitted)


@pytest.mark.parametrize("which", ["c2", "c4"])
def test_dp_allreduce_buckets(which):
    """Data-parallel gradient all-reduces are bucketed and asynchronous: consecutive
    all-reduces of adjacent buffers form one collective (T_ALLREDUCE async), and a T_JOIN
    precedes the first instruction reading any pending value (the parameter updates)."""
    from paper_2201_09210_b200.dp import local_feed_shapes, shard_program
    from paper_2201_09210_b200.graph_gen import ExecOp
    from paper_2201_09210_b200.planner import T_ALLREDUCE, T_JOIN, _ARBucket, _Join
    src = dcgan_program(steps=8, **C2_SMALL) if which == "c2" else gpt2_program(steps=6, **C4_SMALL)
    o = make_orch(src, SyntheticDataset(0), CpuBackend())
    for _ in range(5):
        o.step()
    feed = {(n.id, p): tuple(s) for n in o.tg.all_nodes() if n.typ == "op" for p, s in n.feed_shapes.items()}
    vs = o.be.var_shapes()
    vi = {k: j for j, k in enumerate(sorted(vs))}
    gshapes = Planner(o.sp, o.tg, vi, vs, feed, 4).infer_shapes()
    batch = (C2_SMALL if which == "c2" else C4_SMALL)["batch"]
    dplan = shard_program(o.sp, feed, gshapes, batch, 2)
    assert not dplan.replicated, dplan.reason
    pl = Planner(dplan.sp, o.tg, vi, vs, local_feed_shapes(feed, dplan), 4, bf16=True,
                 force_store=dplan.allreduce_nodes)
    plan = pl.build()
    assert pl.n_ar_buckets >= 1
    n_ar = len([n for n in dplan.allreduce_nodes])
    w = plan.words
    assert T_JOIN in w and T_ALLREDUCE in w
    for lst in pl._ar_lists:
        pending = set()
        members = [m.node_id for x in lst if isinstance(x, _ARBucket) for m in x.members]
        assert len(members) == len(set(members))
        for x in lst:
            if isinstance(x, _ARBucket):
                bufs = [pl._node_buf[m.node_id][0] for m in x.members]
                assert bufs == list(range(bufs[0], bufs[0] + len(bufs)))     # adjacent in the arena
                pending |= {m.node_id for m in x.members}
            elif isinstance(x, _Join):
                pending.clear()
            elif isinstance(x, ExecOp):
                reads = {c for b in x.inputs if not b.fed for c in b.cands}
                assert not (reads & pending), (x.kind, reads & pending)
        assert not pending
    # fewer collectives than gradients: bucketing merged some
    n_coll = sum(len(x.members) > 0 for lst in pl._ar_lists for x in lst if isinstance(x, _ARBucket))
    assert n_coll < n_ar, (n_coll, n_ar)


@pytest.mark.parametrize("which", ["c2", "c4"])
def test_dp_nvls_buckets(which):
    """NVLS plans (csrc/nvls.cuh): every sum all-reduced gradient gets a buffer in the
    multicast region (the plan header's NVLS list), every bucket over them is a T_NVLS_AR
    item, and each list holding such buckets starts with ONE T_NVLS_ZERO over its bucket
    buffers -- before any producer (the GEMM epilogues add into zeroed copies).  Average
    all-reduces (the loss) stay NCCL buckets in the arena; a region too small for the
    plan's gradients falls back to NCCL entirely."""
    from paper_2201_09210_b200.dp import local_feed_shapes, shard_program
    from paper_2201_09210_b200.graph_gen import ExecOp
    from paper_2201_09210_b200.planner import MAGIC, _ARBucket, _NvlsZero, walk
    src = dcgan_program(steps=8, **C2_SMALL) if which == "c2" else gpt2_program(steps=6, **C4_SMALL)
    o = make_orch(src, SyntheticDataset(0), CpuBackend())
    for _ in range(5):
        o.step()
    feed = {(n.id, p): tuple(s) for n in o.tg.all_nodes() if n.typ == "op" for p, s in n.feed_shapes.items()}
    vs = o.be.var_shapes()
    vi = {k: j for j, k in enumerate(sorted(vs))}
    gshapes = Planner(o.sp, o.tg, vi, vs, feed, 4).infer_shapes()
    batch = (C2_SMALL if which == "c2" else C4_SMALL)["batch"]
    dplan = shard_program(o.sp, feed, gshapes, batch, 2)
    assert not dplan.replicated, dplan.reason

    def build(nbytes):
        pl = Planner(dplan.sp, o.tg, vi, vs, local_feed_shapes(feed, dplan), 4, bf16=True,
                     force_store=dplan.allreduce_nodes, nvls_bytes=nbytes)
        return pl, pl.build()

    pl, plan = build(1 << 30)
    sums = {x.node_id for x in walk(dplan.sp.body) if type(x).__name__ == "AllReduce" and not x.avg}
    assert sums and plan.nvls_bufs == len(sums) and plan.nvls_buckets >= 1
    w = plan.words
    assert w[0] == MAGIC and w[3 + w[2]] == len(pl.nvls_bufs)
    assert w[4 + w[2]: 4 + w[2] + len(pl.nvls_bufs)] == pl.nvls_bufs
    assert {pl._node_buf[n][0] for n in sums} == set(pl.nvls_bufs)
    for lst in pl._ar_lists:
        nv = [x for x in lst if isinstance(x, _ARBucket) and pl._node_buf[x.members[0].node_id][0] in pl.nvls_set]
        zeros = [i for i, x in enumerate(lst) if isinstance(x, _NvlsZero)]
        if not nv:
            assert not zeros
            continue
        assert zeros == [0]
        z = lst[0]
        for x in nv:
            assert all(not m.avg for m in x.members)
            for m in x.members:
                assert z.first <= pl._node_buf[m.node_id][0] <= z.last
        produced = [i for i, x in enumerate(lst) if isinstance(x, ExecOp) and x.node_id in sums]
        assert produced and min(produced) > 0
    # too small a region: the whole plan keeps NCCL buckets
    pl2, plan2 = build(4096)
    assert plan2.nvls_bufs == 0 and plan2.nvls_buckets == 0 and pl2.n_ar_buckets >= 1


def test_bias_add_fused_into_gemm():
    """C4: every projection's bias_add(matmul(a, w), c) becomes the GEMM's epilogue (one plan
    op publishing the bias_add's output); the bias_add is never launched on its own."""
    pl, plan = _planner(gpt2_program(steps=6, **C4_SMALL))
    assert pl.n_bias_fused == 6 * C4_SMALL["layers"]
    for m, ba in pl._bias_for.items():
        assert pl.ops[m].kind is OpKind.MATMUL and ba.kind is OpKind.BIAS_ADD
        assert ba.node_id not in pl._emitted and m in pl._emitted


def test_layernorm_backward_fused():
    """C4: layernorm_dx + ln_dgamma + sum_rows over the same (x, dy) become one plan op
    (kind 103, one pass over x and dy) -- two per layer plus the final layernorm."""
    from paper_2201_09210_b200.planner import T_XOP, XOP_LN_BWD
    pl, plan = _planner(gpt2_program(steps=6, **C4_SMALL))
    w = plan.words
    n = sum(1 for i in range(len(w) - 1) if w[i] == T_XOP and w[i + 1] == XOP_LN_BWD)
    assert n == 2 * C4_SMALL["layers"] + 1, n


def test_arm_exclusive_buffers(dcgan):
    """C2's D / G SwitchCase: activations produced and read inside one case share a region
    with the other case's (cases never run in the same pass); views are well-formed and
    nothing fetched / merged / pinned is aliased."""
    from paper_2201_09210_b200.planner import walk
    from paper_2201_09210_b200.graph_gen import SwitchCase
    pl, plan = dcgan
    w = plan.words
    nb = w[2]
    sizes = w[3:3 + nb]
    views = [i for i, x in enumerate(sizes) if x < 0]
    assert views, "no arm-exclusive views"
    unaliased, region = pl.arm_alias_bytes
    assert 0 < region < unaliased
    for i in views:
        v = -sizes[i] - 1
        parent, off = v >> 40, v & ((1 << 40) - 1)
        assert 0 <= parent < i and sizes[parent] >= 0 and off < sizes[parent]
    aliased = {n for n, (b0, _, _) in pl._node_buf.items() if b0 in set(views)}
    assert not aliased & set(pl.sp.fetch_nodes)
    sw = [x for x in walk(pl.sp.body) if isinstance(x, SwitchCase)]
    assert sw


def test_rel_skew_add_fused():
    """C5's attention logits add(q.k^T, rel_skew(q.er^T)): the skew's only reader is the add,
    so the planner emits ONE plan kind 104 item per layer at the add's position (csrc
    k_rel_skew_v4<0, true>) and the skew node itself disappears; f64 parity mode keeps the
    two ops."""
    from paper_2201_09210_b200.planner import T_XOP, XOP_SKEW_ADD
    from paper_2201_09210_b200.workloads import C5_SMALL, music_transformer_program
    src = music_transformer_program(steps=6, **C5_SMALL)
    o = make_orch(src, SyntheticDataset(0), CpuBackend())
    for _ in range(5):
        o.step()
    feed = {(n.id, p): tuple(s) for n in o.tg.all_nodes() if n.typ == "op" for p, s in n.feed_shapes.items()}
    vs = o.be.var_shapes()
    vi = {k: j for j, k in enumerate(sorted(vs))}
    layers = C5_SMALL.get("layers", 2)
    for esize, want in ((4, layers), (8, 0)):
        pl = Planner(o.sp, o.tg, vi, vs, feed, esize, bf16=esize == 4)
        w = pl.build().words
        n = sum(1 for i in range(len(w) - 1) if w[i] == T_XOP and w[i + 1] == XOP_SKEW_ADD)
        assert n == want == len(pl._skew_add), (esize, n)
        for nid in pl._skew_add:
            assert pl.ops[nid].kind is OpKind.ADD
            skews = [c for b in pl.ops[nid].inputs if not b.fed for c in b.cands
                     if pl.ops[c].kind is OpKind.REL_SKEW]
            assert skews and all(c not in pl._emitted for c in skews)
