"""Structuring (acceptance 3 and 6)."""

import random

import pytest

from paper_2201_09210_b200.errors import BudgetExceeded
from paper_2201_09210_b200.graph_gen import (ExecOp, GenConfig, InputFeed, OutputFetch, SwitchCase, UnrolledLoop,
                                             While, count_kind, graph_paths, path_language, post_dominators,
                                             structure, symprog_to_dot)
from paper_2201_09210_b200.lang.ast import SourceLoc
from paper_2201_09210_b200.tensor import OpKind
from paper_2201_09210_b200.trace_graph import Node, TraceGraph, merge_trace
from test_trace_graph import fig3_traces


def dag(edges, n_ops):
    g = TraceGraph()
    ids = {"S": g.start, "E": g.end}
    for i in range(n_ops):
        ids[i] = g._add(Node(g.ids(), "op", OpKind.RELU, {}, SourceLoc(i, ()), ("h",), [set()]))
    for a, b in edges:
        g.add_edge(ids[a], ids[b])
    return g, ids


def test_ipdom_examples():
    g, i = dag([("S", 0), (0, 1), (1, 2), (2, "E")], 3)
    pd = post_dominators(g)
    assert pd[i[0]] == i[1] and pd[i[1]] == i[2] and pd[i[2]] == g.end
    g, i = dag([("S", 0), ("S", 1), (0, 2), (1, 2), (2, "E")], 3)
    assert post_dominators(g)[g.start] == i[2]


def test_fig4_shape():
    tg = TraceGraph()
    for t in fig3_traces():
        merge_trace(tg, t)
    sp, cmap = structure(tg)
    b = sp.body
    assert isinstance(b[0], SwitchCase) and b[0].branch_id == tg.start and len(b[0].cases) == 2
    case_stmts = [[x.node_id for x in c if isinstance(x, ExecOp)] for c in b[0].cases]
    assert sorted(len(c) for c in case_stmts) == [1, 2]
    assert any(isinstance(x, InputFeed) for x in b[0].cases[0] + b[0].cases[1])
    assert isinstance(b[1], ExecOp) and isinstance(b[2], OutputFetch)
    assert isinstance(b[3], While)
    assert cmap[tg.start] == {s: k for k, s in enumerate(tg.succ[tg.start])}
    assert "cluster" in symprog_to_dot(sp)


def test_linear_has_no_control_flow():
    g, _ = dag([("S", 0), (0, 1), (1, "E")], 2)
    sp, _ = structure(g)
    assert count_kind(sp, SwitchCase) == 0 and count_kind(sp, While) == 0
    assert path_language(sp, 2) == {(2, 3)}


def test_tail_duplication():
    # Start->{a,b}, a->x->End, b->x->End with x distinct: x duplicated into both cases
    g, i = dag([("S", 0), ("S", 1), (0, 2), (1, 2), (2, "E")], 3)
    sp, _ = structure(g)
    assert path_language(sp, 1) == graph_paths(g, 1)


def random_dag(r: random.Random, n: int):
    order = list(range(n))
    edges = set()
    for k in range(n):
        # each node gets 1..3 successors among later nodes or End
        outs = r.randint(1, 3)
        for _ in range(outs):
            j = r.randint(k + 1, n)
            edges.add((k, "E" if j == n else j))
    edges.add(("S", 0))
    if r.random() < 0.5 and n > 1:
        edges.add(("S", r.randint(1, n - 1)))
    # make every node reachable from Start
    for k in range(1, n):
        if not any(b == k for a, b in edges):
            edges.add((r.randint(0, k - 1), k))
    return dag(sorted(edges, key=str), n)


@pytest.mark.parametrize("seed", range(1000))
def test_path_language_equals_dag_paths(seed):
    r = random.Random(seed)
    g, _ = random_dag(r, r.randint(1, 10))
    sp, _ = structure(g)
    assert path_language(sp, 1) == graph_paths(g, 1)


def test_budget_exceeded():
    # a ladder of diamonds duplicates exponentially without merge-backs
    edges, n = [], 0
    prev = "S"
    for k in range(12):
        a, b = n, n + 1
        n += 2
        edges += [(prev, a), (prev, b)]
        prev_nodes = (a, b)
        nxt = n
        n += 1
        edges += [(a, nxt), (b, nxt)]
        prev = nxt
    edges.append((prev, "E"))
    g, _ = dag(edges, n)
    with pytest.raises(BudgetExceeded):
        structure(g, GenConfig(max_ops=20))


def test_unrolling_rules():
    from test_trace_graph import TB
    tg = TraceGraph()
    for _ in range(2):
        t = TB()
        x = [t.op(0, "e")]
        t.loop(0, 3, lambda i: x.append(t.op(1, x[-1], loops=(0,))))
        merge_trace(tg, t.end())
    sp, _ = structure(tg)
    assert count_kind(sp, While) == 0 and count_kind(sp, UnrolledLoop) == 1
    t = TB()
    x = [t.op(0, "e")]
    t.loop(0, 1, lambda i: x.append(t.op(1, x[-1], loops=(0,))))
    merge_trace(tg, t.end())
    sp, _ = structure(tg)
    assert count_kind(sp, While) == 1
