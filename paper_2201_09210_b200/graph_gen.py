"""Symbolic program generation from a TraceGraph.

Specification: SPEC.md:348-418 (not shipped by the reference).

* ``post_dominators``: immediate post-dominators per nesting level
  (Cooper-Harvey-Kennedy on the reversed DAG).
* ``structure``: recursive region emission with tail duplication
  (SPEC.md:372-380): a node with out-degree > 1 becomes
  ``SwitchCase{n, cases=[region(s_i, ipdom(n))]}`` with cases in child
  insertion order (the CaseMap); Loop nodes become ``While`` or,
  when every observed trip count is the same k, ``UnrolledLoop`` with k bodies.
  InputFeed precedes and OutputFetch follows each ExecOp instance.  Duplicated
  instances keep their TraceGraph node id.
* ``path_language``: the executable ExecOp-id sequences, the structuring oracle
  (SPEC.md:381-389).
"""

from __future__ import annotations

from dataclasses import dataclass, field

from .errors import BudgetExceeded, ExplosionGuard
from .tensor import OpKind, canonical_attrs
from .trace_graph import Node, TraceGraph

# ---------------------------------------------------------------- IR


@dataclass(frozen=True)
class Bind:
    """An ExecOp input: produced in-graph by the latest of ``cands``, or fed (``slot``)."""

    cands: tuple = ()
    slot: tuple | None = None

    @property
    def fed(self) -> bool:
        return self.slot is not None


@dataclass
class ExecOp:
    node_id: int
    kind: OpKind
    attrs: dict
    inputs: list


@dataclass
class InputFeed:
    slot: tuple


@dataclass
class OutputFetch:
    node_id: int


@dataclass
class SwitchCase:
    branch_id: int
    cases: list


@dataclass
class While:
    loop_id: int
    node_id: int
    body: list


@dataclass
class UnrolledLoop:
    loop_id: int
    node_id: int
    bodies: list


@dataclass
class SymProgram:
    body: list
    case_map: dict = field(default_factory=dict)   # branch node id -> {successor id: case index}
    unrolled: dict = field(default_factory=dict)   # loop node id -> trip count k
    n_execops: int = 0
    fetch_nodes: set = field(default_factory=set)
    feed_slots: set = field(default_factory=set)


@dataclass
class GenConfig:
    max_ops: int = 10_000


# ---------------------------------------------------------------- post-dominators


def post_dominators(g: TraceGraph) -> dict:
    """node id -> immediate post-dominator id for one nesting level (End excluded)."""
    # reverse post-order of the reversed graph, rooted at End
    order, seen = [], set()
    stack = [(g.end, iter(g.pred[g.end]))]
    seen.add(g.end)
    while stack:
        u, it = stack[-1]
        nxt = next((v for v in it if v not in seen), None)
        if nxt is None:
            order.append(u)
            stack.pop()
        else:
            seen.add(nxt)
            stack.append((nxt, iter(g.pred[nxt])))
    rpo = list(reversed(order))
    idx = {u: i for i, u in enumerate(rpo)}
    ipdom = {g.end: g.end}

    def meet(a, b):
        while a != b:
            while idx[a] > idx[b]:
                a = ipdom[a]
            while idx[b] > idx[a]:
                b = ipdom[b]
        return a

    changed = True
    while changed:
        changed = False
        for u in rpo[1:]:
            done = [s for s in g.succ[u] if s in ipdom]
            if not done:
                continue
            new = done[0]
            for s in done[1:]:
                new = meet(new, s)
            if ipdom.get(u) != new:
                ipdom[u] = new
                changed = True
    del ipdom[g.end]
    return ipdom


def all_post_dominators(tg: TraceGraph) -> dict:
    out = dict(post_dominators(tg))
    for n in tg.nodes.values():
        if n.typ == "loop":
            out.update(all_post_dominators(n.body))
    return out


# ---------------------------------------------------------------- structuring


class _Emitter:
    def __init__(self, cfg: GenConfig, sp: SymProgram):
        self.cfg = cfg
        self.sp = sp
        self.ipdom_cache: dict = {}

    def ipdom(self, g: TraceGraph) -> dict:
        key = id(g)
        if key not in self.ipdom_cache:
            self.ipdom_cache[key] = post_dominators(g)
        return self.ipdom_cache[key]

    def count(self, n: int):
        self.sp.n_execops += n
        if self.sp.n_execops > self.cfg.max_ops:
            raise BudgetExceeded(f"symbolic program exceeds max_ops={self.cfg.max_ops}")

    def node(self, g: TraceGraph, n: Node, out: list):
        if n.typ == "op":
            binds = []
            for p, k in enumerate(n.in_kinds):
                if k == "e":
                    out.append(InputFeed((n.id, p)))
                    self.sp.feed_slots.add((n.id, p))
                    binds.append(Bind(slot=(n.id, p)))
                else:
                    binds.append(Bind(cands=tuple(sorted(n.cands[p]))))
            out.append(ExecOp(n.id, n.kind, n.attrs, binds))
            self.count(1)
            if n.fetch:
                out.append(OutputFetch(n.id))
                self.sp.fetch_nodes.add(n.id)
        elif n.typ == "loop":
            body = self.region(n.body, n.body.start, n.body.end)
            if len(n.trip_counts) == 1:
                k = next(iter(n.trip_counts))
                self.count(_count_ops(body) * max(k - 1, 0))
                self.sp.unrolled[n.id] = k
                out.append(UnrolledLoop(n.loop_id, n.id, [body] * k))
            else:
                out.append(While(n.loop_id, n.id, body))

    def region(self, g: TraceGraph, n: int, stop: int) -> list:
        out: list = []
        while n != stop:
            self.node(g, g.nodes[n], out)
            succ = g.succ[n]
            if len(succ) == 1:
                n = succ[0]
                continue
            m = self.ipdom(g)[n]
            self.sp.case_map[n] = {s: i for i, s in enumerate(succ)}
            out.append(SwitchCase(n, [self.region(g, s, m) for s in succ]))
            n = m
        return out


def _count_ops(insts: list) -> int:
    c = 0
    for x in insts:
        if isinstance(x, ExecOp):
            c += 1
        elif isinstance(x, SwitchCase):
            c += sum(_count_ops(cs) for cs in x.cases)
        elif isinstance(x, While):
            c += _count_ops(x.body)
        elif isinstance(x, UnrolledLoop):
            c += sum(_count_ops(b) for b in x.bodies)
    return c


def structure(tg: TraceGraph, config: GenConfig | None = None) -> tuple:
    """TraceGraph -> (SymProgram, CaseMap)."""
    sp = SymProgram([])
    em = _Emitter(config or GenConfig(), sp)
    sp.body = em.region(tg, tg.start, tg.end)
    return sp, sp.case_map


# ---------------------------------------------------------------- path language


def path_language(sp, trip_bound: int, cap: int = 100_000) -> set:
    """All executable ExecOp node-id sequences of ``sp``."""
    insts = sp.body if isinstance(sp, SymProgram) else sp

    def seqs(lst: list) -> set:
        acc = {()}
        for x in lst:
            if isinstance(x, ExecOp):
                opts = {(x.node_id,)}
            elif isinstance(x, SwitchCase):
                opts = set().union(*(seqs(c) for c in x.cases)) if x.cases else {()}
            elif isinstance(x, While):
                one = seqs(x.body)
                opts, layer = {()}, {()}
                for _ in range(trip_bound):
                    layer = {a + b for a in layer for b in one}
                    opts |= layer
                    if len(opts) > cap:
                        raise ExplosionGuard("path enumeration cap exceeded")
            elif isinstance(x, UnrolledLoop):
                opts = {()}
                for b in x.bodies:
                    sb = seqs(b)
                    opts = {a + c for a in opts for c in sb}
            else:
                continue
            acc = {a + b for a in acc for b in opts}
            if len(acc) > cap:
                raise ExplosionGuard("path enumeration cap exceeded")
        return acc

    return seqs(insts)


def graph_paths(tg: TraceGraph, trip_bound: int, cap: int = 100_000) -> set:
    """Brute-force Start->End op-id paths of a TraceGraph (loop bodies expanded
    0..trip_bound times, or exactly k times when trip_counts == {k})."""

    def paths(g: TraceGraph) -> set:
        res = set()

        def walk(u, acc):
            if u == g.end:
                res.add(acc)
                if len(res) > cap:
                    raise ExplosionGuard("path enumeration cap exceeded")
                return
            n = g.nodes[u]
            if n.typ == "op":
                nexts = {acc + (u,)}
            elif n.typ == "loop":
                body = paths(n.body)
                if len(n.trip_counts) == 1:
                    trips = [next(iter(n.trip_counts))]
                else:
                    trips = range(trip_bound + 1)
                nexts = set()
                for t in trips:
                    layer = {acc}
                    for _ in range(t):
                        layer = {a + b for a in layer for b in body}
                    nexts |= layer
            else:
                nexts = {acc}
            for v in g.succ[u]:
                for a in nexts:
                    walk(v, a)

        walk(g.start, ())
        return res

    return paths(tg)


# ---------------------------------------------------------------- DOT


def symprog_to_dot(sp: SymProgram) -> str:
    """Deterministic DOT; SwitchCase/While as clusters."""
    lines = ["digraph SymProgram {", "  node [shape=box];"]
    counter = [0]

    def nid():
        counter[0] += 1
        return f"i{counter[0]}"

    def emit(lst: list, indent: str, prev):
        for x in lst:
            if isinstance(x, ExecOp):
                me = nid()
                a = ",".join(f"{k}={v}" for k, v in canonical_attrs(x.attrs))
                lines.append(f'{indent}{me} [label="{x.kind.value}#{x.node_id}{chr(92) + "n" + a if a else ""}"];')
            elif isinstance(x, InputFeed):
                me = nid()
                lines.append(f'{indent}{me} [shape=invhouse,label="feed {x.slot[0]}.{x.slot[1]}"];')
            elif isinstance(x, OutputFetch):
                me = nid()
                lines.append(f'{indent}{me} [shape=house,label="fetch #{x.node_id}"];')
            elif isinstance(x, SwitchCase):
                me = nid()
                lines.append(f'{indent}{me} [shape=diamond,label="switch #{x.branch_id}"];')
                for ci, case in enumerate(x.cases):
                    lines.append(f"{indent}subgraph cluster_{me}_{ci} {{")
                    lines.append(f'{indent}  label="case {ci}";')
                    emit(case, indent + "  ", me)
                    lines.append(f"{indent}}}")
            elif isinstance(x, While):
                me = nid()
                lines.append(f'{indent}{me} [shape=diamond,label="while loop{x.loop_id}"];')
                lines.append(f"{indent}subgraph cluster_{me} {{")
                lines.append(f'{indent}  label="loop {x.loop_id}";')
                emit(x.body, indent + "  ", me)
                lines.append(f"{indent}}}")
            elif isinstance(x, UnrolledLoop):
                me = nid()
                lines.append(f'{indent}{me} [shape=diamond,label="unrolled loop{x.loop_id} x{len(x.bodies)}"];')
                for bi, b in enumerate(x.bodies):
                    lines.append(f"{indent}subgraph cluster_{me}_{bi} {{")
                    lines.append(f'{indent}  label="iter {bi}";')
                    emit(b, indent + "  ", me)
                    lines.append(f"{indent}}}")
            else:
                continue
            if prev is not None:
                lines.append(f"{indent}{prev} -> {me};")
            prev = me
        return prev

    emit(sp.body, "  ", None)
    lines.append("}")
    return "\n".join(lines) + "\n"


def count_kind(sp_or_list, cls) -> int:
    lst = sp_or_list.body if isinstance(sp_or_list, SymProgram) else sp_or_list
    c = 0
    for x in lst:
        if isinstance(x, cls):
            c += 1
        if isinstance(x, SwitchCase):
            c += sum(count_kind(cs, cls) for cs in x.cases)
        elif isinstance(x, While):
            c += count_kind(x.body, cls)
        elif isinstance(x, UnrolledLoop):
            c += sum(count_kind(b, cls) for b in x.bodies)
    return c
