"""TraceGraph: incremental trace merging, coverage, and the co-execution cursor.

Specification: SPEC.md:266-346 (the reference ships no implementation).

Trace events (produced by :mod:`.interp`):
``OpEvent``, ``LoopEnter``, ``LoopIterStart``, ``LoopExit``, ``StepEnd``; op inputs
are ``Handle(id)`` (output of an earlier op this step) or ``External(slot)``.

Equality key of an op node = (kind, canonical attrs, SourceLoc)
**plus the input-kind signature** (which inputs are fed vs produced in-graph).
The extra component makes a node's feed slots static, which the device graph
needs (an InputFeed must not wait for a value the skeleton never sends).

Dataflow (builder decision): SPEC.md:354 requires
ExecOp inputs to "bind to earlier outputs in scope" but the key ignores
dataflow.  Each op node therefore records, per produced input, the set of
candidate producer nodes observed across traces (``cands``).  At run time an
input resolves to the most recently executed candidate (phi semantics for
branch merges and loop-carried values).  The cursor verifies during skeleton
execution that the actual producer is that latest execution, and diverges
otherwise, so co-execution can never compute with the wrong operand.

Merge: follow a matching child; else merge back into the first
(insertion order) key-equal node of the same level that is not an ancestor of
the current node (keeps the graph acyclic); else add a node.  Loops become Loop
nodes whose body graphs merge each iteration Start->End; op-free loops with no
existing Loop node are dropped.
"""

from __future__ import annotations

import copy
import json
from dataclasses import dataclass, field

from .errors import MalformedTrace
from .lang.ast import SourceLoc
from .tensor import OpKind, canonical_attrs

# ---------------------------------------------------------------- trace events


@dataclass(frozen=True)
class Handle:
    id: int


@dataclass(frozen=True)
class External:
    slot: tuple  # (stmt_id, input position) as recorded by the tracer


@dataclass
class OpEvent:
    kind: OpKind
    attrs: dict
    loc: SourceLoc
    inputs: list
    outputs: list
    fetch_after: bool = False
    out_shape: tuple | None = None      # observed shapes: specialisation hints, not part of the key
    in_shapes: tuple | None = None
    in_values: tuple | None = None      # fed host scalars (float) per input, else None

    def key(self) -> tuple:
        return op_key(self.kind, self.attrs, self.loc, self.in_kinds())

    def in_kinds(self) -> tuple:
        return tuple(["h" if type(r) is Handle else "e" for r in self.inputs])


@dataclass(frozen=True)
class LoopEnter:
    loop: int


@dataclass(frozen=True)
class LoopIterStart:
    loop: int


@dataclass(frozen=True)
class LoopExit:
    loop: int


@dataclass(frozen=True)
class StepEnd:
    pass


VARIES = "varies"        # feed_values marker: the fed scalar changed between traces
_UNSEEN = object()


def _bits(v: float) -> bytes:
    import struct
    return struct.pack("<d", v)


def op_key(kind, attrs, loc, in_kinds) -> tuple:
    return ("op", kind.value, canonical_attrs(attrs) if attrs else (), (loc.stmt_id, loc.loop_path), in_kinds)


# ---------------------------------------------------------------- the graph


class IdGen:
    def __init__(self, start: int = 0):
        self.next = start

    def __call__(self) -> int:
        v = self.next
        self.next += 1
        return v


@dataclass
class Node:
    id: int
    typ: str                      # "start" | "end" | "op" | "loop"
    kind: OpKind | None = None
    attrs: dict | None = None
    loc: SourceLoc | None = None
    in_kinds: tuple = ()
    cands: list = field(default_factory=list)   # per input: set of producer node ids ('e' inputs: None)
    fetch: bool = False
    loop_id: int = -1
    body: "TraceGraph | None" = None
    trip_counts: set = field(default_factory=set)
    out_shape: tuple | None = None      # last observed output shape (planner hint)
    feed_shapes: dict = field(default_factory=dict)   # input pos -> last observed fed shape
    feed_values: dict = field(default_factory=dict)   # input pos -> the one host scalar ever fed, or VARIES

    def key(self) -> tuple:
        k = self.__dict__.get("_key")
        if k is None:
            if self.typ == "op":
                k = op_key(self.kind, self.attrs, self.loc, tuple(self.in_kinds))
            elif self.typ == "loop":
                k = ("loop", self.loop_id)
            else:
                k = (self.typ,)
            self.__dict__["_key"] = k
        return k

    def feed_slots(self) -> list:
        return [(self.id, p) for p, k in enumerate(self.in_kinds) if k == "e"]


class TraceGraph:
    """DAG of op/loop nodes between unique Start and End."""

    def __init__(self, ids: IdGen | None = None):
        self.ids = ids if ids is not None else IdGen()
        self.nodes: dict = {}
        self.succ: dict = {}
        self.pred: dict = {}
        self.kids: dict = {}       # node id -> {child key: child id} (child-distinctness makes it a map)
        self.start = self._add(Node(self.ids(), "start"))
        self.end = self._add(Node(self.ids(), "end"))

    def _add(self, n: Node) -> int:
        self.nodes[n.id] = n
        self.succ[n.id] = []
        self.pred[n.id] = []
        self.kids[n.id] = {}
        return n.id

    def add_edge(self, a: int, b: int):
        self.succ[a].append(b)
        self.pred[b].append(a)
        self.kids[a].setdefault(self.nodes[b].key(), b)

    def has_edge(self, a: int, b: int) -> bool:
        return b in self.succ[a]

    def child_with_key(self, a: int, key: tuple):
        return self.kids[a].get(key)

    def ancestors(self, n: int) -> set:
        seen = {n}
        stack = [n]
        while stack:
            for p in self.pred[stack.pop()]:
                if p not in seen:
                    seen.add(p)
                    stack.append(p)
        return seen

    def op_nodes(self) -> list:
        return [n for n in self.nodes.values() if n.typ in ("op", "loop")]

    # ---- whole-hierarchy lookups (node ids are unique across loop bodies)
    def find(self, nid: int):
        if nid in self.nodes:
            return self.nodes[nid]
        for n in self.nodes.values():
            if n.typ == "loop":
                r = n.body.find(nid)
                if r is not None:
                    return r
        return None

    def all_nodes(self):
        for n in self.nodes.values():
            yield n
            if n.typ == "loop":
                yield from n.body.all_nodes()


@dataclass
class MergeReport:
    covered: bool = True
    nodes_added: int = 0
    edges_added: int = 0
    annotations_added: int = 0

    def _finish(self):
        self.covered = self.nodes_added == 0 and self.edges_added == 0 and self.annotations_added == 0
        return self


def _loop_extent(events: list, i: int) -> tuple:
    """For LoopEnter at i: (index of its LoopExit, [indices of its LoopIterStarts], has_ops)."""
    loop = events[i].loop
    depth = 0
    iters = []
    has_ops = False
    j = i + 1
    while j < len(events):
        e = events[j]
        if isinstance(e, OpEvent):
            has_ops = True
        elif isinstance(e, LoopEnter):
            depth += 1
        elif isinstance(e, LoopExit):
            if depth == 0:
                if e.loop != loop:
                    raise MalformedTrace(f"loop {loop} closed by exit of loop {e.loop}")
                return j, iters, has_ops
            depth -= 1
        elif isinstance(e, LoopIterStart) and depth == 0:
            if e.loop != loop:
                raise MalformedTrace(f"iteration marker of loop {e.loop} inside loop {loop}")
            iters.append(j)
        elif isinstance(e, StepEnd):
            break
        j += 1
    raise MalformedTrace(f"loop {loop} is not closed")


def _validate_trace(events: list):
    if not events or not isinstance(events[-1], StepEnd):
        raise MalformedTrace("trace must end with StepEnd")
    if sum(isinstance(e, StepEnd) for e in events) != 1:
        raise MalformedTrace("trace must contain exactly one StepEnd")
    seen = set()
    for e in events:
        if isinstance(e, OpEvent):
            for r in e.inputs:
                if isinstance(r, Handle) and r.id not in seen:
                    raise MalformedTrace(f"handle {r.id} used before it is produced")
            for o in e.outputs:
                if o in seen:
                    raise MalformedTrace(f"handle {o} produced twice")
                seen.add(o)


class _Merger:
    def __init__(self, rep: MergeReport):
        self.rep = rep
        self.hmap: dict = {}          # handle id -> node id

    def seq(self, g: TraceGraph, events: list, i: int) -> int:
        """Merge one Start->End sequence of ``g`` starting at events[i]; returns the index
        of the terminating marker (StepEnd / LoopIterStart / LoopExit of the enclosing loop)."""
        cur = g.start
        while True:
            e = events[i]
            if isinstance(e, OpEvent):
                cur = self.op(g, cur, e)
                i += 1
            elif isinstance(e, LoopEnter):
                cur, i = self.loop(g, cur, events, i)
            else:
                if not g.has_edge(cur, g.end):
                    g.add_edge(cur, g.end)
                    self.rep.edges_added += 1
                return i

    def _locate(self, g: TraceGraph, cur: int, key: tuple, make):
        c = g.child_with_key(cur, key)
        if c is not None:
            return c
        anc = g.ancestors(cur)
        for n in g.nodes.values():
            if n.typ in ("op", "loop") and n.id not in anc and n.key() == key:
                g.add_edge(cur, n.id)
                self.rep.edges_added += 1
                return n.id
        nid = g._add(make())
        g.add_edge(cur, nid)
        self.rep.nodes_added += 1
        self.rep.edges_added += 1
        return nid

    def op(self, g: TraceGraph, cur: int, e: OpEvent) -> int:
        kinds = e.in_kinds()

        def make():
            return Node(g.ids(), "op", e.kind, dict(e.attrs), e.loc, kinds,
                        [set() if k == "h" else None for k in kinds])

        nid = self._locate(g, cur, e.key(), make)
        node = g.nodes[nid]
        for pos, r in enumerate(e.inputs):
            if isinstance(r, Handle):
                prod = self.hmap[r.id]
                if prod not in node.cands[pos]:
                    node.cands[pos].add(prod)
                    self.rep.annotations_added += 1
        if e.fetch_after and not node.fetch:
            node.fetch = True
            self.rep.annotations_added += 1
        if e.out_shape is not None:
            node.out_shape = tuple(e.out_shape)
        if e.in_shapes is not None:
            for pos, k in enumerate(kinds):
                if k == "e":
                    node.feed_shapes[pos] = tuple(e.in_shapes[pos])
        if e.in_values is not None:
            for pos, k in enumerate(kinds):
                if k == "e":
                    v = e.in_values[pos]
                    old = node.feed_values.get(pos, _UNSEEN)
                    if old is _UNSEEN:
                        node.feed_values[pos] = v if v is not None else VARIES
                    elif old is not VARIES and (v is None or _bits(v) != _bits(old)):
                        node.feed_values[pos] = VARIES
        for o in e.outputs:
            self.hmap[o] = nid
        return nid

    def loop(self, g: TraceGraph, cur: int, events: list, i: int) -> tuple:
        lid = events[i].loop
        exit_i, iters, has_ops = _loop_extent(events, i)
        key = ("loop", lid)
        if not has_ops:
            return cur, exit_i + 1                      # op-free loop occurrence: dropped
        nid = self._locate(g, cur, key, lambda: Node(g.ids(), "loop", loop_id=lid, body=TraceGraph(g.ids)))
        node = g.nodes[nid]
        for s in iters:
            self.seq(node.body, events, s + 1)
        trip = len(iters)
        if trip not in node.trip_counts:
            node.trip_counts.add(trip)
            self.rep.annotations_added += 1
        return nid, exit_i + 1


def merge_trace(tg: TraceGraph, trace: list) -> MergeReport:
    """Merge one step's trace into ``tg``."""
    _validate_trace(trace)
    rep = MergeReport()
    m = _Merger(rep)
    end = m.seq(tg, trace, 0)
    if not isinstance(trace[end], StepEnd):
        raise MalformedTrace("unbalanced loop markers")
    return rep._finish()


def covers(tg: TraceGraph, trace: list) -> bool:
    """True iff merging ``trace`` would add nothing; ``tg`` unmodified."""
    return merge_trace(copy.deepcopy(tg), trace).covered


# ---------------------------------------------------------------- cursor


@dataclass(frozen=True)
class CaseDecision:
    branch_id: int
    case_index: int


@dataclass(frozen=True)
class LoopDecision:
    loop_id: int
    cont: bool


@dataclass
class Advance:
    node_id: int
    exec_index: int
    decisions: list


class Diverged(Exception):
    def __init__(self, why: str):
        super().__init__(why)
        self.why = why


@dataclass
class _Frame:
    g: TraceGraph
    cur: int
    loop: Node | None = None      # enclosing Loop node when g is its body
    iters: int = 0
    in_body: bool = False


class Cursor:
    """Online matcher of a running step against the TraceGraph.

    ``advance`` mirrors a dry-run merge: it reports ``Diverged`` at the first
    event a merge would change the graph for (new node, edge, feed/fetch-kind
    mismatch, unseen producer, or a trip count an unrolled loop cannot run).
    Decisions are produced exactly when the structured program consumes them:
    a CaseDecision when leaving a node with out-degree > 1, a LoopDecision
    before each potential iteration of a non-unrolled loop."""

    def __init__(self, tg: TraceGraph, unrolled: dict | None = None):
        self.tg = tg
        self.stack = [_Frame(tg, tg.start)]
        self.pending: list = []         # loop markers of a loop not yet known to contain ops
        self.pending_depth = 0
        self.execs: dict = {}           # node id -> executions so far this step
        self.clock = 0
        self.last: dict = {}            # node id -> clock of its latest execution
        self.handles: dict = {}         # handle id -> (node id, exec index, clock)
        self.unrolled = unrolled or {}  # loop node id -> unrolled trip count

    @property
    def top(self) -> _Frame:
        return self.stack[-1]

    def _leave(self, f: _Frame, to: int, decisions: list):
        succ = f.g.succ[f.cur]
        if len(succ) > 1:
            decisions.append(CaseDecision(f.cur, succ.index(to)))
        f.cur = to

    def _replay_pending(self) -> list:
        """The buffered loop turned out to contain ops: enter it for real."""
        marks, self.pending, self.pending_depth = self.pending, [], 0
        decisions: list = []
        for kind, lid in marks:
            decisions += (self._enter if kind == 0 else self._iter if kind == 1 else self._exit)(lid)
        return decisions

    def advance_op(self, e: OpEvent) -> Advance:
        hids = [r.id if isinstance(r, Handle) else None for r in e.inputs]
        c, k, decisions = self.advance(e.key(), hids, e.outputs[0] if e.outputs else None)
        for o in e.outputs[1:]:
            self.handles[o] = self.handles[e.outputs[0]]
        return Advance(c, k, decisions)

    def advance(self, key: tuple, hids: list, out_hid) -> tuple:
        """Fast path used by the skeleton: ``key`` is the op's equality key, ``hids`` the
        handle id of each produced input (None for fed inputs).  Returns
        (node id, execution index, decisions)."""
        decisions = self._replay_pending() if self.pending else []
        f = self.stack[-1]
        g = f.g
        c = g.kids[f.cur].get(key)
        if c is None:
            raise Diverged(f"no successor of node {f.cur} matches {key[1]}@{key[3][0]}")
        node = g.nodes[c]
        last = self.last
        for pos, h in enumerate(hids):
            if h is not None:
                prod, _, tick = self.handles[h]
                cs = node.cands[pos]
                if len(cs) == 1:
                    if prod not in cs:
                        raise Diverged(f"node {c} input {pos}: unseen producer {prod}")
                else:
                    if prod not in cs:
                        raise Diverged(f"node {c} input {pos}: unseen producer {prod}")
                    best = -1
                    for q in cs:
                        t = last.get(q, -1)
                        if t > best:
                            best = t
                    if last.get(prod) != best:
                        raise Diverged(f"node {c} input {pos}: producer is not the latest candidate")
                if last.get(prod) != tick:
                    raise Diverged(f"node {c} input {pos}: producer is not the latest candidate")
        succ = g.succ[f.cur]
        if len(succ) > 1:
            decisions.append(CaseDecision(f.cur, succ.index(c)))
        f.cur = c
        k = self.execs.get(c, 0)
        self.execs[c] = k + 1
        self.clock += 1
        last[c] = self.clock
        if out_hid is not None:
            self.handles[out_hid] = (c, k, self.clock)
        return c, k, decisions

    def producer_of(self, handle_id: int) -> tuple:
        nid, k, _ = self.handles[handle_id]
        return nid, k

    # Loop markers are buffered until the loop's first op: an occurrence without
    # ops is dropped by the merge, so it must not reach the graph.
    def loop_enter(self, lid: int) -> list:
        self.pending.append((0, lid))
        self.pending_depth += 1
        return []

    def loop_iter(self, lid: int) -> list:
        if self.pending:
            self.pending.append((1, lid))
            return []
        return self._iter(lid)

    def loop_exit(self, lid: int) -> list:
        if self.pending:
            self.pending.append((2, lid))
            self.pending_depth -= 1
            if self.pending_depth == 0:
                self.pending = []        # the whole buffered loop was op-free
            return []
        return self._exit(lid)

    def _enter(self, lid: int) -> list:
        f = self.top
        c = f.g.child_with_key(f.cur, ("loop", lid))
        if c is None:
            raise Diverged(f"no loop {lid} successor at node {f.cur}")
        decisions: list = []
        self._leave(f, c, decisions)
        self.stack.append(_Frame(f.g.nodes[c].body, -1, f.g.nodes[c]))
        return decisions

    def _end_iteration(self, f: _Frame, decisions: list):
        if f.in_body:
            if not f.g.has_edge(f.cur, f.g.end):
                raise Diverged(f"loop {f.loop.loop_id}: iteration ends where the body cannot")
            self._leave(f, f.g.end, decisions)

    def _iter(self, lid: int) -> list:
        f = self.top
        decisions: list = []
        self._end_iteration(f, decisions)
        f.iters += 1
        k = self.unrolled.get(f.loop.id)
        if k is not None:
            if f.iters > k:
                raise Diverged(f"unrolled loop {lid} runs more than {k} iterations")
        else:
            decisions.append(LoopDecision(lid, True))
        f.cur = f.g.start
        f.in_body = True
        return decisions

    def _exit(self, lid: int) -> list:
        f = self.top
        decisions: list = []
        self._end_iteration(f, decisions)
        k = self.unrolled.get(f.loop.id)
        if k is not None:
            if f.iters != k:
                raise Diverged(f"unrolled loop {lid} ran {f.iters} iterations, graph has {k}")
        else:
            decisions.append(LoopDecision(lid, False))
        self.stack.pop()
        return decisions

    def step_end(self) -> list:
        f = self.top
        if len(self.stack) != 1 or self.pending:
            raise MalformedTrace("StepEnd inside a loop")
        if not f.g.has_edge(f.cur, f.g.end):
            raise Diverged("step ends where the graph cannot")
        decisions: list = []
        self._leave(f, f.g.end, decisions)
        return decisions


def cursor_advance(cursor: Cursor, event) -> Advance | Diverged:
    """Functional form of SPEC.md:306 -- returns ``Diverged`` instead of raising."""
    try:
        if isinstance(event, OpEvent):
            return cursor.advance_op(event)
        if isinstance(event, LoopEnter):
            return Advance(-1, 0, cursor.loop_enter(event.loop))
        if isinstance(event, LoopIterStart):
            return Advance(-1, 0, cursor.loop_iter(event.loop))
        if isinstance(event, LoopExit):
            return Advance(-1, 0, cursor.loop_exit(event.loop))
        if isinstance(event, StepEnd):
            return Advance(cursor.tg.end, 0, cursor.step_end())
    except Diverged as d:
        return d
    raise MalformedTrace(f"unknown event {event!r}")


# ---------------------------------------------------------------- DOT / JSON


def _label(n: Node) -> str:
    if n.typ == "op":
        a = ",".join(f"{k}={v}" for k, v in canonical_attrs(n.attrs))
        lab = f"{n.kind.value}@{n.loc.stmt_id}"
        if n.loc.loop_path:
            lab += "/L" + ".".join(str(x) for x in n.loc.loop_path)
        if a:
            lab += f"\\n{a}"
        feeds = [p for p, k in enumerate(n.in_kinds) if k == "e"]
        if feeds:
            lab += "\\nfeed:" + ",".join(str(p) for p in feeds)
        if n.fetch:
            lab += "\\nfetch"
        return lab
    return n.typ.capitalize()


def to_dot(tg: TraceGraph) -> str:
    """Deterministic DOT: loop bodies as nested clusters."""
    lines = ["digraph TraceGraph {", "  node [shape=box];"]

    def emit(g: TraceGraph, indent: str):
        for nid in sorted(g.nodes):
            n = g.nodes[nid]
            if n.typ == "loop":
                trips = ",".join(str(t) for t in sorted(n.trip_counts))
                lines.append(f'{indent}n{nid} [shape=ellipse,label="Loop {n.loop_id}\\ntrips:{trips}"];')
                lines.append(f"{indent}subgraph cluster_{nid} {{")
                lines.append(f'{indent}  label="loop {n.loop_id}";')
                emit(n.body, indent + "  ")
                lines.append(f"{indent}}}")
            else:
                lines.append(f'{indent}n{nid} [label="{_label(n)}"];')
        for a in sorted(g.succ):
            for b in g.succ[a]:
                lines.append(f"{indent}n{a} -> n{b};")

    emit(tg, "  ")
    lines.append("}")
    return "\n".join(lines) + "\n"


TG_JSON_VERSION = 1


def to_json(tg: TraceGraph) -> dict:
    """Versioned serialisation used by trace-dump and golden tests."""

    def enc(g: TraceGraph) -> dict:
        nodes = []
        for nid in sorted(g.nodes):
            n = g.nodes[nid]
            d = {"id": nid, "type": n.typ}
            if n.typ == "op":
                d.update(kind=n.kind.value, attrs=[[k, list(v) if isinstance(v, tuple) else v]
                                                   for k, v in canonical_attrs(n.attrs)],
                         stmt=n.loc.stmt_id, loop_path=list(n.loc.loop_path),
                         inputs=[("feed" if k == "e" else sorted(n.cands[p])) for p, k in enumerate(n.in_kinds)],
                         fetch=n.fetch)
            elif n.typ == "loop":
                d.update(loop=n.loop_id, trip_counts=sorted(n.trip_counts), body=enc(n.body))
            nodes.append(d)
        edges = [[a, b] for a in sorted(g.succ) for b in g.succ[a]]
        return {"start": g.start, "end": g.end, "nodes": nodes, "edges": edges}

    return {"version": TG_JSON_VERSION, "graph": enc(tg)}


def to_json_text(tg: TraceGraph) -> str:
    return json.dumps(to_json(tg), sort_keys=True, separators=(",", ":"))


def check_invariants(tg: TraceGraph):
    """Acyclicity, unique Start/End, reachability, child-distinctness."""

    def chk(g: TraceGraph):
        if g.pred[g.start] or g.succ[g.end]:
            raise AssertionError("Start has preds or End has succs")
        order, state = [], {}

        def dfs(u):
            state[u] = 1
            for v in g.succ[u]:
                if state.get(v) == 1:
                    raise AssertionError("cycle")
                if v not in state:
                    dfs(v)
            state[u] = 2
            order.append(u)

        dfs(g.start)
        if len(state) != len(g.nodes):
            raise AssertionError("node unreachable from Start")
        for u in g.nodes:
            if u != g.end and not g.succ[u]:
                raise AssertionError(f"node {u} cannot reach End")
            keys = [g.nodes[c].key() for c in g.succ[u]]
            if len(keys) != len(set(keys)):
                raise AssertionError(f"children of {u} are not key-distinct")
        for n in g.nodes.values():
            if n.typ == "loop":
                chk(n.body)

    chk(tg)
