"""Pin the oracle and the host modules against vectors frozen from the REFERENCE
itself (tests/golden/make_golden.py imports /root/reference/pkg/src)."""

import dataclasses
import json
import os

import numpy as np
import pytest

from oracle.kernels import execute_kernel, sum_seq
from paper_2201_09210_b200 import lang, natives, rng
from paper_2201_09210_b200.dataset import SyntheticDataset
from paper_2201_09210_b200.errors import CoexError
from paper_2201_09210_b200.tensor import CostConfig, OpKind, Tensor, infer_shape, kernel_cost
from programs import CORPUS, fuzz_program

G = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")
ARR = np.load(os.path.join(G, "kernels.npz"))
META = json.load(open(os.path.join(G, "kernels_meta.json")))
HOST = json.load(open(os.path.join(G, "host.json")))
FRONT = json.load(open(os.path.join(G, "frontend.json")))


def _attrs(a):
    return {k: tuple(v) if isinstance(v, list) else v for k, v in a.items()}


@pytest.mark.parametrize("m", [m for m in META if m["name"] != "sum_big"], ids=lambda m: m["name"])
def test_oracle_kernels_bitwise(m):
    ins = [Tensor(ARR[f"{m['name']}.in{i}"].shape, ARR[f"{m['name']}.in{i}"]) for i in range(m["nin"])]
    got = execute_kernel(OpKind(m["kind"]), _attrs(m["attrs"]), ins)[0]
    want = ARR[f"{m['name']}.out"]
    assert got.shape == want.shape
    assert got.data.tobytes() == want.tobytes()


def test_oracle_big_sequential_sum():
    x = np.random.default_rng(77).standard_normal(1_000_000)
    assert np.float64(sum_seq(x)).tobytes() == ARR["sum_big.out"].tobytes()


def test_rng_goldens():
    for s, h in HOST["fnv1a64"].items():
        assert rng.fnv1a64(s) == h
    for seed, name, idx, hexv in HOST["draw_at"]:
        assert rng.draw_at(seed, name, idx) == float.fromhex(hexv)


def test_dataset_goldens():
    for seed, name, occ, shape, vals in HOST["dataset"]:
        ds = SyntheticDataset(seed)
        for _ in range(occ):
            ds.next(name, tuple(shape), 0)
        t = ds.next(name, tuple(shape), 0).materialize()
        assert [v.hex() for v in t.data.ravel()] == vals


def test_natives_goldens():
    assert [natives.eval_native("choice", [4, 0], 7, s) for s in range(8)] == HOST["choice_seed7"]
    assert [natives.eval_native("coin", [k], 0, s) for s in range(6) for k in range(3)] == HOST["coin_seed0"]
    assert natives.eval_native("clip", [[-2, 0.5, 9], 0, 1], 0, 0) == HOST["clip"]
    assert natives.eval_native("clip", [[[-2.0, 3.0], [0.25, 1.5]], -1, 1], 0, 0) == HOST["clip_nested"]
    assert [natives.eval_native("mod", [a, b], 0, 0) for a, b in [(7, 3), (-7, 3), (7.5, 2)]] == HOST["mod"]
    assert natives.eval_native("len", [[1, 2, 3]], 0, 0) == HOST["len"]
    for name, err in HOST["native_errors"]:
        args = {"coin": [1.5], "choice": [0, 0], "mod": [1, 0], "len": [3], "nope": []}[name]
        try:
            natives.eval_native(name, args, 0, 0)
            got = None
        except CoexError as e:
            got = type(e).__name__
        assert got == err


def test_infer_shape_goldens():
    for kind, attrs, shapes, want, err in HOST["infer_shape"]:
        a = {k: tuple(v) if isinstance(v, list) else v for k, v in attrs}
        try:
            got = [list(s) for s in infer_shape(OpKind(kind), a, [tuple(s) for s in shapes])]
            assert err is None and got == want
        except CoexError as e:
            assert type(e).__name__ == err


def test_kernel_cost_goldens():
    cfg = CostConfig(base_us={OpKind.MATMUL: 100.0}, per_element_us={OpKind.MATMUL: 1.0})
    assert [kernel_cost(OpKind.MATMUL, [(2, 4)], cfg), kernel_cost(OpKind.RELU, [(9,)], cfg)] == HOST["kernel_cost"]


def _dump(o):
    if dataclasses.is_dataclass(o):
        d = {"_": type(o).__name__}
        for f in dataclasses.fields(o):
            d[f.name] = _dump(getattr(o, f.name))
        if hasattr(o, "loop_path"):
            d["loop_path"] = _dump(o.loop_path)
        return d
    if isinstance(o, (list, tuple)):
        return [_dump(x) for x in o]
    return o


SOURCES = dict(list(CORPUS.items()) + [(f"fuzz{i}", fuzz_program(i)) for i in range(20)])


@pytest.mark.parametrize("name", sorted(FRONT["tokens"]))
def test_frontend_matches_reference(name):
    src = SOURCES[name]
    toks = [[t.kind, t.text, t.line, t.col, t.value] for t in lang.tokenize(src)]
    assert json.loads(json.dumps(toks)) == FRONT["tokens"][name]
    assert json.loads(json.dumps(_dump(lang.parse(src)))) == FRONT["ast"][name]


def test_frontend_errors_match_reference():
    for src, cls, msg in FRONT["errors"]:
        try:
            lang.parse(src)
            got = (None, None)
        except CoexError as e:
            got = (type(e).__name__, str(e))
        assert got == (cls, msg), src
