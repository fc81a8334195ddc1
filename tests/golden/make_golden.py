"""Freeze golden vectors from the REFERENCE implementation (run in the builder
container, where /root/reference exists; the fixtures travel, the reference
does not).  Usage: python tests/golden/make_golden.py

* kernels.npz  -- coex.tensor.execute_kernel (pkg/src/coex/tensor.py:246-291) on
                  seeded inputs and edge cases (signed zeros, NaN, empty, big sums,
                  non-BLAS matmul order); inputs stored or regenerated from a seed.
* host.json    -- coex.rng (fnv1a64, draw_at), coex.dataset.SyntheticDataset
                  (5 (seed, name, occurrence) triples), coex.natives
                  (choice(4,0) steps 0..7 seed 7; coin; clip; mod; len),
                  coex.tensor.infer_shape results / error classes.
* frontend.json -- coex.lang.tokenize / parse dumps of the corpus programs and the
                  error class + message of malformed sources.
"""

import dataclasses
import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, "/root/reference/pkg/src")
sys.path.insert(0, os.path.dirname(HERE))

import coex.dataset as RD  # noqa: E402
import coex.lang as RL  # noqa: E402
import coex.natives as RN  # noqa: E402
import coex.rng as RR  # noqa: E402
import coex.tensor as RT  # noqa: E402
from programs import CORPUS, fuzz_program  # noqa: E402


def kernel_cases():
    r = np.random.default_rng(20260101)

    def rt(*s, scale=1.0):
        return RT.Tensor(s, r.standard_normal(s) * scale)

    K = RT.OpKind
    cases = [
        ("add", {}, [rt(5, 7), rt(5, 7)]), ("add_bcast_r", {}, [rt(5, 7), rt()]), ("add_bcast_l", {}, [rt(), rt(4)]),
        ("sub", {}, [rt(3, 100), rt(3, 100)]), ("mul", {}, [rt(257), rt(257)]), ("mul_bcast", {}, [rt(2, 3), rt()]),
        ("neg", {}, [rt(9, 9)]), ("neg_zero", {}, [RT.Tensor((2,), [0.0, -0.0])]),
        ("relu", {}, [RT.Tensor((7,), [-1.0, -0.0, 0.0, 2.5, float("nan"), -3.0, float("inf")])]),
        ("sigmoid", {}, [RT.Tensor((6,), [0.0, 1.0, -1.0, 800.0, -800.0, 36.5])]),
        ("sum", {}, [rt(64, 10)]), ("sum_zeros", {}, [RT.Tensor((3,), [-0.0, -0.0, -0.0])]),
        ("sum_empty", {}, [RT.Tensor((0,), [])]), ("sum_cancel", {}, [RT.Tensor((4,), [1e16, 1.0, -1e16, 1.0])]),
        ("mean", {}, [rt(33, 17)]), ("mean_scalar", {}, [rt()]),
        ("matmul_identity", {}, [RT.Tensor((2, 2), [[1.0, 2.0], [3.0, 4.0]]), RT.Tensor((2, 2), [[1.0, 0.0], [0.0, 1.0]])]),
        ("matmul", {}, [rt(64, 784), rt(784, 128)]), ("matmul_small", {}, [rt(128, 64), rt(64, 10)]),
        ("matmul_odd", {}, [rt(37, 91), rt(91, 53)]), ("matmul_k0", {}, [rt(3, 0), rt(0, 4)]),
        ("matmul_negzero", {}, [RT.Tensor((1, 2), [[-0.0, 1.0]]), RT.Tensor((2, 1), [[5.0], [-0.0]])]),
        ("matmul_cancel", {}, [RT.Tensor((1, 3), [[1e16, 1.0, -1e16]]), RT.Tensor((3, 1), [[1.0], [1.0], [1.0]])]),
        ("transpose2", {"perm": (1, 0)}, [rt(64, 784)]), ("transpose3", {"perm": (2, 0, 1)}, [rt(3, 4, 5)]),
        ("transpose0", {"perm": ()}, [rt()]),
        ("reshape", {"target_shape": (10, 3)}, [rt(5, 6)]),
        ("fill", {"shape": (4, 5), "value": 0.05}, []), ("fill_scalar", {"shape": (), "value": -2.0}, []),
        ("assign_var", {"var_name": "w"}, [rt(3)]),
    ]
    out = {}
    meta = []
    for name, attrs, ins in cases:
        kind = {"add_bcast_r": K.ADD, "add_bcast_l": K.ADD, "mul_bcast": K.MUL, "neg_zero": K.NEG,
                "sum_zeros": K.SUM, "sum_empty": K.SUM, "sum_cancel": K.SUM, "mean_scalar": K.MEAN,
                "matmul_identity": K.MATMUL, "matmul_small": K.MATMUL, "matmul_odd": K.MATMUL,
                "matmul_k0": K.MATMUL, "matmul_negzero": K.MATMUL, "matmul_cancel": K.MATMUL,
                "transpose2": K.TRANSPOSE, "transpose3": K.TRANSPOSE, "transpose0": K.TRANSPOSE,
                "fill_scalar": K.FILL}.get(name, None) or K(name)
        res = RT.execute_kernel(kind, dict(attrs), ins)[0]
        for i, t in enumerate(ins):
            out[f"{name}.in{i}"] = t.data
        out[f"{name}.out"] = res.data
        meta.append({"name": name, "kind": kind.value, "nin": len(ins),
                     "attrs": {k: list(v) if isinstance(v, tuple) else v for k, v in attrs.items()}})
    # one large sequential sum, regenerated from a seed in the test
    big = np.random.default_rng(77).standard_normal(1_000_000)
    out["sum_big.out"] = RT.execute_kernel(K.SUM, {}, [RT.Tensor(big.shape, big)])[0].data
    meta.append({"name": "sum_big", "kind": "sum", "nin": 1, "attrs": {}, "regen": "default_rng(77).standard_normal(1000000)"})
    return out, meta


def host_goldens():
    g = {}
    g["fnv1a64"] = {s: RR.fnv1a64(s) for s in ["", "x", "native", "w1_init", "ünï"]}
    g["draw_at"] = [[seed, name, idx, RR.draw_at(seed, name, idx).hex()]
                    for seed, name, idx in [(0, "native", 0), (7, "native", 5), (3, "abc", 1000),
                                            (0, "native", 31 * 50 + 2), (123456789, "native", 4096)]]
    trip = []
    for seed, name, occ, shape in [(0, "x", 0, (4,)), (0, "x", 1, (4,)), (1, "x", 0, (4,)), (0, "y", 0, (4,)),
                                   (42, "img", 3, (4,)), (5, "x", 2, (3, 7))]:
        ds = RD.SyntheticDataset(seed)
        for _ in range(occ):
            ds.next(name, shape, 0)
        trip.append([seed, name, occ, list(shape), [v.hex() for v in ds.next(name, shape, 0).data.ravel()]])
    g["dataset"] = trip
    g["choice_seed7"] = [RN.eval_native("choice", [4, 0], 7, s) for s in range(8)]
    g["coin_seed0"] = [RN.eval_native("coin", [k], 0, s) for s in range(6) for k in range(3)]
    g["clip"] = RN.eval_native("clip", [[-2, 0.5, 9], 0, 1], 0, 0)
    g["clip_nested"] = RN.eval_native("clip", [[[-2.0, 3.0], [0.25, 1.5]], -1, 1], 0, 0)
    g["mod"] = [RN.eval_native("mod", [a, b], 0, 0) for a, b in [(7, 3), (-7, 3), (7.5, 2)]]
    g["len"] = RN.eval_native("len", [[1, 2, 3]], 0, 0)
    errs = []
    for name, args in [("coin", [1.5]), ("choice", [0, 0]), ("mod", [1, 0]), ("len", [3]), ("nope", [])]:
        try:
            RN.eval_native(name, args, 0, 0)
            errs.append([name, None])
        except Exception as e:
            errs.append([name, type(e).__name__])
    g["native_errors"] = errs
    K = RT.OpKind
    shp = []
    for kind, attrs, shapes in [(K.MATMUL, {}, [(2, 3), (3, 4)]), (K.SUM, {}, [(5, 7)]),
                                (K.MATMUL, {}, [(2, 3), (4, 4)]), (K.ADD, {}, [(2, 3), ()]),
                                (K.ADD, {}, [(2, 3), (3, 2)]), (K.TRANSPOSE, {"perm": (1, 0)}, [(2, 3)]),
                                (K.TRANSPOSE, {"perm": (0, 0)}, [(2, 3)]), (K.RESHAPE, {"target_shape": (6,)}, [(2, 3)]),
                                (K.RESHAPE, {"target_shape": (7,)}, [(2, 3)]), (K.FILL, {"shape": (2,), "value": 1.0}, []),
                                (K.FILL, {"shape": (2,), "value": 1}, []), (K.NEG, {}, [(2,), (2,)]),
                                (K.MATMUL, {}, [(2,), (2, 2)])]:
        try:
            r = RT.infer_shape(kind, attrs, shapes)
            shp.append([kind.value, [[k, list(v) if isinstance(v, tuple) else v] for k, v in attrs.items()],
                        [list(s) for s in shapes], [list(s) for s in r], None])
        except Exception as e:
            shp.append([kind.value, [[k, list(v) if isinstance(v, tuple) else v] for k, v in attrs.items()],
                        [list(s) for s in shapes], None, type(e).__name__])
    g["infer_shape"] = shp
    cfg = RT.CostConfig(base_us={K.MATMUL: 100.0}, per_element_us={K.MATMUL: 1.0})
    g["kernel_cost"] = [RT.kernel_cost(K.MATMUL, [(2, 4)], cfg), RT.kernel_cost(K.RELU, [(9,)], cfg)]
    return g


def ast_dump(o):
    if dataclasses.is_dataclass(o):
        d = {"_": type(o).__name__}
        for f in dataclasses.fields(o):
            d[f.name] = ast_dump(getattr(o, f.name))
        if hasattr(o, "loop_path"):
            d["loop_path"] = ast_dump(o.loop_path)
        return d
    if isinstance(o, (list, tuple)):
        return [ast_dump(x) for x in o]
    return o


BAD_SOURCES = ["let x = @", "steps 1 { } steps 2 { }", "steps 1 { }\nsteps 2 { }", "let x = 1",
               "steps 0 { }", "steps 1 { var w = 1 }", "steps 1 { y = 1 }", "steps 1 { let a = foo(1) }",
               "steps 1 { let a = add(1) }", "steps 1 { let a = native nope(1) }",
               'steps 1 { let s = "abc }', "steps 1 { let a = reshape(a, 3) }", "steps 1 { while item(x) { } }",
               "if true { }\nsteps 1 { }", "steps 1 { let step = 1 }", "steps 1 { let a = 1 < 2 < 3 }",
               "var a = 1\nvar a = 2\nsteps 1 { }", "steps 1 { let a = fill(1, 2) }", "steps 1 { print(1) }"]


def frontend_goldens():
    f = {"tokens": {}, "ast": {}, "errors": []}
    for name, src in list(CORPUS.items()) + [(f"fuzz{i}", fuzz_program(i)) for i in range(20)]:
        f["tokens"][name] = [[t.kind, t.text, t.line, t.col, t.value] for t in RL.tokenize(src)]
        f["ast"][name] = ast_dump(RL.parse(src))
    for src in BAD_SOURCES:
        try:
            RL.parse(src)
            f["errors"].append([src, None, None])
        except Exception as e:
            f["errors"].append([src, type(e).__name__, str(e)])
    return f


def main():
    arrays, meta = kernel_cases()
    np.savez_compressed(os.path.join(HERE, "kernels.npz"), **arrays)
    with open(os.path.join(HERE, "kernels_meta.json"), "w") as fh:
        json.dump(meta, fh, indent=0)
    with open(os.path.join(HERE, "host.json"), "w") as fh:
        json.dump(host_goldens(), fh, indent=0)
    with open(os.path.join(HERE, "frontend.json"), "w") as fh:
        json.dump(frontend_goldens(), fh)
    print("golden fixtures written to", HERE)


if __name__ == "__main__":
    main()
