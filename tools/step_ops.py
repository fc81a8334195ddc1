"""Per-kernel breakdown of one training step of a workload, from eager re-launches.

The step's op list is recorded from an imperative run (every op of one D step and one
G step for C2), every distinct op is profiled launch by launch through
coex_exec_op_profile (CUDA events on the context stream), and the kernel times are
summed per kernel name, weighted by how often the op occurs in the step.  This is the
evidence for bench.py's ``roofline`` (ncu cannot list kernels inside conditional graph
bodies).

    python tools/step_ops.py [--workload c2] [--precision bf16] [--out json]
"""

import argparse
import collections
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_2201_09210_b200 import coexec, lang  # noqa: E402
from paper_2201_09210_b200.dataset import SyntheticDataset  # noqa: E402
from paper_2201_09210_b200.tensor import OpKind, Tensor, shape_size  # noqa: E402


def record_step_ops(be, src_of_steps, nsteps: int):
    """Multiset of eager ops of steps 1..nsteps (prologue and step 0 subtracted)."""
    def log(n):
        be.op_log = []
        o = coexec.Orchestrator(lang.parse(src_of_steps(n)), SyntheticDataset(0), coexec.Mode.imperative,
                                coexec.RunConfig(), be)
        o.run()
        ops, be.op_log = be.op_log, None
        return collections.Counter((k, tuple(sorted(a.items())), sh) for k, a, sh in ops)
    return log(nsteps + 1) - log(1)


def profile_ops(be, ops: collections.Counter, reps: int = 10):
    import numpy as np
    r = np.random.default_rng(0)
    rows = []
    for (kind, attrs, shapes), count in ops.items():
        if kind in (OpKind.RESHAPE, OpKind.READ_VAR, OpKind.ASSIGN_VAR, OpKind.FILL):
            continue                      # pointer ops / constants: no kernel in the pass graph
        ins = [Tensor(s, r.uniform(-1, 1, s)) for s in shapes]
        launches = be.profile_op(kind, dict(attrs), ins, reps=reps)
        rows.append({"kind": kind.value, "attrs": dict(attrs), "shapes": [list(s) for s in shapes], "count": count,
                     "launches": [{"kernel": k, "ms": ms} for k, ms in launches]})
    return rows


def _conv_geo(kind, attrs, shapes):
    from paper_2201_09210_b200.tensor import infer_shape
    out = infer_shape(kind, attrs, [tuple(x) for x in shapes])[0]
    return out


def launch_work(kind, attrs, shapes, kernel: str, esize: int = 4):
    """Algorithmic work of one launch of an op's lowering: ("flops", F) for the GEMM kernels,
    ("bytes", B) for the memory-bound ones -- compulsory bytes = distinct inputs read + outputs
    written at their storage width (bf16 operand copies count 2 B/elem, fp32 activations 4)."""
    from paper_2201_09210_b200.tensor import flops_of, shape_size
    shapes = [tuple(x) for x in shapes]
    n_in = [shape_size(x) for x in shapes]
    if kind in (OpKind.BMM, OpKind.BMM_NT, OpKind.BMM_TN) and (kernel.startswith("k_gemm_tc")
                                                                or kernel.startswith("k_matmul")):
        return "flops", flops_of(kind, shapes, attrs)
    if kernel.startswith(("k_causal_softmax", "k_softmax_grad", "k_layernorm", "k_ln_dgamma", "k_cross_entropy",
                          "k_rel_skew", "k_bias_add", "k_embed", "k_colsum_wide")):
        # row kernels: every input read once, the output written once
        out = shape_size(_conv_geo(kind, attrs, shapes))
        if kind is OpKind.CROSS_ENTROPY:
            out = 0
        return "bytes", (sum(n_in) + out) * esize
    if kind is OpKind.MATMUL or kind in (OpKind.CONV2D, OpKind.CONV2D_T, OpKind.CONV2D_DW):
        out = _conv_geo(kind, attrs, shapes) if kind is not OpKind.MATMUL else (shapes[0][0], shapes[1][1])
        if kernel.startswith("k_gemm_tc") or kernel.startswith("k_matmul"):
            return "flops", flops_of(kind, shapes, attrs)
        if kernel.startswith("k_im2col"):
            x = shapes[0]
            if kind is OpKind.CONV2D:
                rows, kc = shape_size(out[:3]), shapes[1][0]
            else:                                   # CONV2D_DW: im2col of x over dy's pixels
                rows, kc = shape_size(shapes[1][:3]), shape_size(out[:1])
            return "bytes", n_in[0] * esize + rows * kc * 2
        if kernel.startswith("k_cvt_bf16"):
            if kind is OpKind.CONV2D:
                return "bytes", n_in[1] * (esize + 2)
            if kind is OpKind.CONV2D_DW:
                return "bytes", n_in[1] * (esize + 2)
            return "bytes", (n_in[0] + n_in[1]) * (esize + 2)
        if kernel.startswith("k_col2im"):
            x, w = shapes
            return "bytes", shape_size(x[:3]) * w[0] * esize + shape_size(out) * esize
        if kernel.startswith("k_splitk_reduce"):
            return "bytes", None
    if kernel.startswith("k_colstats"):
        return "bytes", (n_in[0] + (n_in[-1] if kind in (OpKind.BATCHNORM_DX, OpKind.BN_DGAMMA) else 0)) * esize
    if kernel.startswith("k_bn_apply"):
        return "bytes", (2 * n_in[0] + (n_in[2] if kind is OpKind.BATCHNORM_DX else 0)) * esize
    if kernel.startswith("k_elementwise") or kernel.startswith("k_chain") or kernel.startswith("k_transpose") \
            or kernel.startswith("k_reduce"):
        out = shape_size(shapes[0]) if shapes else 0
        return "bytes", (sum(n_in) + out) * esize
    return "bytes", None


def by_family(rows, esize=4):
    """Per kernel family: total ms per step, algorithmic work per step, achieved rate."""
    fam = collections.defaultdict(lambda: {"ms": 0.0, "flops": 0, "bytes": 0, "launches": 0, "unknown_ms": 0.0})
    for r in rows:
        kind = OpKind(r["kind"])
        for ln in r["launches"]:
            name = ln["kernel"]
            key = name.split("E")[0] if name.startswith("k_gemm_tc") else name
            for pre in ("k_gemm_tc", "k_im2col", "k_col2im", "k_colstats", "k_bn_apply", "k_matmul"):
                if name.startswith(pre):
                    key = pre
            f = fam[key]
            f["ms"] += r["count"] * ln["ms"]
            f["launches"] += r["count"]
            what, amount = launch_work(kind, r["attrs"], r["shapes"], name, esize)
            if amount is not None and kind is OpKind.MATMUL and name.startswith("k_cvt_bf16"):
                amount //= max(1, sum(1 for x in r["launches"] if x["kernel"].startswith("k_cvt_bf16")))
            if amount is None:
                f["unknown_ms"] += r["count"] * ln["ms"]
            elif what == "flops":
                f["flops"] += r["count"] * amount
            else:
                f["bytes"] += r["count"] * amount
    return dict(sorted(fam.items(), key=lambda kv: -kv[1]["ms"]))


def by_kernel(rows):
    agg = collections.defaultdict(float)
    for r in rows:
        for ln in r["launches"]:
            agg[ln["kernel"]] += r["count"] * ln["ms"]
    return dict(sorted(agg.items(), key=lambda kv: -kv[1]))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--workload", default="c2")
    ap.add_argument("--precision", default="bf16")
    ap.add_argument("--out", default=None)
    a = ap.parse_args()
    from paper_2201_09210_b200.b200 import B200Backend
    from paper_2201_09210_b200.workloads import C2, C4, C5, dcgan_program, gpt2_program, music_transformer_program
    be = B200Backend(precision=a.precision)
    if a.workload == "c4":
        ops = record_step_ops(be, lambda n: gpt2_program(steps=n, **C4), 1)
    elif a.workload == "c3":
        from paper_2201_09210_b200.workloads import C3, resnet_program
        ops = record_step_ops(be, lambda n: resnet_program(steps=n, **C3), 1)
    elif a.workload == "c5":
        ops = record_step_ops(be, lambda n: music_transformer_program(steps=n, **C5), 1)
    else:
        ops = record_step_ops(be, lambda n: dcgan_program(steps=n, **C2), 2)
    rows = profile_ops(be, ops, reps=int(os.environ.get("STEP_OPS_REPS", "10")))
    agg = by_kernel(rows)
    tot = sum(agg.values())
    print(f"{len(rows)} distinct ops, {sum(ops.values())} op executions per step(s); kernel time {tot:.3f} ms")
    for k, v in agg.items():
        print(f"  {v:8.3f} ms  {100 * v / tot:5.1f}%  {k}")
    for r in sorted(rows, key=lambda r: -r["count"] * sum(l["ms"] for l in r["launches"]))[:25]:
        print(r["count"], r["kind"], r["shapes"], r["attrs"], [(l["kernel"], round(l["ms"] * 1e3, 1)) for l in r["launches"]])
    if a.out:
        with open(a.out, "w") as fh:
            json.dump({"rows": rows, "by_kernel": agg}, fh, indent=1)


if __name__ == "__main__":
    main()
