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
    from paper_2201_09210_b200.workloads import C2, dcgan_program
    be = B200Backend(precision=a.precision)
    ops = record_step_ops(be, lambda n: dcgan_program(steps=n, **C2), 2)
    rows = profile_ops(be, ops)
    agg = by_kernel(rows)
    tot = sum(agg.values())
    print(f"{len(rows)} distinct ops, {sum(ops.values())} op executions per D+G step pair; kernel time {tot:.3f} ms")
    for k, v in agg.items():
        print(f"  {v:8.3f} ms  {100 * v / tot:5.1f}%  {k}")
    for r in sorted(rows, key=lambda r: -r["count"] * sum(l["ms"] for l in r["launches"]))[:25]:
        print(r["count"], r["kind"], r["shapes"], r["attrs"], [(l["kernel"], round(l["ms"] * 1e3, 1)) for l in r["launches"]])
    if a.out:
        with open(a.out, "w") as fh:
            json.dump({"rows": rows, "by_kernel": agg}, fh, indent=1)


if __name__ == "__main__":
    main()
