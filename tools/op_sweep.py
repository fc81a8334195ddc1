"""Per-op parity at a workload's real shapes: every distinct op of one training step
(recorded from an eager imperative run) executed on the B200 in the given precision and
by the CPU oracle (f64, BLAS MATMUL) on the same random inputs; prints the norm-wise
relative error per op, worst first.  Localises which kernel breaks the contract tolerance.

    python tools/op_sweep.py --workload c3 --precision fp32 [--batch 2] [--tol 1e-5]
"""

import argparse
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

from oracle import kernels as OK  # noqa: E402
from paper_2201_09210_b200.b200 import B200Backend  # noqa: E402
from paper_2201_09210_b200.tensor import OpKind, Tensor  # noqa: E402
from paper_2201_09210_b200.workloads import (C2, C3, C4, C5, dcgan_program, gpt2_program,  # noqa: E402
                                             music_transformer_program, resnet_program)
from tools.step_ops import record_step_ops  # noqa: E402

PROGS = {"c2": lambda n, b: dcgan_program(steps=n, **dict(C2, batch=b or C2["batch"])),
         "c3": lambda n, b: resnet_program(steps=n, **dict(C3, batch=b or C3["batch"])),
         "c4": lambda n, b: gpt2_program(steps=n, **dict(C4, batch=b or C4["batch"])),
         "c5": lambda n, b: music_transformer_program(steps=n, **dict(C5, batch=b or C5["batch"]))}
SKIP = {OpKind.RESHAPE, OpKind.READ_VAR, OpKind.ASSIGN_VAR, OpKind.FILL}


def sweep(be, ops, seed=0):
    r = np.random.default_rng(seed)
    rows = []
    OK.FAST_MATMUL = True
    try:
        for (kind, attrs, shapes), count in ops.items():
            if kind in SKIP:
                continue
            ins = [Tensor(s, r.uniform(-1, 1, s)) for s in shapes]
            if kind is OpKind.TO_INDEX and len(shapes) > 1 and shapes[1] == ():
                ins[1] = Tensor((), np.array(1000.0))
            want = OK.execute_kernel(kind, dict(attrs), ins)[0].data
            got = be.get(be.exec_op(kind, dict(attrs), [be.put(t) for t in ins])).data
            den = np.linalg.norm(want)
            err = float(np.linalg.norm(got - want) / den) if den > 0 else float(np.linalg.norm(got))
            rows.append({"kind": kind.name, "attrs": dict(attrs), "shapes": [list(s) for s in shapes],
                         "count": count, "err": err})
    finally:
        OK.FAST_MATMUL = False
    return sorted(rows, key=lambda x: -x["err"])


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--workload", default="c3")
    ap.add_argument("--precision", default="fp32")
    ap.add_argument("--batch", type=int, default=None)
    ap.add_argument("--tol", type=float, default=None)
    ap.add_argument("--out", default=None)
    a = ap.parse_args()
    be = B200Backend(precision=a.precision)
    try:
        nsteps = 2 if a.workload == "c2" else 1
        ops = record_step_ops(be, lambda n: PROGS[a.workload](n, a.batch), nsteps)
        rows = sweep(be, ops)
    finally:
        be.close()
    tol = a.tol if a.tol is not None else {"fp32": 1e-5, "bf16": 2e-2, "f64": 1e-12}[a.precision]
    bad = [x for x in rows if x["err"] > tol]
    print(f"{a.workload} {a.precision}: {len(rows)} distinct ops, {len(bad)} above {tol}")
    for x in rows[:25]:
        print(f"  {x['err']:.3e}  {x['kind']:<20} {x['attrs']} {x['shapes']} x{x['count']}")
    if a.out:
        with open(a.out, "w") as fh:
            json.dump(rows, fh, indent=0)


if __name__ == "__main__":
    main()
