"""Per-op device time of the C2 convolutions with and without the implicit-GEMM lowering."""
import json, os, subprocess, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
code = r'''
import sys, json; sys.path.insert(0, %r)
from tools.step_ops import record_step_ops, profile_ops
from paper_2201_09210_b200.b200 import B200Backend
from paper_2201_09210_b200.tensor import OpKind
from paper_2201_09210_b200.workloads import C2, dcgan_program
import collections
be = B200Backend(precision="bf16")
ops = record_step_ops(be, lambda n: dcgan_program(steps=n, **C2), 2)
ops = collections.Counter({k: v for k, v in ops.items() if k[0] in (OpKind.CONV2D, OpKind.CONV2D_T, OpKind.CONV2D_DW)})
rows = profile_ops(be, ops)
print(json.dumps([[r["kind"], r["shapes"], r["count"], sum(l["ms"] for l in r["launches"])] for r in rows]))
''' % ROOT
res = {}
for mask in ("7", "0"):
    out = subprocess.run([sys.executable, "-c", code], env=dict(os.environ, COEX_IMPLICIT=mask), capture_output=True, text=True)
    res[mask] = json.loads(out.stdout.strip().splitlines()[-1])
tot = {m: 0.0 for m in res}
for a, b in zip(res["7"], res["0"]):
    print(a[0], a[1], a[2], "implicit %.1f us" % (a[3] * 1e3), "explicit %.1f us" % (b[3] * 1e3))
    tot["7"] += a[2] * a[3]; tot["0"] += b[2] * b[3]
print("per pair ms:", tot)
