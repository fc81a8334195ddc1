"""3xTF32 MatMul error against f64 as a function of K (and of COEX_TF32_MAXK / COEX_TF32=0)."""
import json, os, sys
import numpy as np
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2201_09210_b200.b200 import B200Backend
from paper_2201_09210_b200.tensor import OpKind, Tensor
be = B200Backend(precision="fp32")
for K in (768, 3072, 8192, 50257):
    for dist in ("uniform", "gauss"):
        r = np.random.default_rng(K)
        if dist == "uniform":
            a, b = r.uniform(-1, 1, (256, K)), r.uniform(-1, 1, (K, 256))
        else:
            a, b = r.standard_normal((256, K)) * 0.02, r.standard_normal((K, 256))
        got = be.get(be.exec_op(OpKind.MATMUL, {}, [Tensor(a.shape, a), Tensor(b.shape, b)])).data
        want = a @ b
        a32, b32 = a.astype(np.float32).astype(np.float64), b.astype(np.float32).astype(np.float64)
        want32 = a32 @ b32       # exact product of the fp32-rounded operands
        print(json.dumps({"K": K, "dist": dist, "maxk": os.environ.get("COEX_TF32_MAXK"), "tf32": os.environ.get("COEX_TF32", "1"),
                          "err_vs_f64": float(np.linalg.norm(got - want) / np.linalg.norm(want)),
                          "err_vs_fp32_operands": float(np.linalg.norm(got - want32) / np.linalg.norm(want32))}))
be.close()
