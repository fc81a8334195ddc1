"""tcgen05 bf16 GEMM throughput through the C-ABI (CUDA events on the context stream).
python tools/gemm_bench.py [sizes...]  -> JSON lines {m,n,k, ms, tflops, frac_of_measured_bf16}"""

import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2201_09210_b200.b200 import B200Backend  # noqa: E402
from paper_2201_09210_b200.tensor import OpKind, Tensor  # noqa: E402

peak = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["bf16_tflops"] if os.path.exists(
    os.path.join(ROOT, "MEASURED_PEAKS.json")) else 1590.0
be = B200Backend(precision="bf16")
sizes = [int(x) for x in sys.argv[1:]] or [1024, 4096, 8192]
for s in sizes:
    r = np.random.default_rng(s)
    a = Tensor((s, s), r.uniform(-1, 1, (s, s)))
    b = Tensor((s, s), r.uniform(-1, 1, (s, s)))
    ms = be.time_op(OpKind.MATMUL, {}, [a, b], reps=10)
    tf = 2 * s ** 3 / (ms * 1e-3) / 1e12
    print(json.dumps({"m": s, "n": s, "k": s, "ms_incl_bf16_convert": round(ms, 4), "tflops": round(tf, 2),
                      "frac_of_measured_bf16": round(tf / peak, 4)}))
