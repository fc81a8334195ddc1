"""Flash-attention kernels (csrc/attn_tc.cuh) at C4's head shape through coex_flash_attn:
device ms per forward / backward and causal TFLOP/s (CUDA events on the context stream).

    python tools/fa_bench.py [BH T reps]      (ncu: ncu -k regex:k_fa_ ... python tools/fa_bench.py 96 1024 1)
"""
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2201_09210_b200.b200 import B200Backend  # noqa: E402
from paper_2201_09210_b200.tensor import Tensor  # noqa: E402

BH, T, reps = (int(x) for x in (sys.argv[1:4] if len(sys.argv) > 3 else (96, 1024, 20)))
be = B200Backend(precision="bf16")
r = np.random.default_rng(0)
q, k, v, do = (be.put(Tensor((BH, T, 64), r.standard_normal((BH, T, 64)))) for _ in range(4))
(o, lse), fwd_ms = be.flash_attention([q, k, v], 0.125, reps=reps)
_, bwd_ms = be.flash_attention([q, k, v, o, do, lse], 0.125, backward=True, reps=reps)
# causal algorithmic flops: forward 2 GEMMs, backward 4 (S recomputed: 5 issued), half the T x T plane
half = BH * T * (T + 128) / 2 * 64 * 2
print(json.dumps({"BH": BH, "T": T, "fwd_ms": round(fwd_ms, 4), "bwd_ms": round(bwd_ms, 4),
                  "fwd_tflops": round(2 * half / fwd_ms / 1e9, 1), "bwd_tflops": round(4 * half / bwd_ms / 1e9, 1),
                  "bwd_issued_tflops": round(5 * half / bwd_ms / 1e9, 1)}))
be.close()
