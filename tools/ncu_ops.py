"""Eager launches of selected C2 ops for ncu captures (one op per invocation argument).

    ncu --set full -k regex:<kernel> python tools/ncu_ops.py <name> [...]
"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2201_09210_b200.b200 import B200Backend  # noqa: E402
from paper_2201_09210_b200.tensor import OpKind, Tensor  # noqa: E402

OPS = {
    "convt_4x4x512": (OpKind.CONV2D_T, {"conv": (4, 2, 1)}, [(128, 4, 4, 512), (4096, 512)]),
    "convt_16x16x128": (OpKind.CONV2D_T, {"conv": (4, 2, 1)}, [(128, 16, 16, 128), (1024, 128)]),
    "conv_32x32x64": (OpKind.CONV2D, {"conv": (4, 2, 1)}, [(128, 32, 32, 64), (1024, 128)]),
    "dw_32x32x64": (OpKind.CONV2D_DW, {"conv": (4, 2, 1)}, [(128, 32, 32, 64), (128, 16, 16, 128)]),
    "conv_16x16x128": (OpKind.CONV2D, {"conv": (4, 2, 1)}, [(128, 16, 16, 128), (2048, 256)]),
    "bn_16x16x128": (OpKind.BATCHNORM, {}, [(128, 16, 16, 128), (128,), (128,)]),
    "bn_4x4x512": (OpKind.BATCHNORM, {}, [(128, 4, 4, 512), (512,), (512,)]),
    "bn_32x32x64": (OpKind.BATCHNORM, {}, [(128, 32, 32, 64), (64,), (64,)]),
    "c3s1_c64": (OpKind.CONV2D, {"conv": (3, 1, 1)}, [(32, 32, 32, 64), (576, 128)]),
    "c3s1_c128": (OpKind.CONV2D, {"conv": (3, 1, 1)}, [(32, 32, 32, 128), (1152, 64)]),
    "c3s1_c256": (OpKind.CONV2D, {"conv": (3, 1, 1)}, [(32, 32, 32, 256), (2304, 32)]),
    "c4s2_c64": (OpKind.CONV2D, {"conv": (4, 2, 1)}, [(32, 64, 64, 64), (1024, 128)]),
    "bndx_8x8x256": (OpKind.BATCHNORM_DX, {}, [(128, 8, 8, 256), (256,), (128, 8, 8, 256)]),
    "mm_8192x128x1": (OpKind.MATMUL, {}, [(8192, 128), (128, 1)]),
    "gemm_8192": (OpKind.MATMUL, {}, [(8192, 8192), (8192, 8192)]),
    "ce_grad": (OpKind.CROSS_ENTROPY_GRAD, {}, [(8192, 50257), (8192,)]),
    "qkt": (OpKind.BMM_NT, {}, [(96, 1024, 64), (96, 1024, 64)]),
    # C4 (GPT-2 small, batch 8 x 1024 tokens): the step's GEMM shapes
    "c4_qkv": (OpKind.MATMUL, {}, [(8192, 768), (768, 768)]),
    "c4_fc1": (OpKind.MATMUL, {}, [(8192, 768), (768, 3072)]),
    "c4_fc2": (OpKind.MATMUL, {}, [(8192, 3072), (3072, 768)]),
    "c4_head": (OpKind.MATMUL, {}, [(8192, 768), (768, 50257)]),
    "c4_dhead": (OpKind.MATMUL, {}, [(8192, 50257), (50257, 768)]),
    "c4_dw768": (OpKind.MATMUL, {}, [(768, 8192), (8192, 768)]),
    "c4_dw3072": (OpKind.MATMUL, {}, [(768, 8192), (8192, 3072)]),
    "c4_dwte": (OpKind.MATMUL, {}, [(50257, 8192), (8192, 768)]),
}

be = B200Backend(precision=os.environ.get("PREC", "bf16"))
r = np.random.default_rng(0)
for name in sys.argv[1:]:
    kind, attrs, shapes = OPS[name]
    ins = [be.put(Tensor(s, r.uniform(-1, 1, s))) for s in shapes]
    for _ in range(3):
        be.exec_op(kind, attrs, ins)
    prof = be.profile_op(kind, attrs, ins, reps=5)
    flops = 0
    if kind in (OpKind.MATMUL,):
        (m, kk), (_, n) = shapes
        flops = 2 * m * n * kk
    gemm_ms = sum(ms for nm, ms in prof if "gemm" in nm or "splitk" in nm)
    print(name, prof, f"gemm {gemm_ms:.4f} ms" + (f" {flops / gemm_ms / 1e9:.1f} TFLOP/s" if flops else ""))
be.sync()
