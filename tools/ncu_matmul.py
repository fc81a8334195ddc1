"""Launch the C1 forward MatMul [64x784]x[784x128] eagerly a few times (ncu target)."""
import os, sys
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2201_09210_b200.b200 import B200Backend
from paper_2201_09210_b200.tensor import OpKind, Tensor
prec = sys.argv[1] if len(sys.argv) > 1 else "f64"
m, k, n = (int(x) for x in (sys.argv[2:5] if len(sys.argv) > 4 else (64, 784, 128)))
be = B200Backend(precision=prec)
r = np.random.default_rng(0)
a = be.put(Tensor((m, k), r.standard_normal((m, k))))
b = be.put(Tensor((k, n), r.standard_normal((k, n))))
for _ in range(3):
    be.exec_op(OpKind.MATMUL, {}, [a, b])
be.sync()
