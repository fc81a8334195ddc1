import os, sys
import numpy as np
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2201_09210_b200.b200 import B200Backend
from paper_2201_09210_b200.tensor import OpKind, Tensor
be = B200Backend(precision="bf16")
r = np.random.default_rng(0)
xs, F = (1, 8, 8, 64), 8
x = Tensor(xs, r.standard_normal(xs)); w = Tensor((16*F, xs[3]), r.standard_normal((16*F, xs[3])))
got = be.get(be.exec_op(OpKind.CONV2D_T, {"conv": (4,2,1)}, [x, w])).data
np.savez("gpurun_out/dbg_convt.npz", x=x.data, w=w.data, got=got)
