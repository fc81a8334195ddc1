import os, sys
import numpy as np
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from oracle.kernels import execute_kernel
from paper_2201_09210_b200.b200 import B200Backend
from paper_2201_09210_b200.tensor import OpKind, Tensor
be = B200Backend(precision="bf16")
r = np.random.default_rng(0)
for xs, F in [((4,8,8,64), 32), ((1,16,16,64), 64), ((16,4,4,128), 64), ((1,16,16,64), 1)]:
    x = Tensor(xs, r.standard_normal(xs)); w = Tensor((16*F, xs[3]), r.standard_normal((16*F, xs[3])))
    want = execute_kernel(OpKind.CONV2D_T, {"conv": (4,2,1)}, [x, w])[0].data
    got = be.get(be.exec_op(OpKind.CONV2D_T, {"conv": (4,2,1)}, [x, w])).data
    err = np.linalg.norm(got-want)/np.linalg.norm(want)
    print(xs, F, "err", round(float(err),4))
    if err > 0.05:
        for py in range(2):
            for px in range(2):
                g = got[:, py::2, px::2, :]; wv = want[:, py::2, px::2, :]
                print("  phase", py, px, round(float(np.linalg.norm(g-wv)/np.linalg.norm(wv)),4))
        g = got[0, 0::2, 0::2, :]; wv = want[0, 0::2, 0::2, :]
        e = np.linalg.norm(g-wv, axis=-1)/np.linalg.norm(wv, axis=-1)
        print(np.round(e[:6,:6],2))
print(be.profile_op(OpKind.CONV2D_T, {"conv": (4,2,1)}, [Tensor((128,16,16,128), r.standard_normal((128,16,16,128))), Tensor((1024,128), r.standard_normal((1024,128)))]))
print(be.profile_op(OpKind.CONV2D, {"conv": (4,2,1)}, [Tensor((128,32,32,64), r.standard_normal((128,32,32,64))), Tensor((1024,128), r.standard_normal((1024,128)))]))
print(be.profile_op(OpKind.CONV2D_DW, {"conv": (4,2,1)}, [Tensor((128,32,32,64), r.standard_normal((128,32,32,64))), Tensor((128,16,16,128), r.standard_normal((128,16,16,128)))]))
print(be.profile_op(OpKind.CONV2D, {"conv": (4,2,1)}, [Tensor((128,16,16,128), r.standard_normal((128,16,16,128))), Tensor((2048,256), r.standard_normal((2048,256)))]))
