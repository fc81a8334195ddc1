import os, sys
import numpy as np
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from oracle.kernels import execute_kernel
from paper_2201_09210_b200.b200 import B200Backend
from paper_2201_09210_b200.tensor import OpKind, Tensor
be = B200Backend(precision="bf16")
r = np.random.default_rng(0)
cases = [((1,18,18,64),(3,1,0),64), ((1,17,16,64),(2,1,0),64), ((1,16,17,64),(2,1,0),64), ((1,16,16,64),(1,1,0),64), ((1,128,128,64),(1,1,0),64), ((1,32,32,64),(1,2,0),64), ((1,16,16,64),(3,1,1),64),
         ((2,16,16,64),(1,1,0),64), ((1,16,16,128),(1,1,0),64), ((8,16,16,64),(4,2,1),128), ((1,16,16,64),(1,1,0),128)]
for xs, (k,s,p), F in cases:
    x = Tensor(xs, r.standard_normal(xs)); w = Tensor((k*k*xs[3], F), r.standard_normal((k*k*xs[3], F)))
    want = execute_kernel(OpKind.CONV2D, {"conv": (k,s,p)}, [x, w])[0].data
    got = be.get(be.exec_op(OpKind.CONV2D, {"conv": (k,s,p)}, [x, w])).data
    err = np.linalg.norm(got-want)/np.linalg.norm(want)
    print(xs, (k,s,p), F, "err", round(float(err),4))
    if err > 0.05:
        g2 = got.reshape(-1, F); w2 = want.reshape(-1, F)
        # which output rows are right?
        rowerr = np.linalg.norm(g2-w2, axis=1)/np.linalg.norm(w2, axis=1)
        print("   bad rows:", np.nonzero(rowerr > 0.05)[0][:20], "of", len(rowerr))
        # try to find for bad row 0 which input row matches (k=1 only)
        if True:
            xr = x.data.reshape(-1, xs[3]) @ w.data[:xs[3]]
            for m in np.nonzero(rowerr > 0.05)[0][:4]:
                d = np.linalg.norm(xr - g2[m], axis=1)
                print("   row", m, "best match input row", int(np.argmin(d)), round(float(d.min()/np.linalg.norm(g2[m])),3))
