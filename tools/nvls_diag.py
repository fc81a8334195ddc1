"""Forced 1-rank data parallelism with and without the GEMM -> all-reduce fusion
(csrc/nvls.cuh): per-variable relative error against the CPU oracle for both runs."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
from oracle.cpu_backend import CpuBackend  # noqa: E402
from paper_2201_09210_b200 import coexec, lang  # noqa: E402
from paper_2201_09210_b200.b200 import B200Backend  # noqa: E402
from paper_2201_09210_b200.dataset import SyntheticDataset  # noqa: E402
from paper_2201_09210_b200.dp import DPGroup  # noqa: E402
from paper_2201_09210_b200.workloads import C2_SMALL, dcgan_program  # noqa: E402
from test_gpu_coexec import run  # noqa: E402

prec = sys.argv[1] if len(sys.argv) > 1 else "bf16"
src = dcgan_program(steps=6, **C2_SMALL)
ref, _, _ = run(src, "coexec", CpuBackend())
for mode in ("none", "0", "1"):
    if mode == "none":
        be = B200Backend(precision=prec)
    else:
        os.environ["COEX_NVLS"] = mode
        be = B200Backend(precision=prec, dp=DPGroup(0, 1, C2_SMALL["batch"], force=True))
    o = coexec.Orchestrator(lang.parse(src), SyntheticDataset(0), coexec.Mode.coexec, coexec.RunConfig(), be)
    got, st = o.run()
    errs = {k: float(np.linalg.norm(got.vars[k].data - t.data) / max(np.linalg.norm(t.data), 1e-30))
            for k, t in ref.vars.items()}
    worst = sorted(errs.items(), key=lambda kv: -kv[1])[:5]
    print(prec, "dp" if mode != "none" else "single", "nvls=" + mode, be.nvls_mode, "worst:",
          [(k, round(v, 4)) for k, v in worst])
    be.close()
