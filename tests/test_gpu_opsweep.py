"""Per-op parity at the configs' full shapes (north_star tolerances, literal).

Every distinct op of one training step of C2-C5 -- recorded from an eager imperative run
of the full-width model (C2 batch 8, C3 ResNet-50 at 224x224 batch 2, C4 / C5 the full
decoders at one 1024-token sequence) -- is executed on the B200 in fp32 and bf16 through
the C-ABI (coex_exec_op) and by the f64 oracle (oracle.kernels, BLAS MATMUL) on the same
seeded inputs.  Every op's output must agree norm-wise within 1e-5 (fp32) / 2e-2 (bf16):
this pins each kernel at the bench's dispatch paths (tile widths, split-K, DUO, implicit
convolution gathers, causal tile skipping) -- the end-to-end gradients of
tests/test_gpu_contract.py then only add the problem's own conditioning.
"""

import json
import os

import pytest

from paper_2201_09210_b200.workloads import (C2, C3, C4, C5, dcgan_program, gpt2_program,
                                             music_transformer_program, resnet_program)
from tools.op_sweep import sweep
from tools.step_ops import record_step_ops

pytestmark = pytest.mark.gpu

TOL = {"fp32": 1e-5, "bf16": 2e-2}
CASES = {
    "c2": (lambda n: dcgan_program(steps=n, **dict(C2, batch=8)), 2),
    "c3": (lambda n: resnet_program(steps=n, **dict(C3, batch=2)), 1),
    "c4": (lambda n: gpt2_program(steps=n, **dict(C4, batch=1)), 1),
    "c5": (lambda n: music_transformer_program(steps=n, **dict(C5, batch=1)), 1),
}


@pytest.mark.parametrize("prec", ["fp32", "bf16"])
@pytest.mark.parametrize("case", ["c2", "c3", "c4", "c5"])
def test_every_op_at_full_shape(b200_factory, case, prec):
    be = b200_factory(prec, fresh=True)
    try:
        prog, nsteps = CASES[case]
        ops = record_step_ops(be, prog, nsteps)
        rows = sweep(be, ops)
        launched = be.kernel_count()
    finally:
        be.close()
    assert launched > 0 and len(rows) > 10
    path = os.environ.get("CONTRACT_REPORT")
    if path:
        with open(path, "a") as fh:
            fh.write(json.dumps({"test": f"opsweep[{case}-{prec}]", "ops": len(rows), "worst": rows[:5]}) + "\n")
    bad = [r for r in rows if not r["err"] <= TOL[prec]]
    assert not bad, bad[:5]
