"""Cancel promptness on the B200 ("after cancel, the pass stops
within one kernel execution"; the overlay is discarded, the committed store is unchanged).

A pass of 256 dependent f64 MatMuls (each ~0.3 ms on the sequential-k parity kernel) is
cancelled a few milliseconds after launch: the straight-line list is cut into guarded
segments (runtime.cu Builder::seq, k_guard), so the pass must stop within about one segment
-- far fewer kernels and far less time than the full pass -- report Cancelled, count only
the kernels that ran, and leave every variable at its committed value.
"""

import time

import numpy as np
import pytest

from paper_2201_09210_b200 import coexec, lang
from paper_2201_09210_b200.coexec import Phase
from paper_2201_09210_b200.dataset import SyntheticDataset

pytestmark = pytest.mark.gpu

DEPTH = 256


def _program(n=512):
    lines = [f"var w = fill([{n}, {n}], 0.0013)", f"var acc = fill([{n}, {n}], 0.0)", "steps 12 {",
             "  let a0 = matmul(w, w)"]
    lines += [f"  let a{i} = matmul(a{i - 1}, w)" for i in range(1, DEPTH)]
    lines += [f"  acc = add(acc, a{DEPTH - 1})", "  print(item(mean(acc)))", "}"]
    return "\n".join(lines) + "\n"


def test_cancel_stops_within_a_segment(b200_factory):
    be = b200_factory("f64", fresh=True)
    try:
        o = coexec.Orchestrator(lang.parse(_program()), SyntheticDataset(0), coexec.Mode.coexec,
                                coexec.RunConfig(), be)
        o.start()
        n = 0
        while o.phase is not Phase.CoExec and n < 10:
            o.step()
            n += 1
        assert o.phase is Phase.CoExec
        o.step()                                   # one co-executed pass: the graph is built
        t0 = time.perf_counter()
        full = be.begin_pass(o.compiled)
        r_full = full.wait()                       # wait() publishes the commit token: commits
        full_s = time.perf_counter() - t0
        before = be.snapshot_vars()

        p = be.begin_pass(o.compiled)
        time.sleep(0.003)
        t1 = time.perf_counter()
        p.cancel()
        r = p.wait()
        cancel_s = time.perf_counter() - t1
        after = be.snapshot_vars()
    finally:
        be.close()
    assert r_full.ops >= DEPTH, r_full
    assert not r.committed
    # stopped within about one guarded segment (64 kernels), not the 256+ of the full pass
    assert r.ops <= r_full.ops // 2, (r.ops, r_full.ops)
    print(f"cancel: {r.ops} of {r_full.ops} kernels, {cancel_s * 1e3:.1f} ms vs a full pass {full_s * 1e3:.1f} ms")
    assert cancel_s < 0.5 * full_s, (cancel_s, full_s)
    for k in before:
        assert np.array_equal(before[k].data, after[k].data), k
