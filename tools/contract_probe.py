"""Grad-probe parity of one full-width case in one mode (diagnostics for
tests/test_gpu_contract.py): prints per-tensor relative errors against the f64 oracle.

    python tools/contract_probe.py --case c3 --precision fp32 --mode imperative
"""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

import test_gpu_contract as T  # noqa: E402
from contract import compare  # noqa: E402
from oracle import kernels as OK  # noqa: E402
from oracle.cpu_backend import CpuBackend  # noqa: E402
from paper_2201_09210_b200.b200 import B200Backend  # noqa: E402
from test_gpu_coexec import run  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--case", default="c3")
    ap.add_argument("--precision", default="fp32")
    ap.add_argument("--mode", default="imperative")
    ap.add_argument("--env", default="")
    a = ap.parse_args()
    for kv in filter(None, a.env.split(",")):
        k, v = kv.split("=")
        os.environ[k] = v
    src, grads = T.grad_probe(T.CASES[a.case]())
    OK.FAST_MATMUL = True
    ref, _, _ = run(src, a.mode, CpuBackend())
    OK.FAST_MATMUL = False
    be = B200Backend(precision=a.precision)
    try:
        got, st, _ = run(src, a.mode, be)
    finally:
        be.close()
    errs, bad = compare(ref, got, T.TOL[a.precision], grads, T.ZERO.get(a.case))
    items = sorted(errs.items(), key=lambda kv: -kv[1])
    med = sorted(errs.values())[len(errs) // 2]
    print(f"{a.case} {a.precision} {a.mode} {a.env}: {len(bad)} above tol; median {med:.2e}; counters {st.counters()}")
    print("  worst:", " ".join(f"{k}={v:.2e}" for k, v in items[:10]))
    print("  lines:", ref.lines[:4], got.lines[:4])


if __name__ == "__main__":
    main()
