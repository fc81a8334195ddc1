"""One-layer GPT-2 at C4 width (d=768, 12 heads, T=1024, batch 8) co-executed in bf16 for a
few steps: drives the flash-attention kernels for ncu captures (COEX_CANCEL_EVERY=0 keeps
them top-level graph nodes).

    ncu --kernel-name regex:k_fa_ -c 4 --set full python tools/fa_probe.py
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_2201_09210_b200 import coexec, lang  # noqa: E402
from paper_2201_09210_b200.b200 import B200Backend  # noqa: E402
from paper_2201_09210_b200.dataset import SyntheticDataset  # noqa: E402
from paper_2201_09210_b200.workloads import C4, gpt2_program  # noqa: E402


def main():
    steps = int(os.environ.get("FA_STEPS", "5"))
    src = gpt2_program(steps=steps, **dict(C4, layers=1))
    be = B200Backend(precision="bf16")
    try:
        o = coexec.Orchestrator(lang.parse(src), SyntheticDataset(0), coexec.Mode.coexec, coexec.RunConfig(), be)
        res, st = o.run()
        print("counters", st.counters(), "attn groups", o.compiled.last_plan.n_attn, res.lines[-1:])
    finally:
        be.close()


if __name__ == "__main__":
    main()
