"""Per-kernel-kind share of a C1 co-execution step, from device %globaltimer stamps.

ncu cannot list kernels inside conditional CUDA graphs, so the backend can
stamp every graph kernel (coex_ctx_set_trace).  Each stamp interval (to the
next stamp) is charged to the kernel kind that opened it; for wait kernels the
interval up to their "after wait" stamp is host stall.

    python tools/profile_step.py [--steps 50] [--precision f64]
"""

import argparse
import collections
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from bench import make_orch, reach_coexec  # noqa: E402
from paper_2201_09210_b200.b200 import B200Backend  # noqa: E402
from paper_2201_09210_b200.dataset import SyntheticDataset  # noqa: E402
from paper_2201_09210_b200.workloads import C1, c1_program  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--precision", default="f64")
    ap.add_argument("--out", default=None)
    ap.add_argument("--workload", default="c1", choices=["c1", "c2", "c3", "c4", "c5"])
    a = ap.parse_args()
    be = B200Backend(precision=a.precision)
    if a.workload == "c2":
        from paper_2201_09210_b200.workloads import C2, dcgan_program
        src = dcgan_program(steps=100_000, **C2)
    elif a.workload == "c4":
        from paper_2201_09210_b200.workloads import C4, gpt2_program
        src = gpt2_program(steps=100_000, **C4)
    elif a.workload == "c3":
        from paper_2201_09210_b200.workloads import C3, resnet_program
        src = resnet_program(steps=100_000, **C3)
    elif a.workload == "c5":
        from paper_2201_09210_b200.workloads import C5, music_transformer_program
        src = music_transformer_program(steps=100_000, **C5)
    else:
        src = c1_program(steps=100_000, **C1)
    o = make_orch(src, SyntheticDataset(1000), be)
    reach_coexec(o)
    for _ in range(5):
        o.step()
    be.set_trace(65536)
    agg = collections.defaultdict(float)
    cnt = collections.Counter()
    total = 0.0
    for _ in range(a.steps):
        o.step()
        tr = be.read_trace()
        for (t0, k, aw), (t1, _, _) in zip(tr, tr[1:]):
            name = be.STAMP_KINDS.get(k, str(k))
            if aw:
                name += " (after wait)"
            elif k in (6, 7, 10):
                name += " (host stall)"
            agg[name] += (t1 - t0) / 1e3
            cnt[name] += 1
        total += (tr[-1][0] - tr[0][0]) / 1e3
    rows = sorted(agg.items(), key=lambda kv: -kv[1])
    res = {"steps": a.steps, "us_per_step": total / a.steps,
           "by_kind": [{"kind": k, "us_per_step": v / a.steps, "launches_per_step": cnt[k] / a.steps,
                        "share": v / total} for k, v in rows]}
    print(f"device pass time {total / a.steps:.1f} us/step over {a.steps} steps")
    for r in res["by_kind"]:
        print(f"  {r['us_per_step']:8.2f} us  {r['launches_per_step']:5.1f}x  {100 * r['share']:5.1f}%  {r['kind']}")
    if a.out:
        with open(a.out, "w") as fh:
            json.dump(res, fh, indent=1)
    be.set_trace(0)


if __name__ == "__main__":
    main()
