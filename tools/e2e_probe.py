"""Per-step view of bench.py's e2e leg (host-resident inputs through the public API):
device ms per step, counters, shape replays and graph builds -- for diagnosing an e2e figure
that departs from the device-resident one."""
import argparse
import sys
import time

sys.path.insert(0, __file__.rsplit("/tools/", 1)[0])

import bench  # noqa: E402
from paper_2201_09210_b200.b200 import B200Backend  # noqa: E402
from paper_2201_09210_b200.workloads import InMemoryDataset  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--workload", default="c4")
ap.add_argument("--steps", type=int, default=12)
a = ap.parse_args()
args = argparse.Namespace(workload=a.workload, precision="bf16")
src, dataset, recs, h2d, cfg, gb = bench.workload_setup(args, 1)
be = B200Backend(precision="bf16")
o = bench.make_orch(src, InMemoryDataset(recs), be)
print("reach", bench.reach_coexec(o), "settle", bench.settle(o), flush=True)
for i in range(a.steps):
    graphs = len(getattr(o.compiled, "graphs", {}) or {})
    be.event(0)
    t = time.perf_counter()
    o.step()
    be.event(1)
    print(f"step {i}: wall {(time.perf_counter() - t) * 1e3:.1f} ms device {be.elapsed_ms(0, 1):.1f} ms "
          f"counters {o.stats.counters()} shape_replays {o.stats.shape_replays} "
          f"graphs {graphs}->{len(getattr(o.compiled, 'graphs', {}) or {})} dec {o.stats.decision_log[-1] if o.stats.decision_log else None}",
          flush=True)
