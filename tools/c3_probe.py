"""C3 (ResNet-50 + SDPoint) host/device split per step: wall time of each co-executed step,
graph builds (specialise cache misses) and their cost, device time between stream events."""
import sys
import time

sys.path.insert(0, __file__.rsplit("/tools/", 1)[0])

from bench import make_orch, reach_coexec  # noqa: E402
from paper_2201_09210_b200 import b200 as B  # noqa: E402
from paper_2201_09210_b200.dataset import SyntheticDataset  # noqa: E402
from paper_2201_09210_b200.workloads import C3, resnet_program  # noqa: E402

builds = []
_orig = B.B200Program.specialise


def spec(self):
    n0 = len(self.graphs)
    t = time.perf_counter()
    r = _orig(self)
    if len(self.graphs) != n0:
        builds.append(time.perf_counter() - t)
    return r


B.B200Program.specialise = spec
be = B.B200Backend(precision="bf16")
o = make_orch(resnet_program(steps=100_000, **C3), SyntheticDataset(1000), be)
print("tracing steps", reach_coexec(o), "builds", [round(b, 2) for b in builds], flush=True)
for i in range(12):
    nb = len(builds)
    be.event(0)
    t = time.perf_counter()
    o.step()
    be.event(1)
    wall = time.perf_counter() - t
    dev = be.elapsed_ms(0, 1)
    dl = o.stats.decision_log[-1] if o.stats.decision_log else None
    print(f"step {i}: wall {wall * 1e3:.1f} ms device {dev:.1f} ms builds {len(builds) - nb} "
          f"{[round(b, 2) for b in builds[nb:]]} phase {o.phase} counters {o.stats.counters()} "
          f"replays {o.stats.shape_replays} dec {dl}", flush=True)
prog = o.compiled
for k, (h, plan) in prog.graphs.items():
    print(prog.info(h))
