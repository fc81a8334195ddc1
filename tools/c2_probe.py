"""Quick C2 co-execution timing: per-step device time (CUDA events) and host stats."""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from bench import make_orch, reach_coexec, timed_steps  # noqa: E402
from paper_2201_09210_b200.b200 import B200Backend  # noqa: E402
from paper_2201_09210_b200.dataset import SyntheticDataset  # noqa: E402
from paper_2201_09210_b200.workloads import C2, dcgan_program  # noqa: E402

prec = sys.argv[1] if len(sys.argv) > 1 else "bf16"
be = B200Backend(precision=prec)
t0 = time.time()
o = make_orch(dcgan_program(steps=100000, **C2), SyntheticDataset(1000), be)
pre = reach_coexec(o)
print("reach coexec", pre, "steps", time.time() - t0, "s")
for _ in range(6):
    o.step()
be.sync()
for k in (2, 20):
    t0 = time.time()
    ms, launches = timed_steps(o, be, k, flush=False)
    be.sync()
    print(f"{k} steps: {ms / k:.3f} ms/step device, wall {1e3 * (time.time() - t0) / k:.3f} ms/step, launches {launches}")
st = o.stats
print("stats", st.counters(), "graph_exec", st.graph_exec_ms, "graph_stall", st.graph_stall_ms,
      "python_exec", st.python_exec_ms, "python_stall", st.python_stall_ms)
