"""C4 (GPT-2 small) co-execution timing on one B200: per-step device time and host stats.
    python tools/c4_probe.py [precision] [layers]"""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from bench import make_orch, reach_coexec, timed_steps  # noqa: E402
from paper_2201_09210_b200.b200 import B200Backend  # noqa: E402
from paper_2201_09210_b200.dataset import SyntheticDataset  # noqa: E402
from paper_2201_09210_b200.workloads import C4, gpt2_flops, gpt2_program  # noqa: E402

prec = sys.argv[1] if len(sys.argv) > 1 else "bf16"
cfg = dict(C4)
if len(sys.argv) > 2:
    cfg["layers"] = int(sys.argv[2])
be = B200Backend(precision=prec)
t0 = time.time()
o = make_orch(gpt2_program(steps=100000, **cfg), SyntheticDataset(1000), be)
print("prologue", round(time.time() - t0, 1), "s", flush=True)
t0 = time.time()
pre = reach_coexec(o)
print("reach coexec", pre, "steps", round(time.time() - t0, 1), "s", flush=True)
for _ in range(2):
    o.step()
be.sync()
import torch
print("mem GB", torch.cuda.mem_get_info()[1] / 1e9 - torch.cuda.mem_get_info()[0] / 1e9, flush=True)
for k in (3,):
    t0 = time.time()
    ms, launches = timed_steps(o, be, k, flush=False)
    be.sync()
    fl = gpt2_flops(**cfg)
    print(f"{k} steps: {ms / k:.3f} ms/step device, wall {1e3 * (time.time() - t0) / k:.3f} ms/step, "
          f"launches {launches}, {fl / (ms / k * 1e-3) / 1e12:.1f} TFLOP/s (GEMM flops {fl / 1e12:.2f} T)")
st = o.stats
print("stats", st.counters(), "graph_exec", st.graph_exec_ms, "graph_stall", st.graph_stall_ms,
      "python_exec", st.python_exec_ms, "python_stall", st.python_stall_ms)
