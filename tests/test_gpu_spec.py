"""Speculative constants: a host scalar that was constant while tracing is baked into the
graph; when it later changes, the step is replayed inline (shape_replays, not a divergence)
and the program is respecialised with that slot fed.  Results stay bit-identical."""

import pytest

from oracle.cpu_backend import CpuBackend
from paper_2201_09210_b200 import coexec, lang
from paper_2201_09210_b200.b200 import B200Backend
from paper_2201_09210_b200.dataset import SyntheticDataset

pytestmark = pytest.mark.gpu

SRC = """
var w = fill([4], 1.0)
steps 14 {
  let x = input("x", [4])
  let lr = 0.125
  if step > 6 { lr = 0.25 + step * 0.0 }
  if step > 9 { lr = step * 0.01 }
  w = sub(w, mul(add(x, w), lr))
  print(sum(w))
}
"""


def test_constant_miss_replays_and_respecialises():
    ref, ref_st = coexec.run(lang.parse(SRC), SyntheticDataset(0), "coexec", backend=CpuBackend())
    be = B200Backend(precision="f64")
    try:
        got, st = coexec.run(lang.parse(SRC), SyntheticDataset(0), "coexec", backend=be)
    finally:
        be.close()
    assert got.lines == ref.lines
    assert {k: v.data.tobytes() for k, v in got.vars.items()} == {k: v.data.tobytes() for k, v in ref.vars.items()}
    assert st.counters() == ref_st.counters()
    assert st.shape_replays == 1          # miss at step 7; afterwards the slot is fed every step
