"""Benchmark / parity workloads written in the reference's language.

``c1_program`` is BASELINE.json configs[0]: a tiny MLP on
synthetic 784-d data -- sigmoid hidden layer, MSE loss, hand-written backward
(the language has no autodiff), a data-dependent branch on the
fetched loss, a native call mid-step (``clip``, the numpy stand-in), and a
``choice``-driven variable-trip while loop.
"""

from __future__ import annotations

from .dataset import DatasetSource
from .tensor import Tensor


def c1_program(steps: int = 20, batch: int = 64, hidden: int = 128, din: int = 784, dout: int = 10) -> str:
    n = batch * dout
    return f"""
var w1 = mul(input("w1_init", [{din}, {hidden}]), 0.05)
var w2 = mul(input("w2_init", [{hidden}, {dout}]), 0.1)
steps {steps} {{
  let x = input("x", [{batch}, {din}])
  let y = input("y", [{batch}, {dout}])
  let h = sigmoid(matmul(x, w1))
  let p = matmul(h, w2)
  let d = sub(p, y)
  let loss = mean(mul(d, d))
  let l = item(loss)
  let c = native clip([l], 0.0, 10.0)
  let g = mul(d, {2.0 / n})
  if l > 0.4 {{ g = mul(g, 0.5) }}
  let dw2 = matmul(transpose(h), g)
  let dh = mul(matmul(g, transpose(w2)), mul(h, sub(1.0, h)))
  let dw1 = matmul(transpose(x), dh)
  let lr = 0.5
  let k = 0
  while k < native choice(2, 0) {{ dw1 = mul(dw1, 0.9); k = k + 1 }}
  w1 = sub(w1, mul(dw1, lr))
  w2 = sub(w2, mul(dw2, lr))
  print(l)
}}
"""


C1 = dict(batch=64, hidden=128, din=784, dout=10)


def c1_flops(batch=64, hidden=128, din=784, dout=10) -> int:
    """MatMul FLOPs of one C1 step (forward, backward, and the dw1 scaling ignored)."""
    fwd = 2 * batch * din * hidden + 2 * batch * hidden * dout
    bwd = 2 * hidden * batch * dout + 2 * batch * dout * hidden + 2 * din * batch * hidden
    return fwd + bwd


class InMemoryDataset(DatasetSource):
    """Host-resident tensors served per name in order (cycling) -- the dataset a user
    with real data in host memory would pass; every step's inputs cross PCIe."""

    def __init__(self, records: dict):
        self.records = {k: list(v) for k, v in records.items()}
        self._cursors: dict = {}

    def next(self, name: str, shape, step: int) -> Tensor:
        recs = self.records[name]
        i = self._cursors.get(name, 0)
        self._cursors[name] = i + 1
        return recs[i % len(recs)]

    def snapshot(self) -> dict:
        return dict(self._cursors)

    def restore(self, snap: dict):
        self._cursors = dict(snap)
