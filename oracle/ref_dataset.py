"""Reference-faithful synthetic dataset (TEST INFRASTRUCTURE, see oracle/__init__.py).

Restates pkg/src/coex/dataset.py:44-51 and rng.py:30-50 exactly as the
reference executes them -- one Python-level xorshift64* draw per element -- so
the CPU baseline pays the reference's real per-element cost.  Values are
identical to the product's device / vectorised expansion (tests pin both)."""

from __future__ import annotations

import numpy as np

from paper_2201_09210_b200.dataset import OCC_MIX, DatasetSource
from paper_2201_09210_b200.errors import EvalError
from paper_2201_09210_b200.rng import MASK64, seeded_state
from paper_2201_09210_b200.tensor import Tensor, shape_size


class RefSyntheticDataset(DatasetSource):
    def __init__(self, seed: int):
        self.seed = seed
        self._cursors: dict = {}

    def next(self, name, shape, step):
        if shape is None:
            raise EvalError(f"input({name!r}): the synthetic dataset needs an explicit shape", step)
        occ = self._cursors.get(name, 0)
        self._cursors[name] = occ + 1
        x = seeded_state(self.seed, name, (occ * OCC_MIX) & MASK64)
        vals = []
        for _ in range(shape_size(shape)):
            x ^= x >> 12
            x = (x ^ (x << 25)) & MASK64
            x ^= x >> 27
            vals.append((((x * 0x2545F4914F6CDD1D) & MASK64) >> 11) * 2.0 ** -53 * 2.0 - 1.0)
        return Tensor(shape, np.asarray(vals))

    def snapshot(self):
        return dict(self._cursors)

    def restore(self, snap):
        self._cursors = dict(snap)
