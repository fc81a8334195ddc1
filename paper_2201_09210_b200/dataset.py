"""Dataset sources backing ``input(name, shape)``.

Semantics follow the reference (pkg/src/coex/dataset.py:39-95):

* ``SyntheticDataset``: the o-th occurrence of ``input(name)`` is uniform in
  [-1, 1); element e is the e-th xorshift64* draw of the stream seeded with
  ``seed ^ fnv1a64(name) ^ (o * 0x9E3779B97F4A7C15)``.  Cursors are the only
  mutable state; ``snapshot``/``restore`` support step replay.
* ``FileDataset``: JSON-lines records consumed per name in file order.

B200 twist: ``SyntheticDataset.next`` returns a :class:`SyntheticTensor` -- a
lazy descriptor (generator state + shape).  The B200 backend expands it on the
device (``coex_tensor_synth`` / ``coex_pass_feed_synth``), bit-identical to the
reference's Python loop, so a step's input batch never crosses PCIe.  Host code
that needs the numbers (print, natives) calls ``materialize()``, which runs a
vectorised host expansion with the same bits.
"""

from __future__ import annotations

import json

import numpy as np

from .errors import DatasetExhausted, EvalError
from .rng import MASK64, XS_MULT, jump_state, seeded_state, xs_step
from .tensor import Tensor, shape_size

OCC_MIX = 0x9E3779B97F4A7C15


def synth_values(state: int, n: int) -> np.ndarray:
    """Host expansion of ``n`` draws from generator ``state`` mapped to [-1, 1).

    Bit-identical to ``gen.next_unit() * 2.0 - 1.0`` repeated n times
    (dataset.py:49-50): the draws are cut into ``lanes`` contiguous chunks of
    ``rows`` draws; each chunk's first state is reached by the O(log n) GF(2)
    jump-ahead (rng.jump_state) and the chunks then step xorshift64 in lockstep
    on uint64 vectors -- ``rows`` vector steps instead of n scalar ones."""
    out = np.empty(n, dtype=np.float64)
    if n == 0:
        return out
    lanes = max(1, min(4096, n // 32))
    rows = -(-n // lanes)
    starts = np.empty(lanes, dtype=np.uint64)
    x = xs_step(state)
    for i in range(lanes):
        starts[i] = x
        x = jump_state(x, rows)
    states = np.empty((lanes, rows), dtype=np.uint64)
    cur = starts
    s12, s25, s27 = np.uint64(12), np.uint64(25), np.uint64(27)
    for r in range(rows):
        states[:, r] = cur
        cur = cur ^ (cur >> s12)
        cur = cur ^ (cur << s25)
        cur = cur ^ (cur >> s27)
    flat = states.reshape(-1)[:n]
    prod = flat * np.uint64(XS_MULT)
    out[:] = (prod >> np.uint64(11)).astype(np.float64) * (2.0 ** -53) * 2.0 - 1.0
    return out


class SyntheticTensor:
    """Lazy synthetic input: generator ``state`` expands to ``shape`` values."""

    __slots__ = ("state", "shape", "_host")

    def __init__(self, state: int, shape):
        self.state = state & MASK64
        self.shape = tuple(int(d) for d in shape)
        self._host = None

    def size(self) -> int:
        return shape_size(self.shape)

    def rank(self) -> int:
        return len(self.shape)

    def materialize(self) -> Tensor:
        if self._host is None:
            self._host = Tensor._wrap(synth_values(self.state, self.size()).reshape(self.shape))
        return self._host

    @property
    def data(self):
        return self.materialize().data

    def to_nested(self):
        return self.materialize().to_nested()


class DatasetSource:
    def next(self, name: str, shape, step: int):
        raise NotImplementedError

    def snapshot(self) -> dict:
        raise NotImplementedError

    def restore(self, snap: dict):
        raise NotImplementedError


class SyntheticDataset(DatasetSource):
    """Uniform [-1, 1) tensors keyed by (seed, name, occurrence) (dataset.py:39-57)."""

    def __init__(self, seed: int, lazy: bool = True):
        self.seed = seed
        self.lazy = lazy
        self._cursors: dict = {}

    def next(self, name: str, shape, step: int):
        if shape is None:
            raise EvalError(f"input({name!r}): the synthetic dataset needs an explicit shape", step)
        occ = self._cursors.get(name, 0)
        self._cursors[name] = occ + 1
        st = seeded_state(self.seed, name, (occ * OCC_MIX) & MASK64)
        t = SyntheticTensor(st, shape)
        return t if self.lazy else t.materialize()

    def snapshot(self) -> dict:
        return dict(self._cursors)

    def restore(self, snap: dict):
        self._cursors = dict(snap)


class FileDataset(DatasetSource):
    """JSON-lines records ``{"name", "shape", "data"}`` consumed per name (dataset.py:60-95)."""

    def __init__(self, path: str):
        self.path = path
        self._records: dict = {}
        self._cursors: dict = {}
        with open(path, "r", encoding="utf-8") as fh:
            for lineno, raw in enumerate(fh, 1):
                raw = raw.strip()
                if not raw:
                    continue
                try:
                    rec = json.loads(raw)
                    t = Tensor(tuple(rec["shape"]), np.asarray(rec["data"], dtype=float))
                    nm = rec["name"]
                except (KeyError, ValueError, TypeError) as exc:
                    raise EvalError(f"{path}:{lineno}: bad dataset record ({exc})") from exc
                self._records.setdefault(nm, []).append(t)

    def next(self, name: str, shape, step: int):
        recs = self._records.get(name, [])
        i = self._cursors.get(name, 0)
        if i >= len(recs):
            raise DatasetExhausted(f"input({name!r}): dataset exhausted after {i} record(s)", step)
        self._cursors[name] = i + 1
        t = recs[i]
        if shape is not None and t.shape != tuple(shape):
            raise EvalError(f"input({name!r}): record {i} has shape {list(t.shape)}, expected {list(shape)}", step)
        return t

    def snapshot(self) -> dict:
        return dict(self._cursors)

    def restore(self, snap: dict):
        self._cursors = dict(snap)
