"""CPU restatement of the reference kernels (TEST INFRASTRUCTURE, see oracle/__init__.py).

Follows pkg/src/coex/tensor.py:228-291 operation by operation:

* MATMUL (tensor.py:228-236): out starts at +0.0 and accumulates the rounded
  product a[i,k]*b[k,j] for k = 0..K-1 in order -- one rounded add per k.
* SUM / MEAN (tensor.py:239-243, 271-277): sequential row-major sum starting
  from +0.0.  ``np.cumsum`` is a strictly sequential scan; adding +0.0 at the
  end reproduces the +0.0 start for all-(-0.0) inputs.
* ADD/SUB/MUL with rank-0 broadcast, NEG, RELU (np.maximum: NaN kept, -0 -> +0),
  SIGMOID as 1/(1+exp(-x)) with overflow ignored (tensor.py:261-270).
* TRANSPOSE materialised, RESHAPE, FILL, ASSIGN_VAR identity (tensor.py:278-285).
"""

from __future__ import annotations

import numpy as np

from paper_2201_09210_b200.errors import BadAttrs, ShapeMismatch
from paper_2201_09210_b200.tensor import OpKind, Tensor, infer_shape


def matmul_seq(a: np.ndarray, b: np.ndarray) -> np.ndarray:
    m, kk = a.shape
    acc = np.zeros((m, b.shape[1]), dtype=np.float64)
    for k in range(kk):
        acc += a[:, k:k + 1] * b[k:k + 1, :]
    return acc


def sum_seq(x: np.ndarray) -> float:
    flat = np.ascontiguousarray(x, dtype=np.float64).reshape(-1)
    if flat.size == 0:
        return 0.0
    return float(np.cumsum(flat)[-1]) + 0.0


_BINARY = {OpKind.ADD: np.add, OpKind.SUB: np.subtract, OpKind.MUL: np.multiply}


def execute_kernel(kind: OpKind, attrs: dict, inputs: list, var_shapes=None) -> list:
    shapes = [t.shape for t in inputs]
    out_shape = infer_shape(kind, attrs, shapes, var_shapes)[0]
    if kind is OpKind.READ_VAR:
        raise BadAttrs("read_var is executed against a variable store, not as a kernel")
    x = [t.data for t in inputs]
    if kind is OpKind.MATMUL:
        r = matmul_seq(x[0], x[1])
    elif kind in _BINARY:
        r = _BINARY[kind](x[0], x[1])
    elif kind is OpKind.NEG:
        r = np.negative(x[0])
    elif kind is OpKind.RELU:
        r = np.maximum(x[0], 0.0)
    elif kind is OpKind.SIGMOID:
        with np.errstate(over="ignore"):
            r = 1.0 / (1.0 + np.exp(-x[0]))
    elif kind is OpKind.SUM:
        r = np.array(sum_seq(x[0]))
    elif kind is OpKind.MEAN:
        n = inputs[0].size()
        if n == 0:
            raise ShapeMismatch("mean of an empty tensor")
        r = np.array(sum_seq(x[0]) / n)
    elif kind is OpKind.TRANSPOSE:
        r = np.transpose(x[0], attrs["perm"])
    elif kind is OpKind.RESHAPE:
        r = x[0].reshape(attrs["target_shape"])
    elif kind is OpKind.FILL:
        r = np.full(attrs["shape"], attrs["value"], dtype=np.float64)
    elif kind is OpKind.ASSIGN_VAR:
        return [inputs[0]]
    else:  # pragma: no cover
        raise BadAttrs(f"unknown op kind {kind!r}")
    return [Tensor(out_shape, r)]
