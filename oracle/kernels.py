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

Extension op set (configs C2-C5, SURVEY §2.4 / §8(a) row a*): the reference has no
such ops, so these are the builder's f64 definitions -- parity UNPINNED by the
reference; written in tensor.py's style (explicit orders):

* CONV2D = MATMUL(im2col(x), w) with the im2col column order (ky, kx, c) and
  zero padding; CONV2D_T = col2im(MATMUL(x, w^T)) summing the (ky, kx)
  contributions in ascending order from +0.0; CONV2D_DW =
  MATMUL(im2col(x)^T, dy) (sequential over output pixels).
* BATCHNORM / BATCHNORM_DX / BN_DGAMMA / SUM_ROWS: per-channel (last axis)
  statistics over all leading rows, sequential row order from +0.0; biased
  variance of the centred values, eps = 1e-5.
* TANH, LEAKY_RELU (slope 0.2), RELU_GRAD, LEAKY_RELU_GRAD, BCE_TERM
  (max(x,0) - x*t + log1p(exp(-|x|))) elementwise.
* C4 (GPT-2): TO_INDEX(u, V) = clip(floor((u+1)/2*V), 0, V-1); EMBEDDING row gather
  (ids clipped to the table); EMBEDDING_DW scatter-add in row order from +0.0;
  LAYERNORM / LAYERNORM_DX / LN_DGAMMA over the last axis (sequential row sums,
  eps 1e-5); BIAS_ADD (last-axis broadcast); GELU (tanh approximation) and its
  derivative; BMM / BMM_NT / BMM_TN = per-batch MATMUL (sequential k) of a.b,
  a.b^T, a^T.b; CAUSAL_SOFTMAX(x, scale): row softmax of scale*x over j <= i of
  each trailing [T, T] block (masked entries 0, max-subtracted, exp then
  sequential sum); SOFTMAX_GRAD(y, dy, scale) = scale*y*(dy - sum_j dy*y);
  CROSS_ENTROPY(logits, ids) = mean over rows of logsumexp - logit[id];
  CROSS_ENTROPY_GRAD = (softmax - onehot) / R.
* C5 (Music Transformer): REL_SKEW(x)[i, j] = x[i, T-1-i+j] for j <= i else 0 (the
  relative-attention skew of Huang et al.: column T-1-(i-j) of Q.E_r^T holds distance
  j-i); REL_UNSKEW is its adjoint: dx[i, m] = dy[i, m-(T-1)+i] for m >= T-1-i else 0.
* C3 (ResNet-50 / SDPoint): CONV2D_DX(dy, w, x) = col2im(MATMUL(dy, w^T)) onto x's
  geometry (conv2d's input gradient; unlike CONV2D_T it also covers strides whose
  forward rounding left input rows without a window); MAXPOOL (-inf padding, the first
  maximum in (ky, kx) order wins) and MAXPOOL_GRAD (dy routed to that argmax, summed over
  windows in ascending (oy, ox) order from +0.0); AVGPOOL = (window sum in (ky, kx) order,
  zero padding) / k^2; AVGPOOL_GRAD = (sum of covering dy in (oy, ox) order) / k^2;
  GLOBAL_AVGPOOL = (row-major sum over H, W) / (H*W); GLOBAL_AVGPOOL_GRAD = dy / (H*W).
* General: SQRT (IEEE, NaN for negatives), DIV (IEEE, rank-0 broadcast) -- Adam's update;
  SLICE(x, [axis, start, length]), CONCAT(a, b, [axis]); SUM_AXIS(x, [axis]) = sequential sum
  along the axis from +0.0.
"""

from __future__ import annotations

import numpy as np

from paper_2201_09210_b200.errors import BadAttrs, ShapeMismatch
from paper_2201_09210_b200.tensor import (BN_EPS, GELU_C, LEAKY_SLOPE, LN_EPS, OpKind, Tensor,
                                          infer_shape)


# Tolerance-mode switch (tests only): when True, MATMUL and every product built on it
# (conv, bmm) use numpy's BLAS f64 product instead of the sequential-k loop.  The two
# differ by f64 rounding in the summation order only (<= ~K * 2^-53 relative, pinned by
# tests/test_ext_oracle_cpu.py::test_fast_matmul_matches_sequential), which is 8+ orders
# of magnitude below the fp32 (1e-5) and bf16 (2e-2) bars it is used to check; the
# bit-exact f64 parity tests never set it.
FAST_MATMUL = False


# Host threads for the sequential-k product (bench.py's CPU reference arm sets it to the
# host's core count).  Output tiles are independent: every element still accumulates
# a[i,0]*b[0,j], a[i,1]*b[1,j], ... in k order from +0.0, so the result is bit-identical to
# the single-threaded loop (tests/test_ext_oracle_cpu.py::test_threaded_matmul_bitwise).
THREADS = 1
_POOL = None


def _seq_tile(a, b, acc, r0, r1, c0, c1):
    at = np.ascontiguousarray(a[r0:r1].T)          # k-major rows of the tile's A block
    blk = acc[r0:r1, c0:c1]
    tmp = np.empty_like(blk)
    for k in range(a.shape[1]):
        np.multiply(at[k][:, None], b[k:k + 1, c0:c1], out=tmp)
        blk += tmp


def matmul_seq(a: np.ndarray, b: np.ndarray) -> np.ndarray:
    if FAST_MATMUL:
        return np.matmul(a, b) + 0.0
    m, kk = a.shape
    n = b.shape[1]
    acc = np.zeros((m, n), dtype=np.float64)
    if THREADS > 1 and m * n >= 2 * 65536:
        global _POOL
        if _POOL is None or _POOL._max_workers != THREADS:
            from concurrent.futures import ThreadPoolExecutor
            _POOL = ThreadPoolExecutor(THREADS)
        # one large block per thread (the k loop's numpy calls then run long enough between
        # GIL handoffs to overlap): split rows when there are enough, else columns
        t = min(THREADS, max(1, m * n // 65536))       # blocks of >= 64 Ki outputs
        if m >= 4 * t:
            e = [m * i // t for i in range(t + 1)]
            tiles = [(e[i], e[i + 1], 0, n) for i in range(t) if e[i] < e[i + 1]]
        else:
            e = [n * i // t for i in range(t + 1)]
            tiles = [(0, m, e[i], e[i + 1]) for i in range(t) if e[i] < e[i + 1]]
        list(_POOL.map(lambda t: _seq_tile(a, b, acc, *t), tiles))
        return acc
    for k in range(kk):
        acc += a[:, k:k + 1] * b[k:k + 1, :]
    return acc


def sum_seq(x: np.ndarray) -> float:
    flat = np.ascontiguousarray(x, dtype=np.float64).reshape(-1)
    if flat.size == 0:
        return 0.0
    return float(np.cumsum(flat)[-1]) + 0.0


def im2col(x: np.ndarray, k: int, s: int, p: int) -> np.ndarray:
    """[N,H,W,C] -> [N*Ho*Wo, k*k*C], column (ky, kx, c), zero padding."""
    n, h, w, c = x.shape
    ho, wo = (h + 2 * p - k) // s + 1, (w + 2 * p - k) // s + 1
    xp = np.zeros((n, h + 2 * p, w + 2 * p, c), dtype=np.float64)
    xp[:, p:p + h, p:p + w, :] = x
    cols = np.empty((n, ho, wo, k, k, c), dtype=np.float64)
    for ky in range(k):
        for kx in range(k):
            cols[:, :, :, ky, kx, :] = xp[:, ky:ky + s * (ho - 1) + 1:s, kx:kx + s * (wo - 1) + 1:s, :]
    return cols.reshape(n * ho * wo, k * k * c)


def col2im(cols: np.ndarray, x_shape, k: int, s: int, p: int, out_shape) -> np.ndarray:
    """Adjoint of im2col for conv2d_t: cols [N*H*W, k*k*F] -> [N,Ho,Wo,F]; output
    (oy, ox) sums cols[(iy, ix), (ky, kx)] with oy = iy*s - p + ky, (ky, kx) ascending."""
    n, h, w, _ = x_shape
    _, ho, wo, f = out_shape
    c6 = cols.reshape(n, h, w, k, k, f)
    out = np.zeros((n, ho, wo, f), dtype=np.float64)
    for ky in range(k):
        for kx in range(k):
            # input pixel iy lands on output row iy*s - p + ky
            oy0, ox0 = ky - p, kx - p
            iy = [i for i in range(h) if 0 <= i * s + oy0 < ho]
            ix = [i for i in range(w) if 0 <= i * s + ox0 < wo]
            if not iy or not ix:
                continue
            iy_lo, iy_hi, ix_lo, ix_hi = iy[0], iy[-1] + 1, ix[0], ix[-1] + 1
            oys = slice(iy_lo * s + oy0, (iy_hi - 1) * s + oy0 + 1, s)
            oxs = slice(ix_lo * s + ox0, (ix_hi - 1) * s + ox0 + 1, s)
            out[:, oys, oxs, :] += c6[:, iy_lo:iy_hi, ix_lo:ix_hi, ky, kx, :]
    return out + 0.0


def col_sum_seq(x2: np.ndarray) -> np.ndarray:
    """Per-column sum over rows in row order from +0.0 (np.cumsum along axis 0 is sequential)."""
    if x2.shape[0] == 0:
        return np.zeros(x2.shape[1])
    return np.cumsum(x2, axis=0)[-1] + 0.0


def bn_stats(x2: np.ndarray):
    r = x2.shape[0]
    mean = col_sum_seq(x2) / r
    d = x2 - mean
    var = col_sum_seq(d * d) / r
    rstd = 1.0 / np.sqrt(var + BN_EPS)
    return d, rstd


def bn_sync(kind, x, global_rows: float, allreduce) -> np.ndarray:
    """Synchronised batch norm of one rank's row shard (data parallel; the device's
    k_colstats raw mode + all-reduce + k_bn_finalize): rank-local column sums of x, x^2, dy,
    dy*x summed over the ranks by ``allreduce``, statistics over the GLOBAL batch
    (``global_rows``), then the local rows normalised with them.  Equals BATCHNORM /
    BATCHNORM_DX / BN_DGAMMA of the concatenated global batch up to summation order."""
    c = x[0].shape[-1]
    x2 = x[0].reshape(-1, c)
    dy = None if kind is OpKind.BATCHNORM else x[-1].reshape(-1, c)
    raw = np.zeros((4, c))
    raw[0] = col_sum_seq(x2)
    raw[1] = col_sum_seq(x2 * x2)
    if dy is not None:
        raw[2] = col_sum_seq(dy)
        raw[3] = col_sum_seq(dy * x2)
    raw = np.asarray(allreduce(raw.reshape(-1), False)).reshape(4, c)
    r = float(global_rows)
    mean = raw[0] / r
    var = np.maximum(raw[1] / r - mean * mean, 0.0)
    rstd = 1.0 / np.sqrt(var + BN_EPS)
    xhat = (x2 - mean) * rstd
    if kind is OpKind.BATCHNORM:
        return ((xhat * x[1]) + x[2]).reshape(x[0].shape)
    sdx = rstd * (raw[3] - mean * raw[2])                 # global sum(dy * xhat)
    if kind is OpKind.BN_DGAMMA:
        return sdx
    t = dy - raw[2] / r
    t = t - xhat * (sdx / r)
    return (t * (x[1] * rstd)).reshape(x[0].shape)


def _windows(h, w, k, s, p, ho, wo):
    """(oy, ox, [(ky, kx, iy, ix) in (ky, kx) order, in-bounds taps only])."""
    for oy in range(ho):
        for ox in range(wo):
            taps = [(ky, kx, oy * s - p + ky, ox * s - p + kx) for ky in range(k) for kx in range(k)]
            yield oy, ox, [t for t in taps if 0 <= t[2] < h and 0 <= t[3] < w]


def pool_kernel(kind: OpKind, attrs: dict, x: list, out_shape) -> np.ndarray:
    if kind is OpKind.GLOBAL_AVGPOOL:
        n, h, w, c = x[0].shape
        acc = np.zeros((n, c))
        for i in range(h):
            for j in range(w):
                acc = acc + x[0][:, i, j, :]
        return acc / (h * w)
    if kind is OpKind.GLOBAL_AVGPOOL_GRAD:
        n, h, w, c = x[0].shape
        return np.broadcast_to((x[1] / (h * w))[:, None, None, :], (n, h, w, c)).copy()
    k, s, p = attrs["conv"]
    n, h, w, c = x[0].shape
    if kind in (OpKind.MAXPOOL, OpKind.AVGPOOL):
        _, ho, wo, _ = out_shape
        out = np.zeros(out_shape)
        for oy, ox, taps in _windows(h, w, k, s, p, ho, wo):
            if kind is OpKind.MAXPOOL:
                m = np.full((n, c), -np.inf)
                for _, _, iy, ix in taps:
                    m = np.where(x[0][:, iy, ix, :] > m, x[0][:, iy, ix, :], m)
                out[:, oy, ox, :] = m
            else:
                acc = np.zeros((n, c))
                for _, _, iy, ix in taps:
                    acc = acc + x[0][:, iy, ix, :]
                out[:, oy, ox, :] = acc / (k * k)
        return out
    dy = x[1]
    _, ho, wo, _ = dy.shape
    acc = np.zeros((n, h, w, c))
    for oy, ox, taps in _windows(h, w, k, s, p, ho, wo):   # ascending (oy, ox)
        if kind is OpKind.AVGPOOL_GRAD:
            for _, _, iy, ix in taps:
                acc[:, iy, ix, :] = acc[:, iy, ix, :] + dy[:, oy, ox, :]
            continue
        m = np.full((n, c), -np.inf)
        arg = np.zeros((n, c), dtype=np.int64)
        for t, (_, _, iy, ix) in enumerate(taps):
            better = x[0][:, iy, ix, :] > m
            m = np.where(better, x[0][:, iy, ix, :], m)
            arg = np.where(better, t, arg)
        for t, (_, _, iy, ix) in enumerate(taps):
            acc[:, iy, ix, :] = acc[:, iy, ix, :] + np.where(arg == t, dy[:, oy, ox, :], 0.0)
    if kind is OpKind.AVGPOOL_GRAD:
        return acc / (k * k)
    return acc


def ext_kernel(kind: OpKind, attrs: dict, x: list, out_shape) -> np.ndarray:
    if kind is OpKind.SQRT:
        with np.errstate(invalid="ignore"):
            return np.sqrt(x[0])
    if kind is OpKind.SLICE:
        ax, start, length = attrs["dims"]
        return np.take(x[0], np.arange(start, start + length), axis=ax).reshape(out_shape)
    if kind is OpKind.CONCAT:
        return np.concatenate([x[0], x[1]], axis=attrs["dims"][0])
    if kind is OpKind.SUM_AXIS:
        ax = attrs["dims"][0]
        acc = np.zeros(out_shape)
        for j in range(x[0].shape[ax]):
            acc = acc + np.take(x[0], j, axis=ax)
        return acc + 0.0
    if kind in (OpKind.MAXPOOL, OpKind.MAXPOOL_GRAD, OpKind.AVGPOOL, OpKind.AVGPOOL_GRAD, OpKind.GLOBAL_AVGPOOL,
                OpKind.GLOBAL_AVGPOOL_GRAD):
        return pool_kernel(kind, attrs, x, out_shape)
    if kind is OpKind.CONV2D_DX:
        k, s, p = attrs["conv"]
        f = x[0].shape[3]
        cols = matmul_seq(x[0].reshape(-1, f), np.ascontiguousarray(x[1].T))
        return col2im(cols, x[0].shape, k, s, p, out_shape)
    if kind is OpKind.CONV2D:
        k, s, p = attrs["conv"]
        return matmul_seq(im2col(x[0], k, s, p), x[1]).reshape(out_shape)
    if kind is OpKind.CONV2D_T:
        k, s, p = attrs["conv"]
        n, h, w, c = x[0].shape
        cols = matmul_seq(x[0].reshape(n * h * w, c), np.ascontiguousarray(x[1].T))
        return col2im(cols, x[0].shape, k, s, p, out_shape)
    if kind is OpKind.CONV2D_DW:
        k, s, p = attrs["conv"]
        a = im2col(x[0], k, s, p)
        f = x[1].shape[3]
        return matmul_seq(np.ascontiguousarray(a.T), x[1].reshape(-1, f))
    if kind in (OpKind.BATCHNORM, OpKind.BATCHNORM_DX, OpKind.BN_DGAMMA, OpKind.SUM_ROWS):
        c = x[0].shape[-1]
        x2 = x[0].reshape(-1, c)
        if kind is OpKind.SUM_ROWS:
            return col_sum_seq(x2)
        d, rstd = bn_stats(x2)
        xhat = d * rstd
        if kind is OpKind.BATCHNORM:
            return ((xhat * x[1]) + x[2]).reshape(out_shape)
        dy = x[-1].reshape(-1, c)
        if kind is OpKind.BN_DGAMMA:
            return col_sum_seq(dy * xhat)
        r = x2.shape[0]
        t = dy - col_sum_seq(dy) / r
        t = t - xhat * (col_sum_seq(dy * xhat) / r)
        return (t * (x[1] * rstd)).reshape(out_shape)
    t = transformer_kernel(kind, attrs, x, out_shape)
    if t is not None:
        return t
    a = x[0]
    if kind is OpKind.TANH:
        return np.tanh(a)
    if kind is OpKind.LEAKY_RELU:
        return np.where(a > 0.0, a, a * LEAKY_SLOPE)
    b = x[1]
    if kind is OpKind.RELU_GRAD:
        return np.broadcast_to(np.where(a > 0.0, b, 0.0), out_shape)
    if kind is OpKind.LEAKY_RELU_GRAD:
        return np.broadcast_to(np.where(a > 0.0, b, b * LEAKY_SLOPE), out_shape)
    if kind is OpKind.BCE_TERM:
        with np.errstate(over="ignore"):
            return np.broadcast_to((np.maximum(a, 0.0) - a * b) + np.log1p(np.exp(-np.abs(a))), out_shape)
    raise BadAttrs(f"unknown op kind {kind!r}")  # pragma: no cover


def row_stats(x2: np.ndarray):
    """Per-row mean / rstd over the last axis: sequential sums from +0.0."""
    d = x2.shape[1]
    mean = (np.cumsum(x2, axis=1)[:, -1] + 0.0) / d
    dev = x2 - mean[:, None]
    var = (np.cumsum(dev * dev, axis=1)[:, -1] + 0.0) / d
    return dev, 1.0 / np.sqrt(var + LN_EPS)


def _ids(idx: np.ndarray, v: int) -> np.ndarray:
    return np.clip(np.floor(idx), 0, v - 1).astype(np.int64)


def transformer_kernel(kind: OpKind, attrs: dict, x: list, out_shape):
    if kind is OpKind.TO_INDEX:
        v = np.broadcast_to(x[1], np.broadcast_shapes(x[0].shape, x[1].shape))
        return np.clip(np.floor((x[0] + 1.0) * 0.5 * v), 0.0, v - 1.0)
    if kind is OpKind.GELU:
        a = x[0]
        return 0.5 * a * (1.0 + np.tanh(GELU_C * (a + 0.044715 * a * a * a)))
    if kind is OpKind.GELU_GRAD:
        a, g = x
        t = np.tanh(GELU_C * (a + 0.044715 * a * a * a))
        d = 0.5 * (1.0 + t) + 0.5 * a * (1.0 - t * t) * GELU_C * (1.0 + 3.0 * 0.044715 * a * a)
        return np.broadcast_to(g * d, out_shape)
    if kind is OpKind.EMBEDDING:
        table, idx = x
        return table[_ids(idx, table.shape[0])]
    if kind is OpKind.EMBEDDING_DW:
        idx, dy = x
        v = attrs["dims"][0]
        ids = _ids(idx, v).reshape(-1)
        g = dy.reshape(ids.size, -1)
        out = np.zeros((v, g.shape[1]))
        for r in range(ids.size):            # row order, one rounded add per row
            out[ids[r]] += g[r]
        return out + 0.0
    if kind in (OpKind.LAYERNORM, OpKind.LAYERNORM_DX, OpKind.LN_DGAMMA):
        d = x[0].shape[-1]
        x2 = x[0].reshape(-1, d)
        dev, rstd = row_stats(x2)
        xhat = dev * rstd[:, None]
        if kind is OpKind.LAYERNORM:
            return ((xhat * x[1]) + x[2]).reshape(out_shape)
        dy = x[-1].reshape(-1, d)
        if kind is OpKind.LN_DGAMMA:
            return col_sum_seq(dy * xhat)
        dxh = dy * x[1]
        m1 = (np.cumsum(dxh, axis=1)[:, -1] + 0.0) / d
        m2 = (np.cumsum(dxh * xhat, axis=1)[:, -1] + 0.0) / d
        return (((dxh - m1[:, None]) - xhat * m2[:, None]) * rstd[:, None]).reshape(out_shape)
    if kind is OpKind.BIAS_ADD:
        return x[0] + x[1]
    if kind in (OpKind.REL_SKEW, OpKind.REL_UNSKEW):
        t = x[0].shape[-1]
        a = x[0].reshape(-1, t, t)
        out = np.zeros_like(a)
        for i in range(t):
            if kind is OpKind.REL_SKEW:        # out[i, 0..i] = a[i, T-1-i .. T-1]
                out[:, i, :i + 1] = a[:, i, t - 1 - i:]
            else:                              # out[i, T-1-i .. T-1] = a[i, 0..i]
                out[:, i, t - 1 - i:] = a[:, i, :i + 1]
        return out.reshape(out_shape)
    if kind in (OpKind.BMM, OpKind.BMM_NT, OpKind.BMM_TN):
        a, b = x
        out = np.empty(out_shape)
        for i in range(a.shape[0]):
            ai = a[i].T if kind is OpKind.BMM_TN else a[i]
            bi = b[i].T if kind is OpKind.BMM_NT else b[i]
            out[i] = matmul_seq(np.ascontiguousarray(ai), np.ascontiguousarray(bi))
        return out
    if kind is OpKind.CAUSAL_SOFTMAX:
        sc = attrs["value"]
        t = x[0].shape[-1]
        z = x[0].reshape(-1, t, t) * sc
        mask = np.tril(np.ones((t, t), dtype=bool))
        zm = np.where(mask, z, -np.inf)
        e = np.exp(zm - zm.max(axis=2, keepdims=True))
        s_ = np.cumsum(e, axis=2)[:, :, -1:] + 0.0
        return (e / s_).reshape(out_shape)
    if kind is OpKind.SOFTMAX_GRAD:
        sc = attrs["value"]
        y, dy = x
        t = y.shape[-1]
        y3, d3 = y.reshape(-1, t), dy.reshape(-1, t)
        dot = np.cumsum(d3 * y3, axis=1)[:, -1:] + 0.0
        return (sc * (y3 * (d3 - dot))).reshape(out_shape)
    if kind in (OpKind.CROSS_ENTROPY, OpKind.CROSS_ENTROPY_GRAD):
        logits, idx = x
        r, v = logits.shape
        ids = _ids(idx, v)
        mx = logits.max(axis=1, keepdims=True)
        e = np.exp(logits - mx)
        s_ = np.cumsum(e, axis=1)[:, -1:] + 0.0
        if kind is OpKind.CROSS_ENTROPY:
            lse = np.log(s_[:, 0]) + mx[:, 0]
            loss = lse - logits[np.arange(r), ids]
            return np.array(sum_seq(loss) / r)
        g = e / s_
        g[np.arange(r), ids] -= 1.0
        return g / attrs.get("rows", float(r))     # data parallel: the global row count
    return None


def _div(a, b):
    with np.errstate(divide="ignore", invalid="ignore"):
        return np.divide(a, b)


_BINARY = {OpKind.ADD: np.add, OpKind.SUB: np.subtract, OpKind.MUL: np.multiply, OpKind.DIV: _div}


EXT = frozenset(tuple(OpKind)[14:])


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
    elif kind in EXT:
        r = ext_kernel(kind, attrs, x, out_shape)
    else:  # pragma: no cover
        raise BadAttrs(f"unknown op kind {kind!r}")
    return [Tensor(out_shape, r)]
