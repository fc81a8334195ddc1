"""Deterministic xorshift64* streams with O(log n) jump-ahead.

Same generator and stream naming as the reference (pkg/src/coex/rng.py:22-60,
SPEC.md:257): state = seed ^ fnv1a64(name) ^ mix, the all-zero state replaced by
0x9E3779B97F4A7C15, each draw maps the top 53 bits of ``x * 0x2545F4914F6CDD1D``
to [0, 1).

The reference's ``draw_at`` steps the generator ``index`` times (rng.py:53-60),
which makes ``coin``/``choice`` O(step).  The xorshift
state transition is linear over GF(2)^64, so here the n-th state is reached by
applying precomputed 64x64 bit-matrices for the powers of two of n: the result
is bit-identical (tests/test_golden_host.py pins it against vectors generated
from the reference) and costs O(log n).  The same matrices drive the device-side
synthetic-data kernel (csrc/coex_kernels.cuh ``k_synth``).
"""

from __future__ import annotations

MASK64 = (1 << 64) - 1
XS_MULT = 0x2545F4914F6CDD1D
FNV_OFFSET = 0xCBF29CE484222325
FNV_PRIME = 0x100000001B3
ZERO_STATE = 0x9E3779B97F4A7C15
TWO_M53 = 2.0 ** -53


def fnv1a64(text: str) -> int:
    h = FNV_OFFSET
    for byte in text.encode("utf-8"):
        h = ((h ^ byte) * FNV_PRIME) & MASK64
    return h


def xs_step(x: int) -> int:
    """One xorshift64 state transition (no output scrambling)."""
    x ^= x >> 12
    x = (x ^ (x << 25)) & MASK64
    x ^= x >> 27
    return x


def unit_of_state(x: int) -> float:
    """The [0,1) draw produced when the generator lands in state ``x``."""
    return (((x * XS_MULT) & MASK64) >> 11) * TWO_M53


class Xorshift64Star:
    """xorshift64* generator (rng.py:30-46)."""

    __slots__ = ("state",)

    def __init__(self, state: int):
        state &= MASK64
        self.state = state if state else ZERO_STATE

    def next_u64(self) -> int:
        self.state = xs_step(self.state)
        return (self.state * XS_MULT) & MASK64

    def next_unit(self) -> float:
        return (self.next_u64() >> 11) * TWO_M53

    def jump(self, n: int):
        """Advance by ``n`` transitions in O(log n)."""
        self.state = jump_state(self.state, n)


def stream_state(seed: int, name: str, mix: int = 0) -> int:
    return (seed ^ fnv1a64(name) ^ mix) & MASK64


def seeded_state(seed: int, name: str, mix: int = 0) -> int:
    """Initial generator state for a stream, with the zero-state substitution."""
    s = stream_state(seed, name, mix)
    return s if s else ZERO_STATE


# ---- GF(2) jump-ahead -------------------------------------------------------
# A matrix is stored as its 64 columns: col[b] = image of the unit vector 1<<b.
# Application uses 8 byte-indexed tables of 256 precomputed XOR combinations.


def _columns_of_step() -> list:
    return [xs_step(1 << b) for b in range(64)]


def _apply_cols(cols: list, v: int) -> int:
    r = 0
    b = 0
    while v:
        if v & 1:
            r ^= cols[b]
        v >>= 1
        b += 1
    return r


def _square(cols: list) -> list:
    return [_apply_cols(cols, c) for c in cols]


def _tables(cols: list) -> list:
    tabs = []
    for byte in range(8):
        base = cols[8 * byte: 8 * byte + 8]
        t = [0] * 256
        for v in range(1, 256):
            low = v & -v
            t[v] = t[v ^ low] ^ base[low.bit_length() - 1]
        tabs.append(t)
    return tabs


_POW_COLS: list = []   # _POW_COLS[j] = columns of T^(2^j)
_POW_TABS: list = []


def _ensure_powers(nbits: int):
    if not _POW_COLS:
        _POW_COLS.append(_columns_of_step())
        _POW_TABS.append(_tables(_POW_COLS[0]))
    while len(_POW_COLS) < nbits:
        _POW_COLS.append(_square(_POW_COLS[-1]))
        _POW_TABS.append(_tables(_POW_COLS[-1]))


def jump_columns(j: int) -> list:
    """Columns of T^(2^j) (exported for the device generator)."""
    _ensure_powers(j + 1)
    return list(_POW_COLS[j])


def jump_state(x: int, n: int) -> int:
    """State after ``n`` transitions from ``x``."""
    if n < 0:
        raise ValueError(f"negative jump {n}")
    if n < 64:
        for _ in range(n):
            x = xs_step(x)
        return x
    _ensure_powers(n.bit_length())
    j = 0
    while n:
        if n & 1:
            t = _POW_TABS[j]
            x = (t[0][x & 255] ^ t[1][(x >> 8) & 255] ^ t[2][(x >> 16) & 255] ^ t[3][(x >> 24) & 255]
                 ^ t[4][(x >> 32) & 255] ^ t[5][(x >> 40) & 255] ^ t[6][(x >> 48) & 255] ^ t[7][x >> 56])
        n >>= 1
        j += 1
    return x


def draw_at(seed: int, name: str, index: int) -> float:
    """The ``index``-th unit draw of stream ``name`` (rng.py:53-60), in O(log index)."""
    if index < 0:
        raise ValueError(f"negative draw index {index}")
    return unit_of_state(jump_state(seeded_state(seed, name), index + 1))
