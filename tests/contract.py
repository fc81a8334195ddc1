"""Contract-tolerance parity helpers (north_star: fp32 <= 1e-5, bf16 <= 2e-2 relative;
TraceGraph, decisions and counters bit-exact).

``grad_probe(src)`` rewrites a training program so that every parameter update
``p = sub(p, mul(G, LR))`` becomes ``gr_p = G``: the parameters stay at their initial
values and a new variable per parameter holds the gradient the step computed.  Every
co-executed step then checks the forward pass, the hand-written backward pass and the
loss at the same weights -- per tensor, one step's worth of rounding, no training
amplification -- and the final ``gr_*`` variables are the last step's gradients.
"""

from __future__ import annotations

import re

import numpy as np

_VAR_SHAPE = re.compile(r"^var (\w+) = .*?\[([0-9, ]*)\]")
_UPDATE = re.compile(r"\b(\w+) = sub\(\1, mul\((.*?), (\w+|[0-9.e-]+)\)\)")


def grad_probe(src: str) -> tuple:
    """(rewritten source, {parameter: gradient variable})."""
    shapes = {}
    for ln in src.splitlines():
        m = _VAR_SHAPE.match(ln.strip())
        if m:
            shapes[m.group(1)] = [int(t) for t in m.group(2).split(",") if t.strip()]
    head, body = src.split("\nsteps ", 1)
    grads = {}

    def sub(m):
        name, g = m.group(1), m.group(2)
        if name not in shapes:
            return m.group(0)
        grads[name] = f"gr_{name}"
        return f"gr_{name} = {g}"

    body = _UPDATE.sub(sub, body)
    decls = [f"var gr_{n} = fill({shapes[n]}, 0.0)" for n in grads]
    return head + "\n" + "\n".join(decls) + "\nsteps " + body, grads


def rel_err(got: np.ndarray, ref: np.ndarray) -> float:
    return float(np.linalg.norm(got - ref) / max(np.linalg.norm(ref), 1e-300))


def compare(ref, got, tol: float, grads: dict, zero_grads: dict = None) -> tuple:
    """Printed numbers element-wise and every gradient variable norm-wise per tensor against
    ``tol``.  ``zero_grads`` maps a gradient that is exactly zero in exact arithmetic (its
    computed value is rounding noise) to a sibling gradient of the same op: its norm is
    measured against the sibling's instead.  Returns (per-tensor errors, failures)."""
    zero_grads = zero_grads or {}
    assert len(ref.lines) == len(got.lines)
    errs = {}
    worst_line = 0.0
    for a, b in zip(ref.lines, got.lines):
        x, y = float(a), float(b)
        worst_line = max(worst_line, abs(x - y) / max(abs(x), 1e-300))
    errs["_lines"] = worst_line
    for p, gname in grads.items():
        r, g = ref.vars[gname].data, got.vars[gname].data
        assert g.shape == r.shape, gname
        if p in zero_grads:
            sib = ref.vars[grads[zero_grads[p]]].data
            errs[gname] = float(np.linalg.norm(g) / np.linalg.norm(sib))
        else:
            errs[gname] = rel_err(g, r)
    bad = {k: v for k, v in errs.items() if not v <= tol}
    return errs, bad
