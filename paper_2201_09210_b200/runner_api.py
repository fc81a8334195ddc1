"""Backend protocol between the host orchestrator and a symbolic executor.

The reference's graph_runner surface is ``run_pass(sp, ch,
vars)`` + ``ChannelSet`` + ``VariableStore``.  Here a backend exposes it as:

eager side (imperative / traced / replay steps)
    ``put(host_tensor) -> value``, ``get(value) -> Tensor``,
    ``exec_op(kind, attrs, values) -> value``,
    ``var_define / var_read / var_assign / var_shape / var_shapes``,
    ``snapshot_vars() -> {name: Tensor}``, ``rollback()``

symbolic side
    ``compile(sp, tg) -> program``;
    ``begin_pass(program, lazy) -> channel`` with ``decide(decision)``,
    ``feed(slot, value)``, ``fetch(node_id, occurrence) -> Tensor``,
    ``cancel()``, ``wait() -> PassResult`` (Committed / Cancelled).

The product backend is :class:`paper_2201_09210_b200.b200.B200Backend`.
"""

from __future__ import annotations

from dataclasses import dataclass


@dataclass
class PassResult:
    """Committed(stats) | Cancelled(stats); stats per PassStats."""

    committed: bool
    exec_ms: float = 0.0
    stall_ms: float = 0.0
    ops: int = 0
    fetches: int = 0
    error: str | None = None
