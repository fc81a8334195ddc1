"""CPU parity oracle -- TEST INFRASTRUCTURE, not product code.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s CPU-baseline /
``--impl reference`` legs may import this package.  It restates, on the CPU,
the reference's algorithm for the hot path:

* :mod:`oracle.kernels` -- ``execute_kernel`` (pkg/src/coex/tensor.py:228-291),
  float64, pinned accumulation orders; pinned bit-for-bit against vectors
  generated from the reference itself (tests/golden/make_golden.py).
* :mod:`oracle.cpu_backend` -- ``run_pass`` / ``ChannelSet`` / ``VariableStore``
  (SPEC.md:420-486): a structured-walk graph runner on its own thread, plus
  the eager variable store used by imperative/traced steps.  The reference
  ships no graph runner; this restatement follows SPEC.md line by line and is
  cross-checked by mode equivalence (imperative == coexec == lazy).
"""
