"""B200-native symbolic-execution backend for Terra-style imperative/symbolic
co-execution (arXiv 2201.09210).

Host side (Python, keeps the reference ``coex`` API): frontend (:mod:`.lang`),
interpreter (:mod:`.interp`), TraceGraph (:mod:`.trace_graph`), symbolic program
generation (:mod:`.graph_gen`), orchestrator (:mod:`.coexec`).
Device side: ``csrc/`` -> ``libcoexb200.so`` (C-ABI, include/coex_b200.h), bound
by :mod:`.b200`.  There is no CPU execution path in this package.
"""

__version__ = "0.1.0"
