"""ORACLE — test infrastructure only.

A plain, slow, obviously-correct fp64 NumPy implementation of what the
Mumax3-cQED hot path computes (arXiv 2410.00966, /root/reference/PAPER.md),
written step by step in the paper's order and notation.  Only ``tests/``,
``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline`` / ``--impl
reference`` legs may import it.  It shares no code with the CUDA path
(``paper_2410_00966_b200``) and never imports it.

Citation keys: ``P:n`` = PAPER.md line n; ``C#`` = the reading numbered # in
SURVEY.md §8(c) / DESIGN.md "Readings".

Parity status per function is listed in DESIGN.md §Oracle; functions without a
pin say "parity unpinned" in their docstring.
"""
# submodules: constants, tensor, fields, llg, cavity, sim, dicke, analytic
