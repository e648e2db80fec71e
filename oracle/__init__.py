"""ORACLE — TEST INFRASTRUCTURE ONLY.

A plain, slow, obviously correct CPU implementation of what the B200 path
computes, written from PAPER.md (arXiv 1812.03770, "Owl's computation graph")
and the readings of SURVEY.md §8(c) / DESIGN.md.  Only ``tests/``,
``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline`` /
``--impl reference`` legs may import it.  The product path
(``paper_1812_03770_b200``) never imports, calls or links anything here, and
this package never imports the product path: the two share no code.  The only
shared module is ``workloads`` (seeded inputs + graph specs, no method
arithmetic).

Modules (each function cites the passage it follows; "P:n" = PAPER.md line n,
"S:n" = SPEC.md line n):
  ops.py        op table, shape inference, eager f64 semantics
  graph.py      graph G=(V,E,lambda,U) from a spec, add_node checks (Def. 1)
  eager.py      eager evaluation, one fresh allocation per node
  optimise.py   CSE -> CF -> DCE
  schedule.py   post-order DFS gamma, Var signatures, fusion grouping (c6)
  planner.py    Algorithm 1 on groups (readings R1-R13 in DESIGN.md)
  validate.py   brute-force liveness validator
  incremental.py c9 recompute-set model + block-simulated evaluator
  dump.py       canonical JSON dumps compared byte-for-byte with the C++ host compiler
  pebble.py     exact pebble-game search for tiny DAGs (Def. 3)

Parity-pin status: every function here is pinned by tests under
tests/test_oracle_*.py; none is "parity unpinned".
"""
