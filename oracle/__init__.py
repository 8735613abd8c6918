"""CPU oracle for CDFGNN (arXiv 2408.00232) — TEST INFRASTRUCTURE ONLY.

A plain, slow, obviously-correct Python + numpy (+ scipy.sparse as the SpMM
library primitive) implementation of what the paper's per-layer distributed
full-batch GCN step computes.  fp64 by default; an fp32 "kernel replay" mode
follows the canonical fp32 op sequence of reading R15 so the CUDA
cache-test / quantiser can be compared bit-for-bit on identical fp32 inputs.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline``
/ ``--impl reference`` legs may import this package.  It shares no code with
the CUDA path (``paper_2408_00232_b200``) and imports nothing from it; the two
meet only through the seeded inputs of ``synth``.

Modules (each function cites the PAPER.md line — ``P:Lx`` — it follows):
  graph      normalised adjacency  Â = D^-1/2 A D^-1/2
  partition  hierarchical EBV vertex-cut, masters, local order,
             halo lists, RF / imbalance factors
  gcn        unpartitioned full-batch GCN (the plain definition)
  quant      B-bit linear quantisation, error bound
  cache      Alg. 2 adaptive vertex cache + gather/scatter sync
  eps        adaptive threshold controller + EMA
  optim      SGD / Adam parameter update
  cdfgnn     Alg. 1 partitioned epoch

Parity status per function is listed in DESIGN.md §"Oracle pins"; a function
without an independent pin says "parity unpinned" in its docstring.
"""
