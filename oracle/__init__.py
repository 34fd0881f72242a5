"""dflow ORACLE — test infrastructure only.

A plain, slow, obviously-correct CPU implementation (Python + numpy, float64)
of the synchronous replicated data-parallel MLP train step of arXiv 1603.04467
(§2 Fig.1/Fig.2 :96-123, §4.1 gradients :480-524, §5.5 lossy
compression :805-821, §7 synchronous data parallelism :932-945).

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s
``cpu_baseline`` / ``--impl reference`` legs may import anything from here.
The product path (``paper_1603_04467_b200``) never imports it and shares no
code with it; the only shared module is ``synth`` (seeded random inputs, no
arithmetic of the method).

Modules:
  graph     — dataflow graph IR, builder, JSON export, gradient-graph
              construction
  executor  — dependency-counting executor with a FIFO ready queue
              
  kernels   — per-op float64 kernels, fp32-boundary / pure-f64 modes
  codec     — 32->16->32 truncation codec
  exchange  — cross-replica combine (FP32 / TRUNC16), readings A3, A6, A7
  mlp       — stacked Relu(XW+b) MLP graph builder and the replicated step

Parity status per function is listed in DESIGN.md ("Oracle pins").  Every
oracle function is pinned by at least one test under tests/test_oracle_*.py.
"""
