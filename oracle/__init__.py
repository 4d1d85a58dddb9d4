"""CPU oracle for the ZeRO-DP hot path (arXiv 1910.02054) -- TEST INFRASTRUCTURE.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s cpu_baseline /
``--impl reference`` legs may import anything from this package.  The product
path (``paper_1910_02054_b200``) never imports it and has no CPU fallback.

The oracle is a plain, slow, obviously correct implementation of what the path
computes, written from the paper (PAPER.md = "P:n") and the readings recorded in
DESIGN.md §3 (taken from SURVEY.md §8c).  It shares no code with the CUDA path
(no kernels, headers, tables or helpers); the only common module is ``synth``,
which produces seeded inputs and holds none of the method's arithmetic.

Modules
-------
numerics  fp32 <-> fp16 / bf16 conversions (reading c-5)
layout    bucket / partition layout (reading c-7; "N_d equal partitions",
          P:366 buckets, P:420-422 constant-size buffers)
planner   model-state memory (Fig. 1, Table 1), max model size
          (Table 2) and communication volume
step      unpartitioned replicated-DP mixed-precision Adam step (c-1..c-5;
          P:211) with the loss-scale state machine

Pins (what each function is checked against, other than itself) are listed in
each module header and in DESIGN.md §4.  "parity unpinned": none of the
arithmetic functions; the throughput numbers are unpinned (the paper prints
none).
"""
