"""CPU oracle for arXiv 1604.06174 ("Training Deep Nets with Sublinear Memory Cost").

TEST INFRASTRUCTURE ONLY.  Nothing in the product path (``paper_1604_06174_b200``,
``include/``) imports, links or executes anything under ``oracle/``.  The only
callers allowed are ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s
``cpu_baseline`` / ``--impl reference`` legs.

The oracle is a plain, slow, obviously-correct re-statement of the paper:

* ``oracle.graph``   — computation graph G=(V, pred) (Alg. 2 input), op
                       metadata (minimal backward dependencies),
                       validation and the deterministic topological order.
* ``oracle.planner`` — mirror plans m: V -> N: sqrt(n) segmentation
                       (Sec. 4.3, Eq. 1), Alg. 3 budget plan
                       (PAPER.md:281-301), App. A grid search, the
                       recursive plan (Sec. 4.4, Eqs. 2-3), drop-low-cost
                       (Sec. 4.2); Alg. 2 mirrored gradient graph
                       (PAPER.md:259-279); the Fig. 2 liveness-counter allocator
                       (PAPER.md:152-172); pool offsets.
* ``oracle.chain``   — fp64 NumPy forward/backward of the residual BN-ReLU-GEMM chain,
                       plain backprop (definition) and a V'-interpreter that executes a
                       plan through its tags with an interference check (PAPER.md:135,
                       400), plus the bf16-operand emulation and the data-parallel shard
                       emulation.
* ``oracle.lstm``    — fp64 unrolled LSTM with time-segment recompute.

Every function cites the PAPER.md line(s) it follows.  Readings of silent/garbled
passages are listed in DESIGN.md ("Readings") and referenced here as R1..Rn.
The oracle shares no code with the CUDA path.
"""
