"""CPU oracle for the PARTIME per-tick pipeline. TEST INFRASTRUCTURE ONLY.

This package restates, in numpy, the algorithm the reference specifies for
the hot path:
- SPEC.md:26-121 is `netcore`: layer math, losses, optimizers and the
  `sequential_step` oracle.
- SPEC.md:190-272 is `engine`: the lock-step tick with double-buffered
  stage inputs, a delayed forward, a stale backward and per-tick updates.
- PAPER.md:311-366 (Eqs. 6-10) and PAPER.md:579-602 (Alg. 1).
- SPEC.md:123-188 is `partition.balance`: the min-max contiguous DP.

Only these may import it, and only as the checker:
- `tests/`;
- `__graft_entry__.smoke()`;
- `bench.py`'s `cpu_baseline` leg and its `--impl reference` arm.
The product path (`paper_2210_09147_b200`) never imports it. If the CUDA
library is missing, the product fails loudly rather than falling back here.

Parity status: the reference ships no executable engine, so
no reference output pins this oracle. It is pinned by the SPEC worked
examples and properties in `tests/test_oracle.py` (SPEC.md:59-88, 153,
223-225, 232, 246-251, 299). See DESIGN.md §Oracle.
"""
