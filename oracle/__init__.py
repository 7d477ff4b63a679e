"""CPU ORACLE for the FlashOverlap hot path (arXiv 2504.19519) — TEST INFRASTRUCTURE ONLY.

Plain, slow, obviously-correct NumPy (fp64) re-statement of what the paper's
signaling + reordering pipeline computes, step by step in the paper's order:

  O1 tile grid                      -> oracle.plan
  O2 tile execution order / block swizzle
  O3 waves and wave groups
  O4 per-rank GEMM in fp64          -> oracle.numerics
  O5 pre-communication reordering -> oracle.reorder
  O6 collectives as explicit sums / scatters / permutations
                                                    -> oracle.collectives
  O7 post-communication reordering   -> oracle.reorder
  O8 the plain definition (sequential GEMM -> collective) -> oracle.pipeline
  O9 inverse checks                                  -> oracle.pipeline
  Alg. 1 predictive wave-group search -> oracle.alg1
  fused residual-add / RMSNorm after the post-reorder -> oracle.post

Who may use it: only `tests/`, `__graft_entry__.smoke()` and `bench.py`'s
`cpu_baseline` / `--impl reference` legs.  The product package
`paper_2504_19519_b200` never imports, links or executes anything here, and
this package never imports the product package: the two share no code.  Only
the seeded input generators in `synthetic/` (which hold none of the method's
arithmetic) serve both.

Parity status per function is stated in each module header.  Unpinned:
the paper's real default swizzle (its figures are missing; DESIGN.md
reading R1) — the default order is pinned only by the two textual statements
PAPER.md:378 and :388.
"""
from . import plan, numerics, reorder, collectives, pipeline, post, alg1  # noqa: F401
