"""oracle — TEST INFRASTRUCTURE ONLY.

A plain, slow, obviously-correct CPU implementation of what the ozr hot path computes, written from
PAPER.md (Terao & Ozaki, "Forward Error-Oriented Iterative Refinement for Eigenvectors of a Real
Symmetric Matrix", arXiv 2602.19090). Every function cites the passage it follows as
``PAPER.md:<line>`` plus the section / equation / algorithm.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline`` / ``--impl reference``
leg may import this package. The product path (``paper_2602_19090_b200``) never imports it and shares
no code, header, table or constant generator with it; only the seeded input generators in
``workloads/`` (which hold none of the method's arithmetic) serve both.

Modules
  fp        ufp, ⌈log2⌉, TwoSum / pair arithmetic (§2.1-2.2)
  split     σ/τ splitting (§2.3 eq. sigma/tau/a/x), β/α (§3.3 eq. proposed_beta, §4.1), and the
            build's INT8 digit reading of the slices (DESIGN.md "Readings" R4-R7)
  products  same-definition slice products (exact integer planes) and their exact recombination
  refine    Algorithm 1 (§2.4) with the one-sided product (§3.3), the driver, reference
            eigenvectors and forward error
  hermitian the Hermitian extension of Algorithm 1 (R18): complex products as their
            definition in double-double, the truncation on both parts, forward error with phase alignment
  _clib     ctypes loader for ddmm.c (double-double GEMM, __float128 Jacobi)

Parity status: every function is pinned by a ``-m "not gpu"`` test in tests/test_oracle_*.py (closed forms,
exact rationals, exactly known eigensystems, __float128 Jacobi); none is "parity unpinned".
"""
