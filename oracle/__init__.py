"""CPU ORACLE for arXiv 2506.16759 Algorithm 1 — TEST INFRASTRUCTURE ONLY.

This package is a plain, slow, obviously-correct float64 numpy implementation of the
paper's bottom-up sketching H^2 construction, written from PAPER.md (the paper) step by
step.  It exists to check the CUDA path.  Only ``tests/``, ``__graft_entry__.smoke()`` and
``bench.py``'s ``cpu_baseline`` / ``--impl reference`` legs may import it.  The product path
(``paper_2506_16759_b200``) never imports, links or executes anything here, and the
oracle never imports the product: the two share no code.  The only shared module is
``synth`` (seeded point clouds / probes; none of the method's arithmetic).

Modules (each function cites the passage it follows):
  rng       Philox4x32-10 counter-based generator -> the centred binomial Omega of DESIGN.md R8
            ("a random matrix"; Gaussian Omega: a caller's array, R34)
  geometry  KD-tree cluster tree, Eq.(1) admissibility, dual-tree traversal
  kernels   exponential covariance / Helmholtz IE entry evaluation
  cpqr      column-pivoted QR and row interpolative decomposition (Eq.3)
  h2        Algorithm 1 fixed + adaptive, H^2 matvec, to_dense

Pins (tests/test_oracle_*.py, all ``-m "not gpu"``): Philox known-answer vectors; kernel
closed forms printed in PAPER/SPEC; KD-tree tiling by brute force; CPQR pivots vs LAPACK
dgeqp3 (scipy) and reconstruction; whole-build error vs dense K on tiny inputs; exact
recovery of synthetic H^2 matrices of known ranks; identity rows at skeletons; special
cases (zero operator, rank-1 operator, all-dense, weak admissibility = HSS).
Parity unpinned: none of the functions listed above.
"""
