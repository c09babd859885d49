"""ORACLE -- TEST INFRASTRUCTURE ONLY.

A plain, slow, obviously-correct CPU implementation (NumPy/SciPy, float64 /
complex128) of what the CUDA hot path computes: left polynomially
preconditioned Arnoldi/Lanczos for A^{-1/2}b and A^{1/2}b = A^{-1/2}(Ab)
(Algorithm 1), with the Chebyshev
 and Ritz/Newton-Lejà preconditioning
polynomials, plus closed-form reference solutions.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s cpu_baseline /
``--impl reference`` legs may import this package.  The product path
(``paper_2401_06684_b200``) never imports it, and this package never imports the
product path: they share no code (only the seeded generators in ``inputs/``).

Modules (each function cites the passage it follows):
  spmv       O9  row-chunked SciPy CSR mat-vec
  chebyshev  O1, O3  Chebyshev interpolant of z^{-1/2}, forward three-term apply
  newton     O2, O3  Ritz values, Lejà order, divided differences, Newton apply
  contour_ls §5.3    least-squares q on a discretised contour, Arnoldi-like apply
  dense      O6  y = beta0 * H^{-1/2} e_1 by eigendecomposition
  krylov     O4, O5, O7, O8  Algorithm 1 (Lanczos / CGS2 Arnoldi), history, m*
  reference  R1-R4  closed-form / reference f(A)b

Parity status: every function is pinned by a ``-m "not gpu"`` test in
tests/test_oracle_*.py, including the Ritz node VALUES of a finite Arnoldi run
(closed forms: the 1D Laplacian from e_1, invariant subspaces).  For generic
inputs those values carry ~1e-11 of rounding, so the GPU parity
tests compare nodes as multisets at 1e-8 and import the oracle's q for H/x.
"""
