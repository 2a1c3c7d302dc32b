"""Plain CPU oracle for the Q2-Q1* preconditioned-Krylov hot path (arXiv 2303.10233).

TEST INFRASTRUCTURE ONLY.  Only `tests/`, `__graft_entry__.smoke()` and the
`cpu_baseline` / `--impl reference` legs of `bench.py` may import anything from
this package.  The product path (`paper_2303_10233_b200/`, `include/`) never
imports, links or executes it, and it shares no code with the CUDA path:
assembly here is a generic element loop with 3x3 Gauss quadrature and SciPy
CSR matrices; the CUDA side uses closed-form row gathers into SELL slices.

Citation keys: `P:n` = PAPER.md line n; `R#`/`O#` = the readings listed in
DESIGN.md §3 (taken from SURVEY.md §8(c)).

Module map (each function cites the passage it follows):
  fem       grid numbering, bases, element loop, blocks L, B1, B0, M_Q, N, F1,
            Mdiag, Ap, Dirichlet lifting, right-hand sides
  mg        nested-Q2 prolongation, Chebyshev smoother, V-cycle      (reading R9)
  mass      5-colour SGS on M_Q, Chebyshev semi-iteration, Pi.C.Pi,
            exact augmented solve, Lanczos estimate of `a`            (readings R6, R7)
  krylov    MINRES (Algorithm 1), GMRES(m) with CGS2
  precond   P1, P2, Oseen M1, PCD Step I, two-stage driver
  normalize null-space normalisation before comparing solutions       (reading O12)

Parity status: every function above is pinned by a `-m "not gpu"` test in
tests/test_oracle_*.py against a closed form, an invariant, a textbook routine
or brute force; see DESIGN.md §4 for the pin of each.  None is "parity unpinned"
except `mass.estimate_cheb_lo` (a heuristic parameter estimate; pinned only by
its Ritz-value bracketing property).
"""
