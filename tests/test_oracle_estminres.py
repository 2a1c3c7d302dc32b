"""Pin of EST-MINRES: with the exact preconditioner P1 the Lanczos estimate converges
to the smallest nonzero eigenvalue of the singular pencil B A^{-1} B^T v = lam M_Q v (Eq. (7),
P:474-478) restricted to the complement of its null space (dense deflated solve, n <= 8)."""
import numpy as np
import pytest
import scipy.linalg as sla

from oracle import fem, krylov, precond


def deflated_infsup(s):
    """Smallest eigenvalue of S v = lam M_Q v on the complement of null(M_Q) + null(S) (dense)."""
    A = s.Av.toarray(); B = s.B.toarray(); MQ = s.MQ.toarray()
    S = B @ np.linalg.solve(A, B.T)
    # basis of the complement of the common null space: eigenvectors of M_Q + S with positive eigenvalue
    w, V = np.linalg.eigh(MQ + S)
    Q = V[:, w > 1e-10 * w.max()]
    lam = sla.eigh(Q.T @ S @ Q, Q.T @ MQ @ Q, eigvals_only=True)
    return lam[lam > 1e-10].min()


@pytest.mark.parametrize("n", [4, 8])
def test_est_minres_matches_deflated_eigenproblem(n):
    s = fem.assemble_system(n)
    P = precond.StokesP1(s)
    x, rep = krylov.minres(lambda v: s.K @ v, s.b, P, rtol=1e-12, maxit=400)
    g2 = krylov.est_minres_gamma2(rep.delta, rep.gamma)
    ref = deflated_infsup(s)
    assert g2 == pytest.approx(ref, rel=1e-3)
    # inf-sup constant is positive and bounded by the continuity constant (<= 2 for d = 2)
    assert 0.0 < ref < 2.0


def test_est_minres_empty_and_no_negative():
    assert np.isnan(krylov.est_minres_gamma2([], []))
    assert np.isnan(krylov.est_minres_gamma2([1.0, 2.0], [1.0, 0.1]))
