"""Pins for oracle.oseen: Q1 transfers, Ap structure, PCD pieces, block-triangular
preconditioning, GMRES behaviour and the Prop 3.3 bound."""
import numpy as np
import pytest
import scipy.sparse as sp

from oracle import fem, krylov, mass, mg, oseen

NU = 0.01


def test_q1_prolongation_reproduces_bilinears():
    nc = 4
    P1 = oseen.q1_prolongation_1d(nc)
    P = sp.kron(P1, P1)
    xc = -1 + np.arange(nc + 1) * (2 / nc); xf = -1 + np.arange(2 * nc + 1) * (1 / nc)
    Xc, Yc = np.meshgrid(xc, xc); Xf, Yf = np.meshgrid(xf, xf)
    f = lambda x, y: 1 + 2 * x - y + 3 * x * y
    np.testing.assert_allclose(P @ f(Xc, Yc).ravel(), f(Xf, Yf).ravel(), atol=1e-14)


@pytest.mark.parametrize("n", [4, 8])
def test_ap_structure(n):
    """Ap = B1 Mdiag^{-1} B1^T is symmetric PSD with null space = constants (enclosed flow),
    pattern 21n^2 - 2n - 3 (SURVEY §8 nnz table), and D^{-1}Ap spectrum inside (0, 1.6]."""
    Ap = oseen.pcd_ap_grid(n)
    A = Ap.toarray()
    np.testing.assert_allclose(A, A.T, atol=1e-15)
    ev = np.linalg.eigvalsh(A)
    assert abs(ev[0]) < 1e-12 * ev[-1] and ev[1] > 1e-8 * ev[-1]
    assert np.abs(A @ np.ones(A.shape[0])).max() < 1e-13
    assert (np.abs(A) > 1e-14 * np.abs(A).max()).sum() == 21 * n * n - 2 * n - 3
    lam = np.linalg.eigvals(np.diag(1 / np.diag(A)) @ A).real
    assert lam.max() < 1.6
    s = fem.assemble_system(n, nu=NU)
    np.testing.assert_allclose(fem.pcd_ap(s).toarray(), A, atol=1e-14)


def test_mass_jacobi_interval():
    """Eigenvalues of diag(Qk)^{-1} Qk lie in [1/4, 9/4] (1D: [1/2, 3/2], tensor product) —
    the Chebyshev-Jacobi interval of Mp^{-1} (reading R13)."""
    s = fem.assemble_system(6)
    Q = s.Qk.toarray()
    lam = np.linalg.eigvals(np.diag(1 / np.diag(Q)) @ Q).real
    assert lam.min() >= 0.25 - 1e-12 and lam.max() <= 2.25 + 1e-12


def test_ap_vcycle_and_schur_null_space():
    """One Ap V-cycle + projection returns mean-zero vectors; the PCD Schur apply maps into the
    mean-zero subspace, i.e. the null space of the reduced Step-I operator (constants)."""
    n = 8
    s = fem.assemble_system(n, nu=NU)
    S = oseen.PCDSchur(s, NU)
    r = np.random.default_rng(1).standard_normal(s.g.n_k)
    z = S(r)
    assert abs(z.sum()) < 1e-12 * np.abs(z).sum()
    H = S.Ap
    # the V-cycle is a convergent iteration for Ap on the mean-zero subspace
    A = H.levels[0]["A"].toarray()
    nk = A.shape[0]
    Pi = np.eye(nk) - np.ones((nk, nk)) / nk
    V = np.stack([H.solve(e) for e in np.eye(nk)], axis=1)
    rho = np.abs(np.linalg.eigvals(Pi @ (np.eye(nk) - V @ A) @ Pi)).max()
    assert rho < 0.6


def test_f_vcycle_preconditions_convection():
    """The ellipse-smoothed V-cycle on F_s (reading R9') at n = 64 (coarse 32) makes GMRES on F
    converge to 1e-8 in few iterations; with the real interval (bim = 0) it stagnates."""
    h = oseen.velocity_hierarchy(64, NU, n_coarse=32)
    A = h.levels[0]["A"]
    b = np.random.default_rng(0).standard_normal(A.shape[0])
    x, rep = krylov.gmres(lambda v: A @ v, b, lambda v: h.vcycle(v), tol_abs=1e-8 * np.linalg.norm(b),
                          restart=50, maxit=40)
    assert rep.converged and rep.iterations <= 25
    h.levels[0]["bim"] = 0.0
    x, rep = krylov.gmres(lambda v: A @ v, b, lambda v: h.vcycle(v), tol_abs=1e-8 * np.linalg.norm(b),
                          restart=50, maxit=40)
    assert not rep.converged


def test_exact_block_triangular_two_iterations():
    """With the exact F and the exact Schur complement S = B F^{-1} B^T (pseudo-inverse), the
    block upper-triangular preconditioner makes GMRES converge in <= 2 iterations
    (minimal polynomial (lam - 1)^2)."""
    n = 4
    s = fem.assemble_system(n, nu=NU)
    g = s.g
    F = s.Av.toarray(); B = s.B.toarray()
    Finv = np.linalg.inv(F)
    S = B @ Finv @ B.T
    Sp = np.linalg.pinv(S, rcond=1e-12)

    def M(r):
        zp = -Sp @ r[g.n_u:]
        zu = Finv @ (r[:g.n_u] - B.T @ zp)
        return np.concatenate([zu, zp])
    x, rep = krylov.gmres(lambda v: s.K @ v, s.b, M, tol_abs=1e-10 * np.linalg.norm(s.b), restart=20, maxit=20)
    assert rep.iterations <= 2 and rep.converged


def test_two_stage_prop33_bound_and_convergence():
    """Two-stage PCD at n = 16: both stages converge, the transition residual obeys
    Prop 3.3 generalised to g != 0 (reading R16), the final residual meets eta."""
    n = 16
    s = fem.assemble_system(n, nu=NU)
    eta, c = 1e-6, 10.0
    x, (r1, r2), zstar, bound = oseen.two_stage(s, NU, a=0.005, eta=eta, c=c, restart=50, maxit=400)
    assert r1.converged and r2.converged
    assert zstar <= bound * (1 + 1e-9)
    assert np.linalg.norm(s.b - s.K @ x) <= eta * np.linalg.norm(s.b) * (1 + 1e-6)
    # the jump: the transition residual is far above the Step-I tolerance
    nr = s.g.n_u + s.g.n_k
    assert zstar > 2 * c * eta * np.linalg.norm(s.b[:nr])
    # GMRES residual estimates are non-increasing within each restart cycle
    assert np.all(np.diff(r2.history[:50]) <= 1e-12 * r2.history[0])
