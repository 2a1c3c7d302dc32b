"""Pins for oracle.krylov / oracle.precond / oracle.normalize: brute-force minimum residual,
the ideal-preconditioner eigenvalues, null-space invariance,
dense bordered LU of the whole system, and local mass conservation."""
import numpy as np
import pytest
import scipy.linalg as sla
import scipy.sparse as sp

from oracle import fem, krylov, mass, mg, normalize, precond


def _krylov_min_residual(Kd, b, j, Pinv=None):
    """Brute force: min ||b - K x|| over x in K_j(K, b) via an explicit, fully re-orthogonalised
    basis of the Krylov space + dense least squares."""
    Q = (b / np.linalg.norm(b))[:, None]
    for _ in range(j - 1):
        v = Kd @ Q[:, -1]
        for _pass in range(2):
            v = v - Q @ (Q.T @ v)
        Q = np.concatenate([Q, (v / np.linalg.norm(v))[:, None]], axis=1)
    y, *_ = np.linalg.lstsq(Kd @ Q, b, rcond=None)
    return Q @ y


def test_minres_identity_pc_matches_brute_force():
    """P = I on a random SPD-bordered saddle system: MINRES iterate j minimises ||b - K x||
    over the Krylov space."""
    rng = np.random.default_rng(0)
    nA, nB = 30, 10
    X = rng.standard_normal((nA, nA)); A = X @ X.T + nA * np.eye(nA)
    B = rng.standard_normal((nB, nA))
    Kd = np.block([[A, B.T], [B, np.zeros((nB, nB))]])
    b = rng.standard_normal(nA + nB)
    for j in (1, 3, 8, 15):
        x, rep = krylov.minres(lambda v: Kd @ v, b, lambda v: v.copy(), rtol=0.0, maxit=j)
        xb = _krylov_min_residual(Kd, b, j)
        np.testing.assert_allclose(x, xb, rtol=1e-8, atol=1e-8 * np.abs(xb).max())
        # |eta_j| is the residual norm for P = I
        assert rep.history[-1] == pytest.approx(np.linalg.norm(b - Kd @ x), rel=1e-8)


def test_minres_identity_converges_in_one_step():
    b = np.random.default_rng(1).standard_normal(7)
    x, rep = krylov.minres(lambda v: v.copy(), b, lambda v: v.copy(), rtol=1e-12, maxit=5)
    assert rep.iterations == 1
    np.testing.assert_allclose(x, b)


@pytest.mark.parametrize("n", [2, 4])
def test_ideal_preconditioner_three_iterations(n):
    """P_ideal = diag(A, B A^{-1} B^T): eigenvalues of the preconditioned matrix in
    {0, 1, (1 +- sqrt 5)/2}, so MINRES stops in <= 3 iterations."""
    s = fem.assemble_system(n)
    g = s.g
    A = s.Av.toarray(); B = s.B.toarray()
    S = B @ np.linalg.solve(A, B.T)
    Splus = np.linalg.pinv(S, rcond=1e-12)
    Pinv = lambda v: np.concatenate([np.linalg.solve(A, v[:g.n_u]), Splus @ v[g.n_u:]])
    Pmat = np.block([[np.linalg.inv(A), np.zeros((g.n_u, g.n_p))], [np.zeros((g.n_p, g.n_u)), Splus]])
    ev = np.linalg.eigvals(Pmat @ s.K.toarray())
    targets = np.array([0.0, 1.0, (1 + 5 ** 0.5) / 2, (1 - 5 ** 0.5) / 2])
    assert np.abs(ev[:, None] - targets[None, :]).min(axis=1).max() < 1e-8
    x, rep = krylov.minres(lambda v: s.K @ v, s.b, Pinv, rtol=1e-10, maxit=10)
    assert rep.iterations <= 3 and rep.converged


def _bordered_solution(s):
    """Dense LU of [[K, Y], [Z^T, 0]] with Y the 2-D null space and Z^T the O12 constraints
    (SURVEY §8(c) 'Final solution' pin)."""
    g = s.g
    N = g.N
    k = fem.null_vector_k(g)
    y1 = np.zeros(N); y1[g.n_u:g.n_u + g.n_k] = 1.0
    y2 = np.zeros(N); y2[g.n_u + g.n_k:] = 1.0
    z1 = np.zeros(N); z1[g.n_u:] = k
    z2 = np.zeros(N); z2[g.n_u:] = s.MQ @ np.ones(g.n_p)
    Y = np.stack([y1, y2], axis=1); Z = np.stack([z1, z2], axis=1)
    Big = np.block([[s.K.toarray(), Y], [Z.T, np.zeros((2, 2))]])
    sol = np.linalg.solve(Big, np.concatenate([s.b, [0.0, 0.0]]))
    assert np.abs(sol[N:]).max() < 1e-10 * np.abs(sol[:N]).max()   # consistent system
    return sol[:N]


@pytest.mark.parametrize("n", [2, 4, 8])
def test_minres_p1_matches_dense_bordered_lu(n):
    s = fem.assemble_system(n)
    g = s.g
    xd = _bordered_solution(s)
    P = precond.StokesP1(s)
    x, rep = krylov.minres(lambda v: s.K @ v, s.b, P, rtol=1e-12, maxit=300)
    k = fem.null_vector_k(g)
    xn = normalize.normalise_solution(x, g.n_u, s.MQ, k)
    np.testing.assert_allclose(xn, xd, atol=1e-9 * np.abs(xd).max())
    # O12: with P1 and x0 = 0 the normalisation is (nearly) a no-op
    assert np.abs(xn - x).max() < 1e-8 * np.abs(x).max()
    # |eta| non-increasing
    assert np.all(np.diff(rep.history) <= 1e-14 * rep.history[0])


def test_minres_eta_is_preconditioned_residual_norm():
    """|eta_j| = ||r_j||_{P^{-1}} = sqrt(r_j^T P^+ r_j) with P = P1."""
    s = fem.assemble_system(4)
    P = precond.StokesP1(s)
    for j in (1, 5, 12):
        x, rep = krylov.minres(lambda v: s.K @ v, s.b, P, rtol=0.0, maxit=j)
        r = s.b - s.K @ x
        assert rep.history[-1] == pytest.approx(np.sqrt(r @ P(r)), rel=1e-8)


def test_minres_null_component_invariance():
    """Adding alpha w, w = [0; k], to the initial iterate leaves delta_j, gamma_j and the residuals
    unchanged."""
    s = fem.assemble_system(4)
    g = s.g
    k = fem.null_vector_k(g)
    wv = np.concatenate([np.zeros(g.n_u), k])
    P = precond.StokesP1(s)
    x0, r0 = krylov.minres(lambda v: s.K @ v, s.b, P, rtol=0.0, maxit=10, x0=np.zeros(g.N))
    for alpha in (1.0, 1e3):
        x1, r1 = krylov.minres(lambda v: s.K @ v, s.b, P, rtol=0.0, maxit=10, x0=alpha * wv)
        np.testing.assert_allclose(r1.delta, r0.delta, rtol=1e-9)
        np.testing.assert_allclose(r1.gamma, r0.gamma, rtol=1e-9)
        np.testing.assert_allclose(np.linalg.norm(s.b - s.K @ x1), np.linalg.norm(s.b - s.K @ x0), rtol=1e-8)


def test_minres_p2_converges_and_is_positive():
    s = fem.assemble_system(8)
    P = precond.StokesP2(s, a=0.01)
    x, rep = krylov.minres(lambda v: s.K @ v, s.b, P, rtol=1e-8, maxit=300)
    assert rep.converged and rep.iterations < 80
    assert np.linalg.norm(s.b - s.K @ x) < 1e-6 * np.linalg.norm(s.b)


def test_local_mass_conservation_contrast():
    """Q2-Q1*: the converged solution satisfies B0 u = g0 element by element;
    plain Q2-Q1 on the same mesh violates it by orders of magnitude more."""
    n = 8
    s = fem.assemble_system(n)
    g = s.g
    P = precond.StokesP1(s)
    x, _ = krylov.minres(lambda v: s.K @ v, s.b, P, rtol=1e-10, maxit=300)
    u = x[:g.n_u]
    g0 = s.b[g.n_u + g.n_k:]
    star = np.abs(s.B0 @ u - g0).max()
    # plain Taylor-Hood: drop the P0 rows/columns
    Kth = sp.bmat([[s.Av, s.B1.T], [s.B1, None]]).tocsr()
    bth = s.b[:g.n_u + g.n_k]
    xth = np.linalg.lstsq(Kth.toarray(), bth, rcond=None)[0]
    th = np.abs(s.B0 @ xth[:g.n_u] - g0).max()
    assert star <= 10 * 1e-10 * np.linalg.norm(s.b)
    assert th > 100 * star


def test_gmres_matches_brute_force_and_monotone():
    rng = np.random.default_rng(7)
    nn = 40
    A = rng.standard_normal((nn, nn)) + 8 * np.eye(nn)
    b = rng.standard_normal(nn)
    for j in (1, 4, 10):
        x, rep = krylov.gmres(lambda v: A @ v, b, lambda v: v.copy(), tol_abs=0.0, restart=50, maxit=j)
        xb = _krylov_min_residual(A, b, j)
        np.testing.assert_allclose(x, xb, rtol=1e-8, atol=1e-9)
        assert np.all(np.diff(rep.history) <= 1e-12)
    # restarted: true residual non-increasing across restarts
    x, rep = krylov.gmres(lambda v: A @ v, b, lambda v: v.copy(), tol_abs=1e-10, restart=5, maxit=200)
    assert rep.converged and np.linalg.norm(b - A @ x) < 1e-9
    # right preconditioning with the exact inverse: 1 iteration
    Ainv = np.linalg.inv(A)
    x, rep = krylov.gmres(lambda v: A @ v, b, lambda v: Ainv @ v, tol_abs=1e-10, restart=10, maxit=10)
    assert rep.iterations == 1


def test_plain_q2q1_minres_matches_dense_solution():
    """Plain Taylor-Hood (the conservation contrast): MINRES with the oracle's
    diag(V-cycle, Chebyshev-Jacobi(Q_k)) preconditioner reaches the least-squares solution of the
    reduced system [A B1^T; B1 0] (unique up to the constant Q1 pressure, compared mean-free)."""
    n = 8
    s = fem.assemble_system(n)
    g = s.g
    K, b = precond.plain_system(s)
    x, rep = krylov.minres(lambda v: K @ v, b, precond.StokesP2Plain(s), rtol=1e-12, maxit=500)
    assert rep.converged
    xd = np.linalg.lstsq(K.toarray(), b, rcond=None)[0]
    for v in (x, xd):
        v[g.n_u:] -= v[g.n_u:].mean()
    assert np.abs(x - xd).max() <= 1e-8 * np.abs(xd).max()
    # and the plain solution violates element-wise mass conservation
    g0 = s.b[g.n_u + g.n_k:]
    assert np.abs(s.B0 @ x[:g.n_u] - g0).max() > 1e-4
