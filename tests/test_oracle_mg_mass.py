"""Pins for oracle.mg and oracle.mass: Galerkin identity, polynomial closed forms,
brute-force Gauss-Seidel, exact pseudo-inverse, symmetry / definiteness / null space."""
import numpy as np
import pytest
import scipy.sparse as sp

from oracle import fem, mass, mg
import synth


def test_prolongation_weights_and_reproduction():
    P1 = mg.prolongation_1d(2).toarray()
    # fine node 1 is the 1/4 point of coarse element 0: (3/8, 3/4, -1/8)
    np.testing.assert_allclose(P1[1, :3], [3 / 8, 3 / 4, -1 / 8], atol=1e-15)
    np.testing.assert_allclose(P1[3, :3], [-1 / 8, 3 / 4, 3 / 8], atol=1e-15)
    np.testing.assert_allclose(P1[4, 2], 1.0)
    # reproduces coarse Q2 functions: a piecewise quadratic on the coarse grid
    nc = 4
    P = sp.kron(mg.prolongation_1d(nc), mg.prolongation_1d(nc)).toarray()
    gc, gf = fem.Grid(nc), fem.Grid(2 * nc)
    f = lambda x, y: 1 + 2 * x - 3 * y + x * y - 2 * x * x + 0.5 * y * y + x * x * y * y
    xc, yc = gc.node_xy(); xf, yf = gf.node_xy()
    np.testing.assert_allclose(P @ f(xc, yc), f(xf, yf), atol=1e-13)


@pytest.mark.parametrize("nc", [2, 4, 8])
def test_galerkin_identity(nc):
    """P^T L_f P = L_c on interior rows (nested spaces, exact quadrature)."""
    Lf = fem.laplacian(fem.Grid(2 * nc))
    Lc = fem.laplacian(fem.Grid(nc)).toarray()
    P1 = mg.prolongation_1d(nc)
    P = sp.kron(P1, P1)
    G = (P.T @ Lf @ P).toarray()
    np.testing.assert_allclose(G, Lc, atol=1e-12)


def _cheb_poly_apply(lam, lo, hi, degree):
    """Closed form of Chebyshev iteration from x0 = 0: x = (1 - p(lam))/lam * b with
    p(lam) = T_k((hi+lo-2 lam)/(hi-lo)) / T_k((hi+lo)/(hi-lo))  (textbook residual polynomial)."""
    T = np.polynomial.chebyshev.Chebyshev.basis(degree)
    p = T((hi + lo - 2 * lam) / (hi - lo)) / T((hi + lo) / (hi - lo))
    return (1 - p) / lam


def test_chebyshev_smoother_closed_form():
    rng = np.random.default_rng(1)
    lam = rng.uniform(0.05, 2.0, 40)
    A = sp.diags(lam).tocsr()
    b = rng.standard_normal(40)
    for deg in (1, 2, 3, 5):
        x, r = mg.chebyshev_smooth(A, np.ones(40), b, None, 0.16, 1.6, deg)
        np.testing.assert_allclose(x, _cheb_poly_apply(lam, 0.16, 1.6, deg) * b, rtol=1e-12, atol=1e-13)
        np.testing.assert_allclose(r, b - A @ x, atol=1e-13)


@pytest.mark.parametrize("n", [4, 8])
def test_vcycle_symmetric_positive(n):
    h = mg.Hierarchy(n)
    nq = fem.Grid(n).nq
    V = np.stack([h.vcycle(e) for e in np.eye(nq)], axis=1)
    np.testing.assert_allclose(V, V.T, atol=1e-12 * np.abs(V).max())
    assert np.linalg.eigvalsh(0.5 * (V + V.T))[0] > 0
    # V-cycle is a convergent solver for A: spectral radius of I - V A below 1
    A = h.levels[0]["A"].toarray()
    rho = np.abs(np.linalg.eigvals(np.eye(nq) - V @ A)).max()
    assert rho < 0.5


def test_sgs_colour_sweep_equals_sequential():
    """The 5-colour sweep equals scalar Gauss-Seidel in the colour-sorted order (brute force)."""
    n = 4
    s = fem.assemble_system(n)
    col = mass.colours(s.g)
    order = np.concatenate([np.nonzero(col == c)[0] for c in range(5)])
    rng = np.random.default_rng(3)
    r = rng.standard_normal(s.g.n_p); y = rng.standard_normal(s.g.n_p)
    np.testing.assert_allclose(mass.sgs_sweep(s.MQ, r, y, col),
                               mass.sgs_sweep_sequential(s.MQ, r, y, order), rtol=1e-12, atol=1e-12)
    # within one colour no two dofs are coupled
    MQ = s.MQ.toarray()
    for c in range(5):
        idx = np.nonzero(col == c)[0]
        sub = MQ[np.ix_(idx, idx)]
        assert np.count_nonzero(sub - np.diag(np.diag(sub))) == 0


def _sgs_matrix(MQ, col):
    n = MQ.shape[0]
    return np.stack([mass.sgs_sweep(MQ, e, np.zeros(n), col) for e in np.eye(n)], axis=1)


def test_chebyshev_sgs_closed_form():
    """Golub-Varga semi-iteration: with G = I - Cs^{-1} M (spectrum in [0, rho]) and
    G_g = gamma G + (1-gamma) I (spectrum in [-rhohat, rhohat]), the error after m steps
    from y0 = 0 is T_m(G_g/rhohat)/T_m(1/rhohat) e_0 (textbook Chebyshev semi-iteration).
    Checked on an SPD matrix with the same colour structure (M_Q + I shift)."""
    n = 3
    s = fem.assemble_system(n)
    col = mass.colours(s.g)
    M = (s.MQ + sp.identity(s.g.n_p) * 0.02).tocsr()
    Cinv = _sgs_matrix(M, col)
    G = np.eye(M.shape[0]) - Cinv @ M.toarray()
    ev = np.linalg.eigvals(G).real
    rho = ev.max() * 1.0001
    a = 1 - rho
    gam = 2 / (2 - rho); rh = rho / (2 - rho)
    r = np.random.default_rng(5).standard_normal(M.shape[0])
    e0 = np.linalg.solve(M.toarray(), r)
    for m in (1, 2, 3, 7, 20):
        T = np.polynomial.chebyshev.Chebyshev.basis(m)
        w, Vv = np.linalg.eig(gam * G + (1 - gam) * np.eye(len(G)))
        Pm = (Vv @ np.diag(T(w.real / rh) / T(1 / rh)) @ np.linalg.inv(Vv)).real
        y = mass.chebyshev_sgs(M, r, a, m, col)
        np.testing.assert_allclose(e0 - y, Pm @ e0, atol=1e-10 * np.abs(e0).max())


def test_augmented_solve_is_pseudo_inverse():
    """[[M_Q, k],[k^T, 0]] solve gives z = M_Q^+ r (min-norm, orthogonal to k); M_Q z = r - lam k."""
    s = fem.assemble_system(4)
    k = fem.null_vector_k(s.g)
    aug = mass.AugmentedMassSolver(s.MQ, k)
    r = np.random.default_rng(2).standard_normal(s.g.n_p)
    z, lam = aug.solve(r, return_multiplier=True)
    np.testing.assert_allclose(z, np.linalg.pinv(s.MQ.toarray()) @ r, rtol=1e-9, atol=1e-9)
    assert abs(k @ z) <= 1e-12 * np.linalg.norm(z)
    np.testing.assert_allclose(s.MQ @ z, r - lam * k, atol=1e-12 * np.linalg.norm(r))
    # r in span{k}: z = 0
    np.testing.assert_allclose(aug.solve(3.0 * k), 0.0, atol=1e-12)


def test_pi_c_pi_properties_and_limit():
    """Pi C Pi is symmetric PSD with null space exactly span{k}; z is orthogonal to k; as m grows
    it converges to the exact augmented solve (reading R6)."""
    n = 4
    s = fem.assemble_system(n)
    g = s.g
    col = mass.colours(g)
    k = fem.null_vector_k(g)
    a = 0.65 / n ** 2 * 0.9
    C = np.stack([mass.pi_c_pi(s.MQ, e, a, 20, col, k) for e in np.eye(g.n_p)], axis=1)
    np.testing.assert_allclose(C, C.T, atol=1e-10 * np.abs(C).max())
    ev = np.linalg.eigvalsh(0.5 * (C + C.T))
    assert ev[0] > -1e-10 * ev[-1] and ev[1] > 1e-6 * ev[-1]
    np.testing.assert_allclose(k @ C, 0.0, atol=1e-10 * np.abs(C).max())
    r = np.random.default_rng(4).standard_normal(g.n_p)
    exact = mass.AugmentedMassSolver(s.MQ, k).solve(r)
    z = mass.pi_c_pi(s.MQ, r, a, 200, col, k)
    np.testing.assert_allclose(z, exact, atol=1e-11 * np.abs(exact).max())


def test_sgs_spectrum_top_is_one_and_lanczos_brackets():
    """lambda_max(Cs^{-1} M_Q) = 1 exactly (SGS on PSD M_Q); the Lanczos lower-bound estimate
    lies inside [lambda_min on k-complement, 1] (Ritz values bracket)."""
    n = 4
    s = fem.assemble_system(n)
    col = mass.colours(s.g)
    Cinv = _sgs_matrix(s.MQ, col)
    ev = np.sort(np.linalg.eigvals(Cinv @ s.MQ.toarray()).real)
    assert abs(ev[-1] - 1.0) < 1e-12
    lam_min = ev[1]
    assert abs(ev[0]) < 1e-12
    est = mass.estimate_cheb_lo(s.MQ, synth.lanczos_start(s.g.n_p), 10, col)
    assert lam_min * (1 - 1e-10) <= est <= 1.0


def test_ellipse_chebyshev_closed_form():
    """Chebyshev iteration on an ellipse (reading R9'): with D = I and a normal matrix whose
    eigenvalues are mu +- i nu, x = (1 - p(lam))/lam b, p(lam) = T_k((theta-lam)/delta)/T_k(theta/delta),
    delta = sqrt(a^2 - b^2) possibly imaginary (textbook complex Chebyshev polynomials)."""
    rng = np.random.default_rng(9)
    mus = rng.uniform(0.2, 1.5, 6); nus = rng.uniform(0.0, 1.2, 6)
    blocks = [np.array([[m, -v], [v, m]]) for m, v in zip(mus, nus)]
    A = sp.csr_matrix(sp.block_diag(blocks))
    b = rng.standard_normal(12)
    lo, hi, bim = 0.16, 1.6, 1.3
    theta, a = 0.5 * (hi + lo), 0.5 * (hi - lo)
    delta = np.sqrt(complex(a * a - bim * bim))
    Ad = A.toarray()
    w, V = np.linalg.eig(Ad)
    for deg in (1, 2, 3, 4):
        T = np.polynomial.chebyshev.Chebyshev.basis(deg)
        p = T((theta - w) / delta) / T(theta / delta)
        ref = (V @ np.diag((1 - p) / w) @ np.linalg.inv(V) @ b).real
        x, r = mg.chebyshev_smooth_ellipse(A, np.ones(12), b, None, lo, hi, bim, deg)
        np.testing.assert_allclose(x, ref, rtol=1e-10, atol=1e-12)
        np.testing.assert_allclose(r, b - A @ x, atol=1e-12)
    # bim = 0 is the real Chebyshev iteration
    x0, _ = mg.chebyshev_smooth_ellipse(A, np.ones(12), b, None, lo, hi, 0.0, 3)
    x1, _ = mg.chebyshev_smooth(A, np.ones(12), b, None, lo, hi, 3)
    np.testing.assert_array_equal(x0, x1)


@pytest.mark.parametrize("n", [2, 5, 8])
def test_schur_reduction_equals_augmented_solve(n):
    """The Schur-complement reduction of the augmented M_Q system (used by the GPU's exact M_Q
    solve, NEXT-2) reproduces the bordered dense LU solve; S_k is PSD with null space
    the constants and lambda_max(diag(S_k)^{-1} S_k) = 12/7."""
    g = fem.Grid(n)
    s = fem.assemble_system(n)
    k = fem.null_vector_k(g)
    S = mass.schur_mass(g).toarray()
    ev = np.linalg.eigvalsh(S)
    assert abs(ev[0]) < 1e-14 * ev[-1] and ev[1] > 1e-9 * ev[-1]
    assert np.abs(S @ np.ones(g.n_k)).max() < 1e-15
    lam = np.linalg.eigvals(np.diag(1 / np.diag(S)) @ S).real
    assert lam.max() == pytest.approx(12 / 7, rel=1e-12)
    Sp = np.linalg.pinv(S, rcond=1e-12)
    r = np.random.default_rng(8).standard_normal(g.n_p)
    z = mass.augmented_via_schur(g, r, lambda v: Sp @ v)
    np.testing.assert_allclose(z, mass.AugmentedMassSolver(s.MQ, k).solve(r), atol=1e-10 * np.abs(z).max())
    np.testing.assert_allclose(z, mass.SparseAugmentedMassSolver(s.MQ, k).solve(r), atol=1e-10 * np.abs(z).max())
