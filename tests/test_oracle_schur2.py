"""Pins of oracle.schur2: the two-field pressure Laplacian, the P0
convection-diffusion operator F0 (reading R25), the two-field PCD M_S (M2) and LSC (M3)."""
import numpy as np
import pytest
import scipy.sparse as sp

from oracle import fem, krylov, oseen, schur2

NU = 0.01


def _sys(n, nu=NU):
    return fem.assemble_system(n, nu=nu)


def test_two_field_laplacian_structure():
    """Lp = B M^-1 B^T: symmetric PSD, null space exactly the two pressure constants,
    Q1 block = the PCD Ap pinned in test_oracle_oseen."""
    s = _sys(6)
    g = s.g
    Lp = schur2.two_field_laplacian(s)
    D = Lp.toarray()
    assert np.abs(D - D.T).max() <= 1e-15 * np.abs(D).max()
    ev = np.linalg.eigvalsh(D)
    assert np.abs(ev[:2]).max() <= 1e-12 * ev[-1] and ev[2] > 1e-8 * ev[-1]
    c1 = np.r_[np.ones(g.n_k), np.zeros(g.n_0)]
    c0 = np.r_[np.zeros(g.n_k), np.ones(g.n_0)]
    assert np.abs(D @ c1).max() <= 1e-13 * np.abs(D).max() and np.abs(D @ c0).max() <= 1e-13 * np.abs(D).max()
    Ap = fem.pcd_ap(s).toarray()
    assert np.abs(D[:g.n_k, :g.n_k] - Ap).max() <= 1e-15 * np.abs(Ap).max()


def test_f0_diffusion_closed_form_and_linear_exactness():
    """F0 with zero wind = nu x the cell-centred 5-point Neumann Laplacian (Kronecker closed form);
    F0 1 = 0; with w = (1, 0) the central flux is exact for p linear in x on interior cells:
    (F0 p)_T = int_T w . grad p = h^2."""
    n = 5
    g = fem.Grid(n)
    z = np.zeros(g.nq)
    F0 = schur2.f0_jump(g, NU, z, z)
    T = sp.diags([-np.ones(n - 1), np.r_[1.0, 2.0 * np.ones(n - 2), 1.0], -np.ones(n - 1)], [-1, 0, 1])
    ref = NU * (sp.kron(sp.eye(n), T) + sp.kron(T, sp.eye(n)))
    assert abs(F0 - ref).max() <= 1e-16
    x, y = g.node_xy()
    Fw = schur2.f0_jump(g, 0.0, np.ones(g.nq), np.zeros(g.nq))
    assert np.abs(Fw @ np.ones(g.n_0)).max() <= 1e-15
    e, f = g.elements()
    p = -1.0 + (e + 0.5) * g.h                   # cell-centroid x: linear in x
    r = Fw @ p
    interior = (e > 0) & (e < n - 1)
    np.testing.assert_allclose(r[interior], g.h * g.h, rtol=1e-13)
    # convection is skew off the diagonal
    C = (Fw - sp.diags(Fw.diagonal())).toarray()
    assert np.abs(C + C.T).max() <= 1e-16


def test_schur_approximations_share_the_null_space():
    """M2's and LSC's M_S^+ annihilate the pressure constants and return zero-mean fields."""
    s = _sys(6)
    g = s.g
    x, y = g.node_xy()
    wx, wy = fem.cavity_wind(x, y)
    pcd = schur2.TwoFieldPCD(s, NU, fem.pcd_f1(g, NU), schur2.f0_jump(g, NU, wx, wy))
    lsc = schur2.LSCSchur(s)
    rng = np.random.default_rng(1)
    for S in (pcd, lsc):
        for c in (np.r_[np.ones(g.n_k), np.zeros(g.n_0)], np.r_[np.zeros(g.n_k), np.ones(g.n_0)]):
            if S is lsc:
                assert np.abs(S(c)).max() <= 1e-10
        z = S(rng.standard_normal(g.n_p))
        assert abs(z[:g.n_k].mean()) < 1e-12 * np.abs(z).max() and abs(z[g.n_k:].mean()) < 1e-12 * np.abs(z).max()


def test_lsc_is_exact_when_f_is_the_scaling_matrix():
    """With F = H = M (the diagonal velocity mass) the LSC approximation equals the Schur
    complement B M^-1 B^T = Lp exactly, so M_S^+ = Lp^+."""
    s = _sys(5)
    g = s.g
    d = fem.velocity_mass(g).diagonal()
    Mdiag = sp.diags(np.concatenate([d, d]))
    lsc = schur2.LSCSchur(s, F=Mdiag)
    lp = schur2.LpSolver(schur2.two_field_laplacian(s), g.n_k)
    r = np.random.default_rng(2).standard_normal(g.n_p)
    np.testing.assert_allclose(lsc(r), lp(r), atol=1e-10 * np.abs(lp(r)).max())


def test_m2_stagnates_and_lsc_converges():
    """Qualitative paper results on the cavity at nu = 0.01: GMRES with M2 has a fast initial
    phase and then stagnates; with LSC it converges (good for Q2-Q1*)."""
    n = 16
    s = _sys(n)
    g = s.g
    x, y = g.node_xy()
    wx, wy = fem.cavity_wind(x, y)
    hF = oseen.velocity_hierarchy(n, NU)
    nb = np.linalg.norm(s.b)
    M2 = schur2.OseenBlockTriangular(s, hF, schur2.TwoFieldPCD(s, NU, fem.pcd_f1(g, NU), schur2.f0_jump(g, NU, wx, wy)))
    _, rep2 = krylov.gmres(lambda v: s.K @ v, s.b, M2, tol_abs=1e-6 * nb, restart=50, maxit=120)
    assert rep2.history[10] < 1e-2 * rep2.history[0]            # fast initial phase
    assert not rep2.converged and rep2.history[-1] > 1e-3 * rep2.history[0]   # then stagnation
    M3 = schur2.OseenBlockTriangular(s, hF, schur2.LSCSchur(s))
    _, rep3 = krylov.gmres(lambda v: s.K @ v, s.b, M3, tol_abs=1e-6 * nb, restart=50, maxit=120)
    assert rep3.converged and rep3.iterations <= 60
