"""Pins for oracle.fem: closed forms, nnz formulas, paper dof counts, null structure.

Everything here checks the oracle against something other than itself:
hand-derived 1D element matrices (tests/golden/element_1d.txt) combined by
Kronecker products, the paper's Table 1 dof counts (tests/golden/table1_dofs.txt),
Prop 2.1 / Remark 2.2, and analytic properties of the wind.
"""
import os

import numpy as np
import pytest
import scipy.sparse as sp

from oracle import fem

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


def k1d(h):
    return np.array([[7, -8, 1], [-8, 16, -8], [1, -8, 7]]) / (3 * h)


def m1d(h):
    return np.array([[4, 2, -1], [2, 16, 2], [-1, 2, 4]]) * h / 30


def g1d():
    return np.array([[-5, 4, 1], [-1, -4, 5]]) / 6.0


def h1d(h):
    return np.array([[1, 2, 0], [0, 2, 1]]) * h / 6


def ml1d(h):
    return np.array([[2, 1], [1, 2]]) * h / 6


def glob(n, loc, rstride, cstride, rows, cols):
    A = np.zeros((rows, cols))
    r, c = loc.shape
    for e in range(n):
        A[rstride * e:rstride * e + r, cstride * e:cstride * e + c] += loc
    return A


@pytest.mark.parametrize("n", [1, 2, 3, 5])
def test_blocks_match_kronecker_closed_forms(n):
    g = fem.Grid(n)
    h = g.h
    m = g.m
    K = glob(n, k1d(h), 2, 2, m, m)
    M = glob(n, m1d(h), 2, 2, m, m)
    G = glob(n, g1d(), 1, 2, n + 1, m)
    H = glob(n, h1d(h), 1, 2, n + 1, m)
    E = glob(n, np.array([[-1.0, 0.0, 1.0]]), 1, 2, n, m)
    W = glob(n, np.array([[1.0, 4.0, 1.0]]) * h / 6, 1, 2, n, m)
    Ml = glob(n, ml1d(h), 1, 1, n + 1, n + 1)
    L = fem.laplacian(g).toarray()
    np.testing.assert_allclose(L, np.kron(M, K) + np.kron(K, M), atol=1e-13)
    np.testing.assert_allclose(fem.velocity_mass(g).toarray(), np.kron(M, M), atol=1e-15)
    B1, B0 = fem.divergence(g)
    B1, B0 = B1.toarray(), B0.toarray()
    np.testing.assert_allclose(B1[:, :g.nq], -np.kron(H, G), atol=1e-14)
    np.testing.assert_allclose(B1[:, g.nq:], -np.kron(G, H), atol=1e-14)
    np.testing.assert_allclose(B0[:, :g.nq], -np.kron(W, E), atol=1e-14)
    np.testing.assert_allclose(B0[:, g.nq:], -np.kron(E, W), atol=1e-14)
    MQ, Qk, R, Q0 = fem.pressure_mass(g)
    np.testing.assert_allclose(Qk.toarray(), np.kron(Ml, Ml), atol=1e-15)
    Rd = R.toarray()
    assert np.all((np.abs(Rd - h * h / 4) < 1e-15) | (Rd == 0))
    assert np.all((Rd != 0).sum(axis=1) == 4)
    np.testing.assert_allclose(Q0.diagonal(), h * h, rtol=1e-15)


def _nnz(A, rel=1e-12):
    A = A.tocsr()
    return int((np.abs(A.data) > rel * np.abs(A.data).max()).sum())


@pytest.mark.parametrize("n", [8, 16, 32])
def test_nnz_formulas(n):
    """SURVEY §8 nnz table (closed-form counts with Dirichlet identity rows)."""
    s = fem.assemble_system(n)
    assert _nnz(s.Ls) == 60 * n * n - 128 * n + 81
    assert _nnz(s.B1) == 24 * n * n - 20 * n + 4
    assert _nnz(s.B0) == 12 * n * n - 20 * n + 8
    assert _nnz(s.MQ) == (3 * n + 1) ** 2 + 9 * n * n
    assert _nnz(s.K) == 192 * n * n - 336 * n + 186
    # max row lengths: L 25, B1 24, B0 12
    rl = lambda A: np.diff((A.multiply(abs(A) > 1e-12 * abs(A).max())).tocsr().indptr).max()
    assert rl(s.Ls) == 25 and rl(s.B1) == 24 and rl(s.B0) == 12


def test_table1_dof_counts():
    """Velocity dofs 2 (2n+1)^2 equal the paper's Table 1 column."""
    rows = np.loadtxt(os.path.join(GOLDEN, "table1_dofs.txt"), dtype=np.int64)
    for grid, n, nu_paper, _line in rows:
        g = fem.Grid(int(n))
        assert g.n_u == nu_paper
        assert g.n_k == (n + 1) ** 2 and g.n_0 == n * n


@pytest.mark.parametrize("n", [2, 4, 8])
def test_null_structure(n):
    """Prop 2.1 (null M_Q = span k), Remark 2.2 (B^T k = 0),
    reading R17 (B^T [1;0] = B^T [0;1] = 0 after Dirichlet columns are removed)."""
    s = fem.assemble_system(n)
    g = s.g
    k = fem.null_vector_k(g)
    assert np.abs(s.MQ @ k).max() < 1e-15
    assert np.abs(s.B.T @ k).max() < 1e-14
    one_k = np.concatenate([np.ones(g.n_k), np.zeros(g.n_0)])
    one_0 = np.concatenate([np.zeros(g.n_k), np.ones(g.n_0)])
    assert np.abs(s.B.T @ one_k).max() < 1e-14
    assert np.abs(s.B.T @ one_0).max() < 1e-14
    MQd = s.MQ.toarray()
    ev = np.linalg.eigvalsh(MQd)
    assert ev[0] < 1e-14 * ev[-1] and ev[1] > 1e-6 * ev[-1]    # rank n_p - 1
    Kd = s.K.toarray()
    sv = np.linalg.svd(Kd, compute_uv=False)
    assert (sv < 1e-10 * sv[0]).sum() == 2                       # 2-D null space (R17)


def test_schur_of_mass_interior_stencil():
    """S_k = Qk - R^T Q0^{-1} R has the interior stencil (h^2/144)[[-5,-2,-5],[-2,28,-2],[-5,-2,-5]]
    and zero row sums (SURVEY §8(c) pin)."""
    n = 6
    g = fem.Grid(n)
    MQ, Qk, R, Q0 = fem.pressure_mass(g)
    S = (Qk - R.T @ sp.diags(1.0 / Q0.diagonal()) @ R).toarray()
    h = g.h
    a, c = 3, 3
    p = a + (n + 1) * c
    st = np.array([[-5, -2, -5], [-2, 28, -2], [-5, -2, -5]]) * h * h / 144
    for dc in (-1, 0, 1):
        for da in (-1, 0, 1):
            assert S[p, (a + da) + (n + 1) * (c + dc)] == pytest.approx(st[dc + 1, da + 1], abs=1e-15)
    np.testing.assert_allclose(S.sum(axis=1), 0.0, atol=1e-15)


def test_wind_and_convection_properties():
    """w of config c4 is divergence-free with w.n = 0 on the boundary, so the Galerkin
    convection matrices are exactly skew-symmetric (int w.grad(uv) = 0); w = 0 gives F = nu L."""
    x = np.linspace(-1, 1, 7)
    X, Y = np.meshgrid(x, x)
    eps = 1e-6
    wx1, _ = fem.cavity_wind(X + eps, Y); wx0, _ = fem.cavity_wind(X - eps, Y)
    _, wy1 = fem.cavity_wind(X, Y + eps); _, wy0 = fem.cavity_wind(X, Y - eps)
    assert np.abs((wx1 - wx0 + wy1 - wy0) / (2 * eps)).max() < 1e-8
    for n in (2, 4):
        g = fem.Grid(n)
        N = fem.convection(g).toarray()
        assert np.abs(N + N.T).max() < 1e-14
        F1 = fem.pcd_f1(g, 0.01).toarray()
        F1s = fem.pcd_f1(g, 0.01, wind=lambda x, y: (0 * x, 0 * y)).toarray()
        assert np.abs((F1 - F1s) + (F1 - F1s).T).max() < 1e-14
        zero = lambda x, y: (0 * x, 0 * y)
        s0 = fem.assemble_system(n, nu=0.5, wind=zero)
        sL = fem.assemble_system(n)
        Lint = sL.Ls.toarray(); F0 = s0.Ls.toarray()
        bn = g.boundary_nodes()
        inter = np.setdiff1d(np.arange(g.nq), bn)
        np.testing.assert_allclose(F0[np.ix_(inter, inter)], 0.5 * Lint[np.ix_(inter, inter)], atol=1e-14)


def test_convection_quadrature_exact():
    """The c4 wind is biquadratic, so 3x3 Gauss is exact for N (degree <= 5 per direction):
    compare one element matrix with a 6x6 Gauss rule evaluated independently."""
    n = 3
    g = fem.Grid(n)
    N = fem.convection(g).toarray()
    xg, wg = np.polynomial.legendre.leggauss(6)
    xg = 0.5 * (xg + 1.0); wg = 0.5 * wg
    e, f = 1, 2
    h = g.h
    loc = np.zeros((9, 9))
    for qx in range(6):
        for qy in range(6):
            xi, et = xg[qx], xg[qy]
            X, Y = -1 + (e + xi) * h, -1 + (f + et) * h
            wx, wy = fem.cavity_wind(X, Y)
            v, d = fem.q2_basis_1d(np.array([xi, et]))
            phi = np.array([v[a, 0] * v[b, 1] for b in range(3) for a in range(3)])
            dx = np.array([d[a, 0] / h * v[b, 1] for b in range(3) for a in range(3)])
            dy = np.array([v[a, 0] * d[b, 1] / h for b in range(3) for a in range(3)])
            loc += wg[qx] * wg[qy] * h * h * np.outer(phi, wx * dx + wy * dy)
    # isolate element (1,2): assemble the same element contribution from the 6x6 rule and compare
    # against N restricted to the element's interior node (local 4), which only that element touches
    d2 = [(2 * e + a) + g.m * (2 * f + b) for b in range(3) for a in range(3)]
    i4 = d2[4]
    np.testing.assert_allclose(N[i4, d2], loc[4], atol=1e-14)


def test_lifting_consistency():
    """The lifted right-hand side is consistent with the null space of the enclosed system:
    sum(g1) = sum(g0) = 0 because the lid is tangential (reading R3, oint u.n = 0)."""
    s = fem.assemble_system(8)
    g = s.g
    gp = s.b[g.n_u:]
    assert abs(gp[:g.n_k].sum()) < 1e-14
    assert abs(gp[g.n_k:].sum()) < 1e-14
    assert np.abs(gp).max() > 1e-3                             # g != 0 (reading R3)
    # Dirichlet values are carried by the identity rows
    bn = g.boundary_nodes()
    np.testing.assert_array_equal(s.b[bn], s.u_bc[bn])
    x, _ = g.node_xy()
    top = bn[np.isclose(g.node_xy()[1][bn], 1.0)]
    np.testing.assert_allclose(s.b[top], 1 - x[top] ** 4)
