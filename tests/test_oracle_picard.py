"""Pins of oracle.picard: nodal-wind convection with 4 x 4 Gauss points, the
Q1 PCD operator with a nodal wind, the exact bordered Oseen solve and the Picard loop."""
import numpy as np
import pytest

from oracle import fem, picard


def _random_q2_wind(g, seed):
    rng = np.random.default_rng(seed)
    return rng.standard_normal(g.nq), rng.standard_normal(g.nq)


def test_nodal_cavity_wind_reproduces_analytic_convection():
    """The c4 wind (2y(1-x^2), -2x(1-y^2)) lies in Q2, so its nodal interpolant gives the same N
    and F1 as the analytic-wind assembly pinned in test_oracle_fem."""
    g = fem.Grid(6)
    x, y = g.node_xy()
    wx, wy = fem.cavity_wind(x, y)
    N_ref = fem.convection(g)
    N = picard.convection_nodal(g, wx, wy)
    assert abs(N - N_ref).max() <= 1e-14 * abs(N_ref).max()
    F1_ref = fem.pcd_f1(g, 0.01)
    F1 = picard.pcd_f1_nodal(g, 0.01, wx, wy)
    assert abs(F1 - F1_ref).max() <= 1e-14 * abs(F1_ref).max()


def test_four_point_gauss_is_exact_for_q2_winds():
    """With a Q2 wind the integrand has degree <= 6 per direction: 4 x 4 Gauss equals 6 x 6 Gauss;
    3 x 3 Gauss (the Stokes/c4 rule) does not."""
    g = fem.Grid(3)
    wx, wy = _random_q2_wind(g, 1)
    N4 = picard.convection_nodal(g, wx, wy)
    x6, w6 = picard.gauss_1d(6)
    N6 = picard.convection_nodal(g, wx, wy, x6, w6)
    assert abs(N4 - N6).max() <= 1e-13 * abs(N6).max()
    x3, w3 = picard.gauss_1d(3)
    N3 = picard.convection_nodal(g, wx, wy, x3, w3)
    assert abs(N3 - N6).max() > 1e-6 * abs(N6).max()


def test_convection_annihilates_constants_and_matches_trilinear_form():
    """N(w) 1 = 0 (grad 1 = 0) for any wind, and v^T N(w) u equals the trilinear form
    sum_e int (w . grad u) v evaluated pointwise from interpolated fields with a 6 x 6 rule."""
    g = fem.Grid(3)
    wx, wy = _random_q2_wind(g, 2)
    N = picard.convection_nodal(g, wx, wy)
    assert np.abs(N @ np.ones(g.nq)).max() <= 1e-13 * abs(N).max()
    rng = np.random.default_rng(3)
    u, v = rng.standard_normal(g.nq), rng.standard_normal(g.nq)
    x6, w6 = picard.gauss_1d(6)
    t = picard.tabulate(g.h, x6, w6)
    e, f = g.elements()
    d = g.q2_dofs(e, f)
    wxq, wyq = wx[d] @ t["phi"], wy[d] @ t["phi"]
    ux, uy = u[d] @ t["phix"], u[d] @ t["phiy"]
    vq = v[d] @ t["phi"]
    tri = np.sum(t["W"][None, :] * (wxq * ux + wyq * uy) * vq)
    assert abs(v @ (N @ u) - tri) <= 1e-12 * abs(tri)


def test_exact_oseen_solve_and_stokes_limit():
    """The bordered solve satisfies K x = b with zero-sum pressures; with w = 0 the Oseen velocity
    is the Stokes velocity (the velocity of -nu lap u + grad p = 0 does not depend on nu)."""
    n = 6
    g = fem.Grid(n)
    s = picard.oseen_system(n, 0.01, *_random_q2_wind(g, 4))
    x = picard.solve_exact(s)
    assert np.linalg.norm(s.K @ x - s.b) <= 1e-10 * np.linalg.norm(s.b)
    assert abs(x[g.n_u:g.n_u + g.n_k].sum()) < 1e-10 and abs(x[g.n_u + g.n_k:].sum()) < 1e-10
    xs = picard.solve_exact(fem.assemble_system(n))
    x0 = picard.solve_exact(picard.oseen_system(n, 0.01, np.zeros(g.nq), np.zeros(g.nq)))
    np.testing.assert_allclose(x0[:g.n_u], xs[:g.n_u], atol=1e-10 * np.abs(xs[:g.n_u]).max())


def test_picard_converges_to_a_discrete_navier_stokes_solution():
    """At nu = 0.1 the Picard map contracts; the limit solves the discrete Navier-Stokes system
    F(u) u + B^T p = f(u), B u = g (re-assembled at the limit)."""
    n = 8
    g = fem.Grid(n)
    xs, _ = picard.picard(n, 0.1, steps=16)
    diffs = [np.linalg.norm(xs[k][:g.n_u] - xs[k - 1][:g.n_u]) for k in range(1, len(xs))]
    assert diffs[-1] < 1e-12 * np.linalg.norm(xs[-1][:g.n_u])
    assert all(diffs[k + 1] < 0.5 * diffs[k] for k in range(10))   # linear contraction above rounding
    u = xs[-1][:g.n_u]
    s = picard.oseen_system(n, 0.1, u[:g.nq], u[g.nq:])
    assert np.linalg.norm(s.K @ xs[-1] - s.b) <= 1e-8 * np.linalg.norm(s.b)
