"""oracle.oseen — Oseen preconditioners and the two-stage PCD driver.

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

* F V-cycle: Q2 GMG on F_s = nu L + N with the ellipse-aware Chebyshev smoother (reading R9'),
  exact coarse solve at n_c = 32 (or n when smaller)
* PCD Step-I Schur complement: M_S1^{-1} = Ap^{-1} F1 Mp^{-1} (paper order, reading R11):
  Mp^{-1} = m_p-step Chebyshev-Jacobi on the Q1 mass over [1/4, 9/4] (reading R13),
  F1, Ap^{-1} = one Q1-GMG V-cycle on Ap = B1 Mdiag^{-1} B1^T plus a mean-zero
  projection (reading R13)
* block upper-triangular preconditioners M = [[M_F, B^T], [0, -M_S]]:
  Step I  [[V_F, B1^T], [0, -M_S1]] on the reduced system
  Step II M1 = [[V_F, B^T], [0, -(1/nu) M_Q~]] with M_Q~^{-1} = Pi C Pi
* two-stage driver and the Prop 3.3 bound
"""
from __future__ import annotations

import numpy as np
import scipy.sparse as sp

from . import fem, krylov, mass, mg


def velocity_hierarchy(n: int, nu: float, n_coarse: int = 32, wind=fem.cavity_wind):
    """Q2-GMG on F_s = nu L + N(w) with the ellipse smoother (reading R9')."""
    op = lambda g: (nu * fem.laplacian(g) + fem.convection(g, wind)).tocsr()
    skew = lambda g: fem.convection(g, wind)
    return mg.Hierarchy(n, n_coarse=min(n_coarse, n), operator=op, skew=skew)


def q1_prolongation_1d(n_coarse: int):
    """P1d[k, I] = N^c_I(x^f_k): coarse Q1 hat functions at the fine Q1 vertices (nested)."""
    nf = 2 * n_coarse
    hc = 2.0 / n_coarse
    xf = -1.0 + np.arange(nf + 1) * (2.0 / nf)
    P = np.zeros((nf + 1, n_coarse + 1))
    for k, x in enumerate(xf):
        e = min(int(np.floor((x + 1.0) / hc + 1e-12)), n_coarse - 1)
        xi = (x - (-1.0 + e * hc)) / hc
        val, _ = fem.q1_basis_1d(np.array([xi]))
        P[k, e] += val[0, 0]
        P[k, e + 1] += val[1, 0]
    P[np.abs(P) < 1e-15] = 0.0
    return sp.csr_matrix(P)


def pcd_ap_grid(n: int):
    """Ap = B1 Mdiag^{-1} B1^T on an n x n grid, B1 with Dirichlet velocity columns removed
    (reading R12: Mdiag = diagonal of the consistent velocity mass)."""
    g = fem.Grid(n)
    B1, _ = fem.divergence(g)
    keep = np.ones(g.n_u)
    bn = g.boundary_nodes()
    keep[bn] = 0.0
    keep[bn + g.nq] = 0.0
    B1 = (B1 @ sp.diags(keep)).tocsr()
    d = fem.velocity_mass(g).diagonal()
    Dm = sp.diags(1.0 / np.concatenate([d, d]))
    Ap = (B1 @ Dm @ B1.T).tocsr()
    Ap.sort_indices()
    return Ap


class ApHierarchy:
    """One Q1-GMG V-cycle for the singular Ap (null space: constants), reading R13:
    rediscretised Ap_l, nested Q1 interpolation (no boundary rows: pressure has no BC),
    Chebyshev degree 3 in D^{-1}Ap on [0.16, 1.6], coarse pseudo-inverse at n_c = 2."""

    def __init__(self, n: int, n_coarse: int = 2, lo: float = 0.16, hi: float = 1.6, degree: int = 3):
        self.levels = []
        m = n
        while True:
            A = pcd_ap_grid(m)
            self.levels.append({"n": m, "A": A, "dinv": 1.0 / A.diagonal()})
            if m <= n_coarse:
                break
            m //= 2
        for l in range(len(self.levels) - 1):
            P1 = q1_prolongation_1d(self.levels[l + 1]["n"])
            self.levels[l]["P"] = sp.kron(P1, P1).tocsr()
        self.coarse_pinv = np.linalg.pinv(self.levels[-1]["A"].toarray())
        self.lo, self.hi, self.degree = lo, hi, degree

    def vcycle(self, b, l: int = 0):
        lev = self.levels[l]
        if l == len(self.levels) - 1:
            return self.coarse_pinv @ b
        A, dinv, P = lev["A"], lev["dinv"], lev["P"]
        x, r = mg.chebyshev_smooth(A, dinv, b, None, self.lo, self.hi, self.degree)
        x = x + P @ self.vcycle(P.T @ r, l + 1)
        x, _ = mg.chebyshev_smooth(A, dinv, b, x, self.lo, self.hi, self.degree)
        return x

    def solve(self, b):
        """Ap^{-1} b ~ V(b) projected to mean zero (Euclidean mean)."""
        z = self.vcycle(b)
        return z - z.mean()


class PCDSchur:
    """M_S1^{-1} r = Ap^{-1} (F1 (Mp^{-1} r)), paper order of Eq. (discrete-commutator1x)."""

    def __init__(self, s: fem.SaddleSystem, nu: float, mp_steps: int = 10, wind=fem.cavity_wind):
        g = s.g
        self.Mp = s.Qk
        self.mp_dinv = 1.0 / s.Qk.diagonal()
        self.mp_steps = mp_steps
        self.F1 = fem.pcd_f1(g, nu, wind)
        self.Ap = ApHierarchy(g.n)

    def mp_solve(self, r):
        x, _ = mg.chebyshev_smooth(self.Mp, self.mp_dinv, r, None, 0.25, 2.25, self.mp_steps)
        return x

    def __call__(self, r):
        return self.Ap.solve(self.F1 @ self.mp_solve(r))


class OseenPCD1:
    """Step-I preconditioner on the reduced vector [u; p1]: z_p = -M_S1^{-1} r_p,
    z_u = V_F(r_u - B1^T z_p)  (block upper-triangular)."""

    def __init__(self, s, hF, schur):
        self.n_u = s.g.n_u
        self.B1T = s.B1.T.tocsr()
        self.hF = hF
        self.S = schur

    def __call__(self, r):
        zp = -self.S(r[self.n_u:])
        zu = self.hF.apply_velocity(r[:self.n_u] - self.B1T @ zp)
        return np.concatenate([zu, zp])


class OseenM1:
    """M1 = [[V_F, B^T], [0, -(1/nu) M_Q~]]: z_p = -nu Pi C Pi r_p,
    z_u = V_F(r_u - B^T z_p)."""

    def __init__(self, s, hF, nu, a, m=20):
        self.n_u = s.g.n_u
        self.BT = s.B.T.tocsr()
        self.hF = hF
        self.nu = nu
        self.MQ = s.MQ
        self.col = mass.colours(s.g)
        self.k = fem.null_vector_k(s.g)
        self.a, self.m = a, m

    def __call__(self, r):
        zp = -self.nu * mass.pi_c_pi(self.MQ, r[self.n_u:], self.a, self.m, self.col, self.k)
        zu = self.hF.apply_velocity(r[:self.n_u] - self.BT @ zp)
        return np.concatenate([zu, zp])


def two_stage(s, nu, a, eta=1e-6, c=10.0, restart=50, maxit=2000, hF=None, schur=None):
    """Two-stage PCD, readings R14-R16.

    Step I: GMRES on the reduced system [F B1^T; B1 0][u; q1] = [f; g1] from 0 with the PCD
    preconditioner, stopped at ||r|| <= c eta ||b_red||.
    Step II: GMRES on the full system with M1 from [u1*; q1*; 0], stopped at ||r|| <= eta ||b||.
    Returns x, (report I, report II), ||z*|| (residual of the intermediate solution in the full
    system) and the Prop 3.3 bound sqrt(c^2 eta^2 ||b_red||^2 + ||g0 - B0 u1*||^2)."""
    g = s.g
    nr = g.n_u + g.n_k
    if hF is None:
        hF = velocity_hierarchy(g.n, nu)
    if schur is None:
        schur = PCDSchur(s, nu)
    Kr = fem.reduced_operator(s)
    b_red = s.b[:nr]
    M_I = OseenPCD1(s, hF, schur)
    x1, rep1 = krylov.gmres(lambda v: Kr @ v, b_red, M_I, tol_abs=c * eta * np.linalg.norm(b_red),
                            restart=restart, maxit=maxit)
    x0 = np.concatenate([x1, np.zeros(g.n_0)])
    zstar = np.linalg.norm(s.b - s.K @ x0)
    g0 = s.b[nr:]
    bound = np.sqrt((c * eta * np.linalg.norm(b_red)) ** 2 + np.linalg.norm(g0 - s.B0 @ x1[:g.n_u]) ** 2)
    M_II = OseenM1(s, hF, nu, a)
    x, rep2 = krylov.gmres(lambda v: s.K @ v, s.b, M_II, tol_abs=eta * np.linalg.norm(s.b),
                           restart=restart, maxit=maxit, x0=x0)
    return x, (rep1, rep2), zstar, bound
