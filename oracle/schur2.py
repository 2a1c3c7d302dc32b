"""oracle.schur2 — SURVEY §8(f) NEXT-4: the two alternative Oseen Schur-complement approximations
for the two-field (Q1 + P0) pressure.

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

* M2 = [[F, B^T], [0, -M_S]] with the two-field PCD approximation (Eq. twofield-pcd)
      M_S = diag(Q1, Q0) diag(F1^{-1}, F0^{-1}) B M^{-1} B^T,
  i.e. M_S^+ r = Lp^+ diag(F1 Q1^{-1}, F0 Q0^{-1}) r with the two-field pressure Laplacian
  Lp = B M^{-1} B^T (M = diagonal of the velocity mass).  The paper reports that GMRES
  with M2 stagnates after a fast initial phase.
* M3 = [[F, B^T], [0, -M_S]] with the least-squares commutator (Eq. lsc-definition)
      M_S = (B H^{-1} B^T) (B M^{-1} F H^{-1} B^T)^{-1} (B M^{-1} B^T),
  i.e. M_S^+ r = Lp^+ (B M^{-1} F M^{-1} B^T) Lp^+ r with H = M (reading R26: the boundary scaling D
  is unspecified; D = I).
Both M_S have the null space of B F^{-1} B^T (the two pressure constants).

Readings: R25 the P0 convection-diffusion operator F0 ("jumps in pressure across
inter-element boundaries"): cell-centred finite volumes on the squares — diffusion
nu sum_{interior edges} (p_i - p_j) (edge length / centroid distance = 1), convection by the central
edge flux (w_e . n_e) h (p_j - p_i) / 2 with w_e the wind at the edge midpoint (a Q2 node), natural
(no-flux) boundary like F1 (R13); Q0 = h^2 I.  Q1^{-1} is applied as in the Step-I PCD (R13:
10 Chebyshev-Jacobi steps on Q_k); Lp^+ exactly (sparse LU bordered by the two constants).
"""
from __future__ import annotations

import numpy as np
import scipy.sparse as sp
import scipy.sparse.linalg as spla

from . import fem, mg


def two_field_laplacian(s: fem.SaddleSystem):
    """Lp = B M^{-1} B^T on [Q1; P0] with the Dirichlet velocity columns removed from B."""
    d = fem.velocity_mass(s.g).diagonal()
    Dm = sp.diags(1.0 / np.concatenate([d, d]))
    Lp = (s.B @ Dm @ s.B.T).tocsr()
    Lp.sort_indices()
    return Lp


def f0_jump(g: fem.Grid, nu: float, wx_nodal, wy_nodal):
    """P0 convection-diffusion operator F0 (reading R25) for a wind given at the Q2 nodes."""
    n, m, h = g.n, g.m, g.h
    rows, cols, vals = [], [], []
    for f in range(n):
        for e in range(n):
            T = e + n * f
            # (neighbour cell, midpoint node of the shared edge, outward normal)
            for de, df, node, nx, ny in ((1, 0, (2 * e + 2) + m * (2 * f + 1), 1.0, 0.0),
                                         (-1, 0, (2 * e) + m * (2 * f + 1), -1.0, 0.0),
                                         (0, 1, (2 * e + 1) + m * (2 * f + 2), 0.0, 1.0),
                                         (0, -1, (2 * e + 1) + m * (2 * f), 0.0, -1.0)):
                e2, f2 = e + de, f + df
                if not (0 <= e2 < n and 0 <= f2 < n):
                    continue
                T2 = e2 + n * f2
                flux = (wx_nodal[node] * nx + wy_nodal[node] * ny) * h / 2.0
                rows += [T, T]; cols += [T, T2]; vals += [nu - flux, -nu + flux]
    F0 = sp.coo_matrix((vals, (rows, cols)), shape=(g.n_0, g.n_0)).tocsr()
    F0.sum_duplicates(); F0.sort_indices()
    return F0


class LpSolver:
    """Lp^+ r: project r onto the range (zero mean in each field), solve with Lp bordered by
    the two constants (sparse LU), zero-mean result."""

    def __init__(self, Lp, n_k: int):
        n_p = Lp.shape[0]
        C = np.zeros((n_p, 2)); C[:n_k, 0] = 1.0; C[n_k:, 1] = 1.0
        Cs = sp.csr_matrix(C)
        self.lu = spla.splu(sp.bmat([[Lp, Cs], [Cs.T, None]]).tocsc())
        self.n_k, self.n_p = n_k, n_p

    def project(self, r):
        r = np.array(r, dtype=float)
        r[:self.n_k] -= r[:self.n_k].mean()
        r[self.n_k:] -= r[self.n_k:].mean()
        return r

    def __call__(self, r):
        return self.lu.solve(np.concatenate([self.project(r), [0.0, 0.0]]))[:self.n_p]


class TwoFieldPCD:
    """M_S^+ r = Lp^+ [F1 Q1^{-1} r_1 ; F0 Q0^{-1} r_0] (two-field PCD)."""

    def __init__(self, s: fem.SaddleSystem, nu: float, F1, F0, mp_steps: int = 10):
        g = s.g
        self.n_k = g.n_k
        self.Qk, self.q_dinv, self.mp_steps = s.Qk, 1.0 / s.Qk.diagonal(), mp_steps
        self.h2 = g.h * g.h
        self.F1, self.F0 = F1, F0
        self.Lp = LpSolver(two_field_laplacian(s), g.n_k)

    def __call__(self, r):
        t1, _ = mg.chebyshev_smooth(self.Qk, self.q_dinv, r[:self.n_k], None, 0.25, 2.25, self.mp_steps)
        t0 = r[self.n_k:] / self.h2
        return self.Lp(np.concatenate([self.F1 @ t1, self.F0 @ t0]))


class LSCSchur:
    """M_S^+ r = Lp^+ (B M^{-1} F M^{-1} B^T) Lp^+ r (LSC with H = M, reading R26)."""

    def __init__(self, s: fem.SaddleSystem, F=None):
        g = s.g
        d = fem.velocity_mass(g).diagonal()
        self.minv = 1.0 / np.concatenate([d, d])
        self.B, self.BT = s.B, s.B.T.tocsr()
        self.F = s.Av if F is None else F
        self.Lp = LpSolver(two_field_laplacian(s), g.n_k)

    def __call__(self, r):
        t = self.Lp(r)
        w = self.F @ (self.minv * (self.BT @ t))
        return self.Lp(self.B @ (self.minv * w))


class OseenBlockTriangular:
    """[[V_F, B^T], [0, -M_S]]: z_p = -M_S^+ r_p, z_u = V_F(r_u - B^T z_p)."""

    def __init__(self, s, hF, schur):
        self.n_u = s.g.n_u
        self.BT = s.B.T.tocsr()
        self.hF, self.S = hF, schur

    def __call__(self, r):
        zp = -self.S(r[self.n_u:])
        zu = self.hF.apply_velocity(r[:self.n_u] - self.BT @ zp)
        return np.concatenate([zu, zp])
