"""oracle.precond — block preconditioners for the Q2-Q1* saddle systems.

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

Stokes, block diagonal P = diag(M, M_S) (Eq. stokes_pre):
  P1 = diag(A, M_Q) with exact solves; the M_Q block through the augmented
       system [[M_Q, k], [k^T, 0]]            -> StokesP1
  P2 = diag(one V-cycle, 20 Chebyshev-SGS steps) (AMG -> GMG per
       BASELINE.json, reading R9; k-constraint by Pi C Pi, reading R6) -> StokesP2
Plain Taylor-Hood Q2-Q1 on the same mesh (the local-conservation contrast):
  diag(one V-cycle, m_p Chebyshev-Jacobi steps on the Q1 mass Q_k over [1/4, 9/4]) on the
  reduced system [A B1^T; B1 0] (reading R13)                -> StokesP2Plain
"""
from __future__ import annotations

import numpy as np
import scipy.sparse.linalg as spla

from . import fem, mass, mg


class StokesP1:
    """z_u = A^{-1} r_u (sparse direct), z_p = augmented exact M_Q solve."""

    def __init__(self, s: fem.SaddleSystem):
        self.n_u = s.g.n_u
        self.lu = spla.splu(s.Av.tocsc())
        self.aug = mass.AugmentedMassSolver(s.MQ, fem.null_vector_k(s.g))

    def __call__(self, r):
        return np.concatenate([self.lu.solve(r[:self.n_u]), self.aug.solve(r[self.n_u:])])


class StokesP2:
    """z_u = one Q2-GMG V-cycle per component, z_p = Pi C Pi r_p (R6, R7, R9)."""

    def __init__(self, s: fem.SaddleSystem, a: float, m: int = 20, n_coarse: int = 2,
                 lo: float = 0.16, hi: float = 1.6, degree: int = 3, hierarchy=None):
        self.n_u = s.g.n_u
        self.h = hierarchy if hierarchy is not None else \
            mg.Hierarchy(s.g.n, n_coarse=n_coarse, lo=lo, hi=hi, degree=degree)
        self.MQ = s.MQ
        self.col = mass.colours(s.g)
        self.k = fem.null_vector_k(s.g)
        self.a, self.m = a, m

    def velocity(self, r_u):
        return self.h.apply_velocity(r_u)

    def pressure(self, r_p):
        return mass.pi_c_pi(self.MQ, r_p, self.a, self.m, self.col, self.k)

    def __call__(self, r):
        return np.concatenate([self.velocity(r[:self.n_u]), self.pressure(r[self.n_u:])])


class StokesP2Plain:
    """Plain Q2-Q1 Stokes preconditioner on [u; p_1]: z_u = one V-cycle per component,
    z_p = m_p-step Chebyshev-Jacobi approximation of Q_k^{-1} (interval [1/4, 9/4], reading R13)."""

    def __init__(self, s: fem.SaddleSystem, mp_steps: int = 10, hierarchy=None):
        self.n_u = s.g.n_u
        self.h = hierarchy if hierarchy is not None else mg.Hierarchy(s.g.n)
        self.Qk = s.Qk
        self.dinv = 1.0 / s.Qk.diagonal()
        self.mp_steps = mp_steps

    def __call__(self, r):
        zp, _ = mg.chebyshev_smooth(self.Qk, self.dinv, r[self.n_u:], None, 0.25, 2.25, self.mp_steps)
        return np.concatenate([self.h.apply_velocity(r[:self.n_u]), zp])


def plain_system(s: fem.SaddleSystem):
    """Plain Taylor-Hood operator [A B1^T; B1 0] and right-hand side [f; g1] (P0 dropped)."""
    return fem.reduced_operator(s), s.b[:s.g.n_u + s.g.n_k].copy()


class StokesP3:
    """NEXT-2 hybrid: z_u = one Q2-GMG V-cycle per component (as P2),
    z_p = exact augmented M_Q solve (as P1)."""

    def __init__(self, s: fem.SaddleSystem, hierarchy=None):
        self.n_u = s.g.n_u
        self.h = hierarchy if hierarchy is not None else mg.Hierarchy(s.g.n)
        self.aug = mass.SparseAugmentedMassSolver(s.MQ, fem.null_vector_k(s.g))

    def __call__(self, r):
        return np.concatenate([self.h.apply_velocity(r[:self.n_u]), self.aug.solve(r[self.n_u:])])
