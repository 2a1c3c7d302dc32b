"""oracle.picard — SURVEY §8(f) NEXT-3: the Picard (fixed-point) outer loop of the steady
Navier-Stokes cavity ("5 fixed-point iterations of the discretised Navier-Stokes system
starting from the corresponding Stokes flow solution"; P:855-857 for the cavity).

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

Picard step k solves the Oseen system of P:734-773 with the frozen wind w = u^{k-1}, the previous
discrete Q2 velocity (including its boundary values).  A Q2 wind makes the convection integrand
int (w . grad phi_j) phi_i a polynomial of degree 6 in the undifferentiated direction, so it is
integrated with 4 x 4 Gauss points per square (exact to degree 7).  Each Oseen
system is solved exactly (sparse LU of the system bordered by the two pressure constants that
span its null space, reading R17), so the iterates are the Picard iterates themselves.
"""
from __future__ import annotations

import numpy as np
import scipy.sparse as sp
import scipy.sparse.linalg as spla

from . import fem

# 4-point Gauss-Legendre on [0, 1] (exact for degree 7)
_G4 = np.sqrt(3.0 / 7.0 - 2.0 / 7.0 * np.sqrt(6.0 / 5.0))
_G4b = np.sqrt(3.0 / 7.0 + 2.0 / 7.0 * np.sqrt(6.0 / 5.0))
GAUSS4_X = 0.5 + 0.5 * np.array([-_G4b, -_G4, _G4, _G4b])
GAUSS4_W = 0.5 * np.array([(18.0 - np.sqrt(30.0)) / 36.0, (18.0 + np.sqrt(30.0)) / 36.0,
                           (18.0 + np.sqrt(30.0)) / 36.0, (18.0 - np.sqrt(30.0)) / 36.0])


def gauss_1d(npts: int):
    """npts-point Gauss-Legendre rule on [0, 1] (numpy's rule mapped; used for cross-checks)."""
    x, w = np.polynomial.legendre.leggauss(npts)
    return 0.5 + 0.5 * x, 0.5 * w


def tabulate(h: float, gx=GAUSS4_X, gw=GAUSS4_W):
    """Q2 / Q1 basis values and derivatives at the tensor Gauss points of one square of side h:
    arrays (nbasis, nq) with q = qx + npts qy, weights W (nq,) including the Jacobian h^2."""
    npts = len(gx)
    v2, d2 = fem.q2_basis_1d(gx)
    v1, d1 = fem.q1_basis_1d(gx)
    qx = np.tile(np.arange(npts), npts)
    qy = np.repeat(np.arange(npts), npts)
    W = (gw[qx] * gw[qy]) * h * h
    phi = np.empty((9, qx.size)); phix = np.empty_like(phi); phiy = np.empty_like(phi)
    for beta in range(3):
        for alpha in range(3):
            a = alpha + 3 * beta
            phi[a] = v2[alpha, qx] * v2[beta, qy]
            phix[a] = d2[alpha, qx] / h * v2[beta, qy]
            phiy[a] = v2[alpha, qx] * d2[beta, qy] / h
    psi = np.empty((4, qx.size)); psix = np.empty_like(psi); psiy = np.empty_like(psi)
    for c in range(2):
        for a in range(2):
            k = a + 2 * c
            psi[k] = v1[a, qx] * v1[c, qy]
            psix[k] = d1[a, qx] / h * v1[c, qy]
            psiy[k] = v1[a, qx] * d1[c, qy] / h
    return dict(W=W, phi=phi, phix=phix, phiy=phiy, psi=psi, psix=psix, psiy=psiy)


def _wind_at_quad(g: fem.Grid, t, wx_nodal, wy_nodal):
    """Q2-interpolated wind at the quadrature points of every element: (nel, nq) each."""
    e, f = g.elements()
    d = g.q2_dofs(e, f)
    return d, wx_nodal[d] @ t["phi"], wy_nodal[d] @ t["phi"]


def convection_nodal(g: fem.Grid, wx_nodal, wy_nodal, gx=GAUSS4_X, gw=GAUSS4_W):
    """Scalar Q2 convection N_ij = int (w_h . grad phi_j) phi_i for a Q2 nodal wind w_h
    (Eq. generic-conv-diff), 4 x 4 Gauss points per square."""
    t = tabulate(g.h, gx, gw)
    d, wq_x, wq_y = _wind_at_quad(g, t, np.asarray(wx_nodal, float), np.asarray(wy_nodal, float))
    loc = np.einsum("q,eq,jq,iq->eij", t["W"], wq_x, t["phix"], t["phi"]) + \
        np.einsum("q,eq,jq,iq->eij", t["W"], wq_y, t["phiy"], t["phi"])
    return fem._assemble(loc, d, d, (g.nq, g.nq))


def pcd_f1_nodal(g: fem.Grid, nu: float, wx_nodal, wy_nodal):
    """F1_ij = nu int grad psi_j . grad psi_i + int (w_h . grad psi_j) psi_i on Q1 with a Q2
    nodal wind (natural boundary, reading R13), 4 x 4 Gauss points."""
    t = tabulate(g.h)
    e, f = g.elements()
    d1 = g.q1_dofs(e, f)
    _, wq_x, wq_y = _wind_at_quad(g, t, np.asarray(wx_nodal, float), np.asarray(wy_nodal, float))
    diff = np.einsum("q,iq,jq->ij", t["W"], t["psix"], t["psix"]) + \
        np.einsum("q,iq,jq->ij", t["W"], t["psiy"], t["psiy"])
    conv = np.einsum("q,eq,jq,iq->eij", t["W"], wq_x, t["psix"], t["psi"]) + \
        np.einsum("q,eq,jq,iq->eij", t["W"], wq_y, t["psiy"], t["psi"])
    return fem._assemble(nu * diff[None, :, :] + conv, d1, d1, (g.n_k, g.n_k))


def oseen_system(n: int, nu: float, wx_nodal, wy_nodal, bc: str = "lid") -> fem.SaddleSystem:
    """The Oseen system of P:734-773 (lifting and Dirichlet rows as reading R2) with a nodal wind."""
    g = fem.Grid(n)
    N = convection_nodal(g, wx_nodal, wy_nodal)
    return fem.assemble_system(n, bc=bc, nu=nu, convection_matrix=N)


def solve_exact(s: fem.SaddleSystem):
    """x with K x = b and zero-sum Q1 and P0 pressures: sparse LU of K bordered by the two
    pressure constants (null(K) = null(K^T) = span of them for enclosed flow, R17)."""
    g = s.g
    C = np.zeros((g.N, 2))
    C[g.n_u:g.n_u + g.n_k, 0] = 1.0
    C[g.n_u + g.n_k:, 1] = 1.0
    Cs = sp.csr_matrix(C)
    Kb = sp.bmat([[s.K, Cs], [Cs.T, None]]).tocsc()
    sol = spla.splu(Kb).solve(np.concatenate([s.b, [0.0, 0.0]]))
    return sol[:g.N]


def picard(n: int, nu: float, steps: int = 5, bc: str = "lid"):
    """Picard iterates [x^0 (Stokes), x^1, ..., x^steps]; step k uses the wind u^{k-1}.
    Returns (iterates, systems) with systems[k] the Oseen system solved at step k (k >= 1)."""
    g = fem.Grid(n)
    s0 = fem.assemble_system(n, bc=bc)
    xs = [solve_exact(s0)]
    systems = [s0]
    for _ in range(steps):
        u = xs[-1][:g.n_u]
        s = oseen_system(n, nu, u[:g.nq], u[g.nq:], bc=bc)
        xs.append(solve_exact(s))
        systems.append(s)
    return xs, systems
