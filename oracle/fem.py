"""oracle.fem — Q2-Q1* finite elements on the uniform square grid of [-1,1]^2.

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

Everything here is the plain definition: a generic element loop with 3x3 Gauss
quadrature on each square, local matrices summed into SciPy COO -> CSR.

Numbering:
  Q2 node (i, j), i, j in [0, 2n], at (-1 + i h/2, -1 + j h/2) -> i + (2n+1) j
  Q1 vertex (a, c) -> a + (n+1) c        (the C^0 pressure, "Q_h^TH")
  element (e, f)  -> e + n f             (the P0 pressure "Q_h^0")
  system vector   [u_x; u_y; p_1; p_0]   (frame ordering [Q1; P0])
"""
from __future__ import annotations

import numpy as np
import scipy.sparse as sp

# ---------------------------------------------------------------- quadrature
# 3-point Gauss-Legendre rule on [0, 1] (exact for degree 5 per direction).
GAUSS_X = np.array([0.5 - 0.5 * np.sqrt(3.0 / 5.0), 0.5, 0.5 + 0.5 * np.sqrt(3.0 / 5.0)])
GAUSS_W = np.array([5.0 / 18.0, 8.0 / 18.0, 5.0 / 18.0])


def q2_basis_1d(xi):
    """Quadratic Lagrange basis on local nodes {0, 1/2, 1} and its derivative."""
    xi = np.asarray(xi, dtype=np.float64)
    val = np.stack([2.0 * (xi - 0.5) * (xi - 1.0),
                    4.0 * xi * (1.0 - xi),
                    2.0 * xi * (xi - 0.5)])
    der = np.stack([4.0 * xi - 3.0,
                    4.0 - 8.0 * xi,
                    4.0 * xi - 1.0])
    return val, der


def q1_basis_1d(xi):
    """Linear Lagrange basis on local nodes {0, 1} and its derivative."""
    xi = np.asarray(xi, dtype=np.float64)
    val = np.stack([1.0 - xi, xi])
    der = np.stack([-np.ones_like(xi), np.ones_like(xi)])
    return val, der


class Grid:
    """n x n squares on [-1,1]^2 ("subdivided uniformly", BASELINE.json configs)."""

    def __init__(self, n: int):
        if n < 1:
            raise ValueError("n must be >= 1")
        self.n = n
        self.h = 2.0 / n
        self.m = 2 * n + 1                 # Q2 nodes per direction
        self.nq = self.m * self.m          # scalar Q2 nodes
        self.n_u = 2 * self.nq
        self.n_k = (n + 1) ** 2
        self.n_0 = n * n
        self.n_p = self.n_k + self.n_0
        self.N = self.n_u + self.n_p
        self.x1d = -1.0 + np.arange(self.m) * (self.h / 2.0)

    # element -> local dof maps ------------------------------------------------
    def elements(self):
        e, f = np.meshgrid(np.arange(self.n), np.arange(self.n), indexing="xy")
        return e.ravel(), f.ravel()        # element id = e + n f

    def q2_dofs(self, e, f):
        """(nel, 9) global Q2 nodes of each element, local order alpha + 3 beta."""
        out = np.empty((e.size, 9), dtype=np.int64)
        for beta in range(3):
            for alpha in range(3):
                out[:, alpha + 3 * beta] = (2 * e + alpha) + self.m * (2 * f + beta)
        return out

    def q1_dofs(self, e, f):
        """(nel, 4) global Q1 vertices of each element, local order a + 2 c."""
        out = np.empty((e.size, 4), dtype=np.int64)
        for c in range(2):
            for a in range(2):
                out[:, a + 2 * c] = (e + a) + (self.n + 1) * (f + c)
        return out

    def boundary_nodes(self):
        """Scalar Q2 nodes on the boundary of [-1,1]^2."""
        i, j = np.meshgrid(np.arange(self.m), np.arange(self.m), indexing="xy")
        i, j = i.ravel(), j.ravel()
        mask = (i == 0) | (j == 0) | (i == self.m - 1) | (j == self.m - 1)
        return np.nonzero(mask)[0]

    def node_xy(self):
        i, j = np.meshgrid(np.arange(self.m), np.arange(self.m), indexing="xy")
        return self.x1d[i.ravel()], self.x1d[j.ravel()]


# ------------------------------------------------------- element-level tables
def _tabulate(h):
    """Basis values/derivatives at the 9 tensor Gauss points of one square of side h.

    Returns dict of arrays with shape (nbasis, 9 quadrature points) and the
    quadrature weights W (9,) including the Jacobian h^2.  Quadrature point
    q = qx + 3 qy.
    """
    v2, d2 = q2_basis_1d(GAUSS_X)          # (3 basis, 3 points)
    v1, d1 = q1_basis_1d(GAUSS_X)
    qx = np.tile(np.arange(3), 3)
    qy = np.repeat(np.arange(3), 3)
    W = (GAUSS_W[qx] * GAUSS_W[qy]) * h * h
    phi = np.empty((9, 9)); phix = np.empty((9, 9)); phiy = np.empty((9, 9))
    for beta in range(3):
        for alpha in range(3):
            a = alpha + 3 * beta
            phi[a] = v2[alpha, qx] * v2[beta, qy]
            phix[a] = d2[alpha, qx] / h * v2[beta, qy]
            phiy[a] = v2[alpha, qx] * d2[beta, qy] / h
    psi = np.empty((4, 9)); psix = np.empty((4, 9)); psiy = np.empty((4, 9))
    for c in range(2):
        for a in range(2):
            k = a + 2 * c
            psi[k] = v1[a, qx] * v1[c, qy]
            psix[k] = d1[a, qx] / h * v1[c, qy]
            psiy[k] = v1[a, qx] * d1[c, qy] / h
    xi = GAUSS_X[qx]
    eta = GAUSS_X[qy]
    return dict(W=W, phi=phi, phix=phix, phiy=phiy, psi=psi, psix=psix, psiy=psiy,
                xi=xi, eta=eta)


def _assemble(loc, rows, cols, shape):
    """Sum local matrices into a global CSR matrix.

    loc: (9_or_4, 9_or_4) shared by every element, or (nel, r, c) per element.
    rows: (nel, r) global row indices; cols: (nel, c) global column indices.
    """
    nel, r = rows.shape
    c = cols.shape[1]
    if loc.ndim == 2:
        vals = np.broadcast_to(loc, (nel, r, c))
    else:
        vals = loc
    R = np.broadcast_to(rows[:, :, None], (nel, r, c)).ravel()
    C = np.broadcast_to(cols[:, None, :], (nel, r, c)).ravel()
    A = sp.coo_matrix((np.ascontiguousarray(vals).ravel(), (R, C)), shape=shape).tocsr()
    A.sum_duplicates()
    A.sort_indices()
    return A


# --------------------------------------------------------------- the blocks
def laplacian(g: Grid):
    """Scalar Q2 Laplacian L_ij = int grad phi_j . grad phi_i  (a(u,v))."""
    t = _tabulate(g.h)
    loc = np.einsum("q,iq,jq->ij", t["W"], t["phix"], t["phix"]) + \
        np.einsum("q,iq,jq->ij", t["W"], t["phiy"], t["phiy"])
    e, f = g.elements()
    d = g.q2_dofs(e, f)
    return _assemble(loc, d, d, (g.nq, g.nq))


def velocity_mass(g: Grid):
    """Scalar consistent Q2 mass int phi_i phi_j (Galerkin load; Mdiag source)."""
    t = _tabulate(g.h)
    loc = np.einsum("q,iq,jq->ij", t["W"], t["phi"], t["phi"])
    e, f = g.elements()
    d = g.q2_dofs(e, f)
    return _assemble(loc, d, d, (g.nq, g.nq))


def divergence(g: Grid):
    """B = [B1; B0] with b(u, p) = -int p div u  ("B^T = [B1^T, B0^T]").

    B1: n_k x n_u, (B1)_{p,(x,i)} = -int psi_p d_x phi_i, (B1)_{p,(y,i)} = -int psi_p d_y phi_i.
    B0: n_0 x n_u, (B0)_{T,(x,i)} = -int_T d_x phi_i (indicator basis of Q_h^0).
    Columns are ordered [u_x nodes; u_y nodes].
    """
    t = _tabulate(g.h)
    e, f = g.elements()
    d2 = g.q2_dofs(e, f)
    d1 = g.q1_dofs(e, f)
    bx = -np.einsum("q,pq,iq->pi", t["W"], t["psi"], t["phix"])
    by = -np.einsum("q,pq,iq->pi", t["W"], t["psi"], t["phiy"])
    B1x = _assemble(bx, d1, d2, (g.n_k, g.nq))
    B1y = _assemble(by, d1, d2, (g.n_k, g.nq))
    b0x = -np.einsum("q,iq->i", t["W"], t["phix"])[None, :]
    b0y = -np.einsum("q,iq->i", t["W"], t["phiy"])[None, :]
    el = (e + g.n * f)[:, None]
    B0x = _assemble(b0x, el, d2, (g.n_0, g.nq))
    B0y = _assemble(b0y, el, d2, (g.n_0, g.nq))
    B1 = sp.hstack([B1x, B1y]).tocsr()
    B0 = sp.hstack([B0x, B0y]).tocsr()
    return B1, B0


def pressure_mass(g: Grid):
    """Two-level pressure mass M_Q = [[Qk, R^T], [R, Q0]]  (Prop 2.1).

    Qk_ij = int phi_j phi_i (Q1), R_{T,p} = int_T psi_p, Q0 = |T| on the diagonal.
    Returns (M_Q, Qk, R, Q0) as CSR matrices.
    """
    t = _tabulate(g.h)
    e, f = g.elements()
    d1 = g.q1_dofs(e, f)
    qk = np.einsum("q,iq,jq->ij", t["W"], t["psi"], t["psi"])
    Qk = _assemble(qk, d1, d1, (g.n_k, g.n_k))
    r = np.einsum("q,pq->p", t["W"], t["psi"])[None, :]
    el = (e + g.n * f)[:, None]
    R = _assemble(r, el, d1, (g.n_0, g.n_k))
    q0 = np.array([[t["W"].sum()]])
    Q0 = _assemble(q0, el, el, (g.n_0, g.n_0))
    MQ = sp.bmat([[Qk, R.T], [R, Q0]]).tocsr()
    MQ.sort_indices()
    return MQ, Qk, R, Q0


def null_vector_k(g: Grid):
    """k = [1_{n_k}; -1_{n_0}]  (Eq. pressure_null_vector)."""
    return np.concatenate([np.ones(g.n_k), -np.ones(g.n_0)])


# ------------------------------------------------------------------ Oseen
def cavity_wind(x, y):
    """Frozen wind of config c4: w = (2y(1-x^2), -2x(1-y^2)) (BASELINE.json configs[3])."""
    return 2.0 * y * (1.0 - x * x), -2.0 * x * (1.0 - y * y)


def _element_quad_xy(g: Grid, e, f, t):
    """Physical coordinates of the 9 quadrature points of each element: (nel, 9)."""
    x0 = -1.0 + e * g.h
    y0 = -1.0 + f * g.h
    return x0[:, None] + g.h * t["xi"][None, :], y0[:, None] + g.h * t["eta"][None, :]


def convection(g: Grid, wind=cavity_wind, chunk=1 << 16):
    """Scalar Q2 convection N_ij = int (w . grad phi_j) phi_i  (Eq. generic-conv-diff)."""
    t = _tabulate(g.h)
    e, f = g.elements()
    d = g.q2_dofs(e, f)
    parts = []
    for s in range(0, e.size, chunk):
        es, fs = e[s:s + chunk], f[s:s + chunk]
        X, Y = _element_quad_xy(g, es, fs, t)
        wx, wy = wind(X, Y)
        loc = np.einsum("q,eq,jq,iq->eij", t["W"], wx, t["phix"], t["phi"]) + \
            np.einsum("q,eq,jq,iq->eij", t["W"], wy, t["phiy"], t["phi"])
        parts.append(_assemble(loc, d[s:s + chunk], d[s:s + chunk], (g.nq, g.nq)))
    N = parts[0]
    for p in parts[1:]:
        N = N + p
    N = N.tocsr(); N.sort_indices()
    return N


def pcd_f1(g: Grid, nu: float, wind=cavity_wind):
    """F1_ij = nu int grad psi_j . grad psi_i + int (w . grad psi_j) psi_i on Q1.

    No boundary modification (reading R13)."""
    t = _tabulate(g.h)
    e, f = g.elements()
    d1 = g.q1_dofs(e, f)
    X, Y = _element_quad_xy(g, e, f, t)
    wx, wy = wind(X, Y)
    diff = np.einsum("q,iq,jq->ij", t["W"], t["psix"], t["psix"]) + \
        np.einsum("q,iq,jq->ij", t["W"], t["psiy"], t["psiy"])
    conv = np.einsum("q,eq,jq,iq->eij", t["W"], wx, t["psix"], t["psi"]) + \
        np.einsum("q,eq,jq,iq->eij", t["W"], wy, t["psiy"], t["psi"])
    loc = nu * diff[None, :, :] + conv
    return _assemble(loc, d1, d1, (g.n_k, g.n_k))


# ------------------------------------------------------------ boundary data
def lid_values(g: Grid):
    """Dirichlet data of the regularised lid: u = (1 - x^4, 0) on y = 1, 0 elsewhere.

    Reading R1: the paper's "u_y = 1 - x^4" is the tangential component."""
    x, y = g.node_xy()
    ux = np.zeros(g.nq)
    uy = np.zeros(g.nq)
    top = np.isclose(y, 1.0)
    ux[top] = 1.0 - x[top] ** 4
    return np.concatenate([ux, uy])


class SaddleSystem:
    """Assembled Q2-Q1* system [Av B^T; B 0] with Dirichlet rows (reading R2 / O4).

    Attributes: g, Av (n_u x n_u velocity block, identity rows on the boundary),
    Ls (scalar block with identity boundary rows), B1, B0, B (with boundary
    columns zeroed), K (full system CSR), b (right-hand side), MQ, Qk, R, Q0,
    Mv (scalar Q2 mass), bnodes (scalar boundary nodes), u_bc.
    """


def assemble_system(n: int, bc: str = "lid", nu: float | None = None, wind=None,
                    f_nodal=None, convection_matrix=None) -> SaddleSystem:
    """Assemble the Stokes (nu=None) or Oseen system and its right-hand side.

    Stokes velocity block A = I_2 (x) L; Oseen F = I_2 (x) (nu L + N)
    (P:734-773).  Dirichlet handling follows reading R2 (O4): lift the boundary
    values into f and g, then zero boundary rows/columns of A (identity
    diagonal, f = u_bc there) and zero the boundary columns of B.
    Body force (reading R10 / O5): f = M_v f_nodal, rows on the boundary set to 0.
    convection_matrix: a precomputed scalar N (e.g. a Picard wind, oracle.picard) instead of wind.
    """
    g = Grid(n)
    s = SaddleSystem()
    s.g = g
    L = laplacian(g)
    if nu is not None:
        Nc = convection_matrix if convection_matrix is not None else \
            convection(g, wind if wind is not None else cavity_wind)
        Ls = (nu * L + Nc).tocsr()
    else:
        Ls = L
    Mv = velocity_mass(g)
    B1, B0 = divergence(g)
    B = sp.vstack([B1, B0]).tocsr()
    Av = sp.block_diag([Ls, Ls]).tocsr()
    bscal = g.boundary_nodes()
    bnd = np.concatenate([bscal, bscal + g.nq])
    if bc == "lid":
        u_bc = lid_values(g)
    elif bc == "homogeneous":
        u_bc = np.zeros(g.n_u)
    else:
        raise ValueError(bc)
    f = np.zeros(g.n_u)
    if f_nodal is not None:
        f = sp.block_diag([Mv, Mv]).tocsr() @ np.asarray(f_nodal, dtype=np.float64)
    ub = np.zeros(g.n_u)
    ub[bnd] = u_bc[bnd]
    # lifting (O4): f <- f - A[:, bnd] u_bnd ; g <- -B[:, bnd] u_bnd
    f = f - Av @ ub
    gvec = -(B @ ub)
    # identity rows/columns on the boundary
    keep = np.ones(g.n_u)
    keep[bnd] = 0.0
    Dk = sp.diags(keep)
    Av_d = (Dk @ Av @ Dk + sp.diags(1.0 - keep)).tocsr()
    B_d = (B @ Dk).tocsr()
    f[bnd] = u_bc[bnd]
    Dks = sp.diags(keep[:g.nq])
    s.Ls = (Dks @ Ls @ Dks + sp.diags(1.0 - keep[:g.nq])).tocsr()
    s.Av = Av_d
    s.B = B_d
    s.B1 = B_d[:g.n_k].tocsr()
    s.B0 = B_d[g.n_k:].tocsr()
    s.K = sp.bmat([[Av_d, B_d.T], [B_d, None]]).tocsr()
    s.b = np.concatenate([f, gvec])
    s.MQ, s.Qk, s.R, s.Q0 = pressure_mass(g)
    s.Mv = Mv
    s.bnodes = bscal
    s.u_bc = u_bc
    s.nu = nu
    return s


def reduced_operator(s: SaddleSystem):
    """Reduced Taylor-Hood operator [F B1^T; B1 0] of Step I (Eq. reduced-system)."""
    return sp.bmat([[s.Av, s.B1.T], [s.B1, None]]).tocsr()


def mdiag(s: SaddleSystem):
    """Diagonal of the velocity mass matrix, both components (reading R12)."""
    d = s.Mv.diagonal()
    return np.concatenate([d, d])


def pcd_ap(s: SaddleSystem):
    """Ap = B1 Mdiag^{-1} B1^T after Dirichlet column removal (Eq. discrete-commutator1x)."""
    Dm = sp.diags(1.0 / mdiag(s))
    Ap = (s.B1 @ Dm @ s.B1.T).tocsr()
    Ap.sort_indices()
    return Ap
