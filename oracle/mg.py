"""oracle.mg — geometric multigrid V-cycle on the scalar Q2 velocity block.

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

The paper's P2 uses "one AMG V-cycle, with the default parameters in T-IFISS"
(P:531-533); BASELINE.json replaces AMG by a Q2 geometric multigrid V-cycle with
a Chebyshev-3 smoother.  Reading R9 fixes the parameters:
rediscretised level operators with identity Dirichlet rows, nested-Q2
interpolation, Chebyshev degree 3 on [lam_hi/10, lam_hi] with lam_hi = 1.6 in
D^{-1}A, exact dense coarse solve.
"""
from __future__ import annotations

import numpy as np
import scipy.sparse as sp

from . import fem


def prolongation_1d(n_coarse: int):
    """P1d[k, I] = phi^c_I(x^f_k): coarse Q2 Lagrange functions evaluated at fine Q2 nodes.

    This is the natural injection of the coarse Q2 space into the fine one
    (nested spaces), so coarse Q2 functions are reproduced exactly."""
    nf = 2 * n_coarse
    hc = 2.0 / n_coarse
    xf = -1.0 + np.arange(2 * nf + 1) * (1.0 / nf)   # fine node spacing h_f/2 = 1/nf
    P = np.zeros((2 * nf + 1, 2 * n_coarse + 1))
    for k, x in enumerate(xf):
        e = min(int(np.floor((x + 1.0) / hc + 1e-12)), n_coarse - 1)
        xi = (x - (-1.0 + e * hc)) / hc
        val, _ = fem.q2_basis_1d(np.array([xi]))
        for a in range(3):
            P[k, 2 * e + a] += val[a, 0]
    P[np.abs(P) < 1e-15] = 0.0
    return sp.csr_matrix(P)


def prolongation(n_coarse: int):
    """2D nested-Q2 prolongation with fine boundary rows and coarse boundary columns zeroed.

    P = Z_f (P1d (x) P1d) Z_c; restriction is its transpose (symmetric V-cycle)."""
    P1 = prolongation_1d(n_coarse)
    P = sp.kron(P1, P1).tocsr()
    gf = fem.Grid(2 * n_coarse)
    gc = fem.Grid(n_coarse)
    zf = np.ones(gf.nq); zf[gf.boundary_nodes()] = 0.0
    zc = np.ones(gc.nq); zc[gc.boundary_nodes()] = 0.0
    P = (sp.diags(zf) @ P @ sp.diags(zc)).tocsr()
    P.eliminate_zeros()
    return P


def dirichlet_scalar(A, g: fem.Grid):
    """Identity rows/columns on the boundary of a scalar Q2 operator (reading R2)."""
    keep = np.ones(g.nq); keep[g.boundary_nodes()] = 0.0
    D = sp.diags(keep)
    return (D @ A @ D + sp.diags(1.0 - keep)).tocsr()


def chebyshev_smooth(A, dinv, b, x0, lo, hi, degree):
    """Chebyshev iteration in D^{-1}A on [lo, hi] (Saad, Iterative Methods, Alg. 12.1).

    theta = (hi+lo)/2, delta = (hi-lo)/2, sigma = theta/delta, rho_0 = 1/sigma
    r_0 = b - A x_0, d_0 = D^{-1} r_0 / theta
    for k = 0..degree-1:
        x_{k+1} = x_k + d_k ; r_{k+1} = r_k - A d_k
        rho_{k+1} = 1/(2 sigma - rho_k)
        d_{k+1} = rho_{k+1} rho_k d_k + (2 rho_{k+1}/delta) D^{-1} r_{k+1}
    Returns (x_degree, r_degree) with r_degree = b - A x_degree.
    A zero x0 (None) skips the initial product (r_0 = b)."""
    theta = 0.5 * (hi + lo)
    delta = 0.5 * (hi - lo)
    sigma = theta / delta
    rho = 1.0 / sigma
    if x0 is None:
        x = np.zeros_like(b)
        r = b.copy()
    else:
        x = x0.copy()
        r = b - A @ x
    d = dinv * r / theta
    for _ in range(degree):
        x = x + d
        r = r - A @ d
        rho_new = 1.0 / (2.0 * sigma - rho)
        d = rho_new * rho * d + (2.0 * rho_new / delta) * (dinv * r)
        rho = rho_new
    return x, r


def chebyshev_smooth_ellipse(A, dinv, b, x0, lo, hi, bim, degree):
    """Chebyshev iteration in D^{-1}A for a spectrum enclosed by the ellipse with centre
    theta = (hi+lo)/2, real semi-axis a = (hi-lo)/2 and imaginary semi-axis bim (Manteuffel's
    Chebyshev iteration for nonsymmetric matrices; reading R9' for the convection-diffusion
    block).  Same recurrence as chebyshev_smooth with delta = sqrt(a^2 - bim^2), which is
    imaginary when bim > a; the coefficients rho_{k+1} rho_k and 2 rho_{k+1}/delta stay real.
    bim = 0 reduces to chebyshev_smooth."""
    if bim == 0.0:
        return chebyshev_smooth(A, dinv, b, x0, lo, hi, degree)
    theta = 0.5 * (hi + lo)
    a = 0.5 * (hi - lo)
    delta = np.sqrt(complex(a * a - bim * bim))
    sigma = theta / delta
    rho = 1.0 / sigma
    if x0 is None:
        x = np.zeros_like(b)
        r = b.copy()
    else:
        x = x0.copy()
        r = b - A @ x
    d = dinv * r / theta
    for _ in range(degree):
        x = x + d
        r = r - A @ d
        rho_new = 1.0 / (2.0 * sigma - rho)
        c1 = (rho_new * rho).real
        c2 = (2.0 * rho_new / delta).real
        d = c1 * d + c2 * (dinv * r)
        rho = rho_new
    return x, r


def gershgorin_offdiag(N, A):
    """max_i sum_{j != i} |N_ij| / |A_ii|: the imaginary semi-axis used for D^{-1}F (reading R9')."""
    N = N.tocsr().copy()
    N.setdiag(0.0)
    N.eliminate_zeros()
    rs = np.asarray(abs(N).sum(axis=1)).ravel()
    return float(np.max(rs / np.abs(A.diagonal())))


class Hierarchy:
    """Level operators A_l (rediscretised at n/2^l), prolongations and coarse factor."""

    def __init__(self, n: int, n_coarse: int = 2, lo: float = 0.16, hi: float = 1.6,
                 degree: int = 3, operator=None, skew=None):
        """operator(g) -> scalar CSR matrix before Dirichlet rows (default: Laplacian).
        skew(g) -> the convection part N of the operator: if given, each level smooths on the
        ellipse with imaginary semi-axis gershgorin_offdiag(N_l, A_l) (reading R9')."""
        if operator is None:
            operator = fem.laplacian
        self.levels = []
        m = n
        while True:
            g = fem.Grid(m)
            A = dirichlet_scalar(operator(g), g)
            bim = 0.0
            if skew is not None:
                bim = gershgorin_offdiag(dirichlet_scalar(skew(g), g), A)
            self.levels.append({"n": m, "A": A, "dinv": 1.0 / A.diagonal(), "bim": bim})
            if m <= n_coarse:
                break
            if m % 2:
                raise ValueError("n / n_coarse must be a power of two")
            m //= 2
        for l in range(len(self.levels) - 1):
            self.levels[l]["P"] = prolongation(self.levels[l + 1]["n"])
        self.coarse_dense = self.levels[-1]["A"].toarray()
        import scipy.linalg as sla
        self.coarse_lu = sla.lu_factor(self.coarse_dense)   # LAPACK getrf, as np.linalg.solve
        self.lo, self.hi, self.degree = lo, hi, degree

    def vcycle(self, b, l: int = 0):
        """One V-cycle applied to a scalar right-hand side b on level l (reading R9)."""
        lev = self.levels[l]
        if l == len(self.levels) - 1:
            import scipy.linalg as sla
            return sla.lu_solve(self.coarse_lu, b)              # exact coarse solve (LU)
        A, dinv, P, bim = lev["A"], lev["dinv"], lev["P"], lev["bim"]
        x, r = chebyshev_smooth_ellipse(A, dinv, b, None, self.lo, self.hi, bim, self.degree)
        ec = self.vcycle(P.T @ r, l + 1)
        x = x + P @ ec
        x, _ = chebyshev_smooth_ellipse(A, dinv, b, x, self.lo, self.hi, bim, self.degree)
        return x

    def apply_velocity(self, r_u):
        """V-cycle on each velocity component (the same scalar operator)."""
        nq = self.levels[0]["A"].shape[0]
        return np.concatenate([self.vcycle(r_u[:nq]), self.vcycle(r_u[nq:])])
