"""oracle.mass — the singular two-level pressure mass matrix M_Q and its approximations.

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

* exact augmented solve [[M_Q, k], [k^T, 0]] [z; lam] = [r; 0]     (P:409-427, P1 of P:515-516)
* symmetric Gauss-Seidel (SGS) sweeps on M_Q in 5-colour order        (reading R7)
* Chebyshev semi-iteration on SGS, m = 20 steps                       (reading R7)
* symmetric projection Pi C Pi with Pi = I - k k^T / k^T k            (reading R6)
* Lanczos estimate of the lower bound `a` of the SGS-preconditioned
  spectrum on the complement of k                                    (reading R7; heuristic parameter)
"""
from __future__ import annotations

import numpy as np
import scipy.sparse as sp

from . import fem


def colours(g: fem.Grid):
    """Colour of every pressure dof: Q1 vertex (a, c) -> (a mod 2) + 2 (c mod 2); P0 cell -> 4.

    Q1 vertices of one colour share no element, so they are uncoupled in Q_k;
    P0 cells couple only to Q1 vertices (Q0 is diagonal).  (Reading R7.)"""
    a, c = np.meshgrid(np.arange(g.n + 1), np.arange(g.n + 1), indexing="xy")
    col1 = (a.ravel() % 2) + 2 * (c.ravel() % 2)
    return np.concatenate([col1, np.full(g.n_0, 4)])


FORWARD = (0, 1, 2, 3, 4)
BACKWARD = (4, 3, 2, 1, 0)


def gs_colour_step(MQ, diag, r, z, idx):
    """Gauss-Seidel update of the (mutually uncoupled) unknowns idx:
    z_i <- (r_i - sum_{j != i} M_ij z_j) / M_ii."""
    Mi = MQ[idx]
    off = Mi @ z - diag[idx] * z[idx]
    z = z.copy()
    z[idx] = (r[idx] - off) / diag[idx]
    return z


def sgs_sweep(MQ, r, y, col):
    """S(y): one forward then one backward Gauss-Seidel sweep on M_Q z = r from z = y
    (symmetric Gauss-Seidel), colour order (0,1,2,3,P0) then (P0,3,2,1,0)."""
    diag = MQ.diagonal()
    z = y.copy()
    for c in FORWARD + BACKWARD:
        z = gs_colour_step(MQ, diag, r, z, np.nonzero(col == c)[0])
    return z


def sgs_sweep_sequential(MQ, r, y, order):
    """Reference scalar Gauss-Seidel: forward over `order`, then backward (brute-force pin)."""
    A = MQ.toarray()
    z = y.copy()
    for i in list(order) + list(order)[::-1]:
        z[i] = (r[i] - A[i] @ z + A[i, i] * z[i]) / A[i, i]
    return z


def chebyshev_sgs(MQ, r, a: float, m: int = 20, col=None):
    """C r: m steps of Chebyshev semi-iteration based on SGS.

    Golub-Varga semi-iteration for the SGS iteration matrix with spectrum in
    [0, rho], rho = 1 - a (reading R7):
        gamma = 2/(2 - rho), rhohat = rho/(2 - rho)
        omega_1 = 1, omega_2 = 1/(1 - rhohat^2/2), omega_{k+1} = 1/(1 - rhohat^2 omega_k / 4)
        y_0 = 0, y_1 = gamma S(y_0)
        y_{k+1} = omega_{k+1} (gamma (S(y_k) - y_k) + y_k - y_{k-1}) + y_{k-1},  k = 1..m-1
    returns y_m."""
    if col is None:
        raise ValueError("colour array required")
    rho = 1.0 - a
    gam = 2.0 / (2.0 - rho)
    rh = rho / (2.0 - rho)
    y_prev = np.zeros_like(r)
    y = gam * sgs_sweep(MQ, r, y_prev, col)
    omega = 1.0
    for k in range(1, m):
        if k == 1:
            omega = 1.0 / (1.0 - 0.5 * rh * rh)
        else:
            omega = 1.0 / (1.0 - 0.25 * rh * rh * omega)
        s = sgs_sweep(MQ, r, y, col)
        y_new = omega * (gam * (s - y) + y - y_prev) + y_prev
        y_prev, y = y, y_new
    return y


def project_k(v, k):
    """Pi v = v - (k^T v / k^T k) k (reading R6)."""
    return v - (k @ v) / (k @ k) * k


def pi_c_pi(MQ, r, a, m, col, k):
    """Pressure block of P2: z = Pi C Pi r (reading R6; P:406-427 asks for z orthogonal to w)."""
    return project_k(chebyshev_sgs(MQ, project_k(r, k), a, m, col), k)


def augmented_c(MQ, r, a, m, col, k):
    """Flag alternative (reading R6): literal augmented system with M_S := C^{-1}:
    z = C r - (k^T C r / k^T C k) C k."""
    Cr = chebyshev_sgs(MQ, r, a, m, col)
    Ck = chebyshev_sgs(MQ, k, a, m, col)
    return Cr - (k @ Cr) / (k @ Ck) * Ck


class AugmentedMassSolver:
    """Exact solve of [[M_Q, k], [k^T, 0]] [z; lam] = [r; 0] by dense LU (P:414-427, P1 of P:516)."""

    def __init__(self, MQ, k):
        n = MQ.shape[0]
        Aug = np.zeros((n + 1, n + 1))
        Aug[:n, :n] = MQ.toarray()
        Aug[:n, n] = k
        Aug[n, :n] = k
        import scipy.linalg as sla
        self.lu = sla.lu_factor(Aug)
        self.n = n

    def solve(self, r, return_multiplier=False):
        import scipy.linalg as sla
        sol = sla.lu_solve(self.lu, np.concatenate([r, [0.0]]))
        return (sol[:self.n], sol[self.n]) if return_multiplier else sol[:self.n]


def lanczos_sgs(MQ, v0, steps, col):
    """Lanczos for the pencil (M_Q, C_sgs): eigenvalues of C_sgs^{-1} M_Q.

    C_sgs^{-1} r is one SGS sweep from zero (sgs_sweep(MQ, r, 0)).  Start
    p_1 = M_Q v0 (so k^T p_1 = 0 and the Krylov space stays C_sgs-orthogonal to k),
    q_1 = C_sgs^{-1} p_1 / beta_0, beta_0 = sqrt(q^T p).
        w = M_Q q_j - alpha... (three-term recurrence in the C_sgs inner product):
        w = M_Q q_j ; alpha_j = q_j^T w ; w -= alpha_j p_j + beta_{j-1} p_{j-1}
        z = C_sgs^{-1} w ; beta_j = sqrt(z^T w) ; q_{j+1} = z / beta_j ; p_{j+1} = w / beta_j
    Returns (alpha[steps], beta[steps-1])."""
    zero = np.zeros(MQ.shape[0])
    p = MQ @ v0
    q = sgs_sweep(MQ, p, zero, col)
    b0 = np.sqrt(q @ p)
    p = p / b0
    q = q / b0
    p_prev = np.zeros_like(p)
    beta_prev = 0.0
    alphas, betas = [], []
    for j in range(steps):
        w = MQ @ q
        alpha = q @ w
        w = w - alpha * p - beta_prev * p_prev
        alphas.append(alpha)
        if j == steps - 1:
            break
        z = sgs_sweep(MQ, w, zero, col)
        beta = np.sqrt(z @ w)
        betas.append(beta)
        p_prev, p = p, w / beta
        q = z / beta
        beta_prev = beta
    return np.array(alphas), np.array(betas)


def estimate_cheb_lo(MQ, v0, steps, col):
    """Lower bound `a` for the Chebyshev-SGS interval: the smallest Ritz value of the
    Lanczos tridiagonal (reading R7).  Parity unpinned as a *value* (heuristic
    estimate); pinned by the Ritz bracketing property lam_min <= a <= lam_max."""
    al, be = lanczos_sgs(MQ, v0, steps, col)
    T = np.diag(al) + np.diag(be, 1) + np.diag(be, -1)
    return float(np.linalg.eigvalsh(T)[0])


def cheb_lo_rule(lam_est: float, m: int) -> float:
    """Default lower end `a` of the Chebyshev-SGS interval (reading R7):
    a = max(lam_est, 2/m^2).  A degree-m polynomial cannot resolve eigenvalues below
    ~1/m^2, and measured MINRES counts are lower with this floor than with a = lam_min
    (n = 32: 42 vs 74 iterations at m = 20)."""
    return max(float(lam_est), 2.0 / (m * m))


class SparseAugmentedMassSolver:
    """Exact solve of [[M_Q, k], [k^T, 0]] [z; lam] = [r; 0] by sparse LU of the bordered matrix
    (same system as AugmentedMassSolver, usable at larger n)."""

    def __init__(self, MQ, k):
        import scipy.sparse.linalg as spla
        n = MQ.shape[0]
        kk = sp.csr_matrix(k.reshape(-1, 1))
        Aug = sp.bmat([[MQ, kk], [kk.T, None]]).tocsc()
        self.lu = spla.splu(Aug)
        self.n = n

    def solve(self, r):
        return self.lu.solve(np.concatenate([r, [0.0]]))[:self.n]


def schur_mass(g: fem.Grid):
    """S_k = Qk - R^T Q0^{-1} R on the Q1 vertices (symmetric PSD, null space = constants)."""
    MQ, Qk, R, Q0 = fem.pressure_mass(g)
    S = (Qk - R.T @ sp.diags(1.0 / Q0.diagonal()) @ R).tocsr()
    S.sort_indices()
    return S


def augmented_via_schur(g: fem.Grid, r, S_pinv_solve):
    """The augmented M_Q solve written through the Schur complement S_k (the reduction the GPU
    uses; derived in DESIGN.md §3 'NEXT-2'):  with a = 1 + R^T 1 / h^2,
        lam = k^T r / 1^T a,  g = r_k - R^T r_0 / h^2 - lam a,  zhat = S_k^+ g,
        beta = ((1^T r_0 + lam n_0) / h^2 - a^T zhat) / 1^T a,  z_k = zhat + beta 1,
        z_0 = (r_0 - R z_k + lam 1) / h^2.
    S_pinv_solve(g) must return a solution of S_k x = g (any constant shift)."""
    MQ, Qk, R, Q0 = fem.pressure_mass(g)
    h2 = g.h * g.h
    rk, r0 = r[:g.n_k], r[g.n_k:]
    one_k = np.ones(g.n_k)
    a = one_k + (R.T @ np.ones(g.n_0)) / h2
    lam = (rk.sum() - r0.sum()) / a.sum()
    gg = rk - (R.T @ r0) / h2 - lam * a
    zhat = S_pinv_solve(gg)
    beta = ((r0.sum() + lam * g.n_0) / h2 - a @ zhat) / a.sum()
    zk = zhat + beta * one_k
    z0 = (r0 - R @ zk + lam) / h2
    return np.concatenate([zk, z0])
