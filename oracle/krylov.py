"""oracle.krylov — preconditioned MINRES (Algorithm 1) and right-preconditioned GMRES(m).

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).
"""
from __future__ import annotations

import numpy as np


class Report(dict):
    """iterations, converged, history (|eta| or ||r||), delta, gamma, ..."""

    def __getattr__(self, k):
        return self[k]


def minres(Kop, b, Pinv, rtol=1e-8, maxit=1000, x0=None):
    """Preconditioned MINRES, Algorithm 1 line by line.

    Readings R5: delta_j uses the system matrix (the printed "A" at P:353 is the
    calligraphic A); the gamma_j/gamma_{j-1} v^{(j-1)} term is 0 at j = 1 (gamma_0 = 0,
    v^{(0)} = 0); the test is |eta| / gamma_1 < rtol (||r_k||_{P^-1} = |eta|).
    Kop(x) and Pinv(v) are callables.  Raises ValueError if <z, v> < 0 (indefinite P).
    """
    nN = b.shape[0]
    x = np.zeros(nN) if x0 is None else np.array(x0, dtype=np.float64)
    v_prev = np.zeros(nN)                      # v^{(0)}
    w_prev = np.zeros(nN)                      # w^{(0)}
    w = np.zeros(nN)                           # w^{(1)}
    gamma_prev = 0.0                           # gamma_0
    v = b - Kop(x) if x0 is not None else b.copy()   # v^{(1)}
    z = Pinv(v)                                # z^{(1)}
    zv = z @ v
    if zv < 0:
        raise ValueError("indefinite preconditioner")
    gamma = np.sqrt(zv)                        # gamma_1
    eta = gamma
    gamma1 = gamma
    s_prev, s = 0.0, 0.0                       # s_0, s_1
    c_prev, c = 1.0, 1.0                       # c_0, c_1
    hist, deltas, gammas = [abs(eta)], [], [gamma]
    it = 0
    converged = gamma1 == 0.0
    while not converged and it < maxit:
        it += 1
        z = z / gamma                          # line 6
        Az = Kop(z)
        delta = Az @ z                         # line 7
        v_new = Az - (delta / gamma) * v       # line 8
        if gamma_prev != 0.0:
            v_new = v_new - (gamma / gamma_prev) * v_prev
        z_new = Pinv(v_new)                    # line 9
        zv = z_new @ v_new
        if zv < 0:
            raise ValueError("indefinite preconditioner")
        gamma_new = np.sqrt(zv)                # line 10
        a0 = c * delta - c_prev * s * gamma    # line 11
        a1 = np.sqrt(a0 * a0 + gamma_new * gamma_new)   # line 12
        a2 = s * delta + c_prev * c * gamma    # line 13
        a3 = s_prev * gamma                    # line 14
        c_new = a0 / a1                        # line 15
        s_new = gamma_new / a1
        w_new = (z - a3 * w_prev - a2 * w) / a1     # line 16
        x = x + c_new * eta * w_new            # line 17
        eta = -s_new * eta                     # line 18
        deltas.append(delta); gammas.append(gamma_new); hist.append(abs(eta))
        # shift
        v_prev, v = v, v_new
        z = z_new
        w_prev, w = w, w_new
        gamma_prev, gamma = gamma, gamma_new
        c_prev, c = c, c_new
        s_prev, s = s, s_new
        converged = abs(eta) / gamma1 < rtol   # line 19
    return x, Report(iterations=it, converged=bool(converged), history=np.array(hist),
                     delta=np.array(deltas), gamma=np.array(gammas), gamma1=gamma1)


def gmres(Kop, b, Minv, tol_abs, restart=50, maxit=1000, x0=None):
    """Right-preconditioned restarted GMRES(m) with classical Gram-Schmidt applied twice (CGS2).

    GMRES with a block preconditioner, residual in the Euclidean norm
    (Eq. residual-norm); reading R18 fixes restart m = 50 and CGS2.
      r_0 = b - K x_0, beta = ||r_0||, v_1 = r_0 / beta
      for j = 1..m: z = M^{-1} v_j, w = K z;
                    h = V^T w, w -= V h, h' = V^T w, w -= V h', h += h';  h_{j+1,j} = ||w||
                    previous Givens rotations, new rotation, |g_{j+1}| = residual estimate
      x <- x_0 + M^{-1}(V_m y); true residual recomputed at each restart.
    Stops when the residual estimate <= tol_abs.  A zero h_{j+1,j} is a happy breakdown.
    """
    nN = b.shape[0]
    x = np.zeros(nN) if x0 is None else np.array(x0, dtype=np.float64)
    hist = []
    total = 0
    restarts = 0
    converged = False
    while True:
        r = b - Kop(x)
        beta = np.linalg.norm(r)
        if not hist:
            hist.append(beta)
        if beta <= tol_abs:
            converged = True
            break
        if total >= maxit:
            break
        m = min(restart, maxit - total)
        V = np.zeros((m + 1, nN))
        H = np.zeros((m + 1, m))
        cs = np.zeros(m); sn = np.zeros(m)
        gvec = np.zeros(m + 1); gvec[0] = beta
        V[0] = r / beta
        k = 0
        res = beta
        for j in range(m):
            z = Minv(V[j])
            w = Kop(z)
            h = V[:j + 1] @ w
            w = w - V[:j + 1].T @ h
            h2 = V[:j + 1] @ w
            w = w - V[:j + 1].T @ h2
            h = h + h2
            hn = np.linalg.norm(w)
            H[:j + 1, j] = h
            H[j + 1, j] = hn
            for i in range(j):
                t = cs[i] * H[i, j] + sn[i] * H[i + 1, j]
                H[i + 1, j] = -sn[i] * H[i, j] + cs[i] * H[i + 1, j]
                H[i, j] = t
            den = np.hypot(H[j, j], H[j + 1, j])
            cs[j] = H[j, j] / den
            sn[j] = H[j + 1, j] / den
            H[j, j] = den
            H[j + 1, j] = 0.0
            gvec[j + 1] = -sn[j] * gvec[j]
            gvec[j] = cs[j] * gvec[j]
            res = abs(gvec[j + 1])
            hist.append(res)
            k = j + 1
            if res <= tol_abs or hn == 0.0:
                break
            V[j + 1] = w / hn
        y = np.zeros(k)
        for i in range(k - 1, -1, -1):
            y[i] = (gvec[i] - H[i, i + 1:k] @ y[i + 1:k]) / H[i, i]
        x = x + Minv(V[:k].T @ y)
        total += k
        restarts += 1
        if res <= tol_abs:
            converged = True                   # stop on the residual estimate (O10)
            break
    true_res = np.linalg.norm(b - Kop(x))
    return x, Report(iterations=total, converged=bool(converged), history=np.array(hist),
                     restarts=restarts, true_residual=true_res)


def est_minres_gamma2(delta, gamma):
    """EST-MINRES inf-sup estimate (reading of S:439/S:461).

    The MINRES recurrences of Algorithm 1 are the Lanczos process for P^{-1} K with the
    tridiagonal T_k = tridiag(gamma_{j+1}; delta_j; gamma_{j+1}) (delta_1..delta_k on the diagonal,
    gamma_2..gamma_k off the diagonal).  With the exact velocity block, eigenvalues lam of P^{-1} K
    satisfy lam (lam - 1) = sigma, sigma an eigenvalue of M_S^{-1} B A^{-1} B^T (Eq. (7)), so the
    negative Ritz value mu closest to 0 gives gamma^2 ~ mu (mu - 1).  Returns nan if T_k has no
    negative Ritz value yet.  gamma: [gamma_1, gamma_2, ...] as recorded by minres()."""
    k = len(delta)
    if k == 0:
        return float("nan")
    off = np.asarray(gamma[1:k], dtype=np.float64)
    T = np.diag(np.asarray(delta[:k], dtype=np.float64)) + np.diag(off, 1) + np.diag(off, -1)
    mu = np.linalg.eigvalsh(T)
    neg = mu[mu < 0]
    if neg.size == 0:
        return float("nan")
    m = neg.max()
    return float(m * (m - 1.0))
