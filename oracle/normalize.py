"""oracle.normalize — remove null-space components before comparing solutions.

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

The enclosed-flow system is singular: k = [1; -1] and, with Dirichlet
data on the whole boundary, the hydrostatic pressure (reading R17; the 2-D
pressure null space of P:858-859).  Solutions are unique only modulo
alpha k + beta 1 in the pressure (reading R19).  Reading O12: choose alpha, beta
such that k^T p = 0 and 1^T M_Q p = 0 (zero mean pressure, int p_h = 0).
"""
from __future__ import annotations

import numpy as np


def normalise_pressure(p, MQ, k):
    """Return p - alpha k - beta 1 with k^T p' = 0 and 1^T M_Q p' = 0 (2x2 solve)."""
    one = np.ones_like(p)
    mq1 = MQ @ one
    # conditions: k^T(p - a k - b 1) = 0 ; mq1^T (p - a k - b 1) = 0
    Amat = np.array([[k @ k, k @ one], [mq1 @ k, mq1 @ one]])
    rhs = np.array([k @ p, mq1 @ p])
    a, b = np.linalg.solve(Amat, rhs)
    return p - a * k - b * one


def normalise_solution(x, n_u, MQ, k):
    out = np.array(x, dtype=np.float64, copy=True)
    out[n_u:] = normalise_pressure(out[n_u:], MQ, k)
    return out
