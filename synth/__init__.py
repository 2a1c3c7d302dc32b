"""Seeded synthetic inputs shared by the oracle tests, the GPU tests and bench.py.

This module holds NONE of the method's arithmetic: it only draws seeded
random numbers and fixes the workload shapes (BASELINE.json configs c1-c5,
SURVEY.md §8(d) "Synthetic inputs").  Both the oracle (`oracle/`) and the
CUDA path receive the arrays produced here as plain inputs.
"""
from __future__ import annotations

import numpy as np


def sizes(n: int) -> dict:
    """Dof counts of the Q2-Q1* space on an n x n grid (SURVEY §8 sizes)."""
    nq = (2 * n + 1) ** 2
    n_u = 2 * nq
    n_k = (n + 1) ** 2
    n_0 = n * n
    return {"n": n, "nq": nq, "n_u": n_u, "n_k": n_k, "n_0": n_0,
            "n_p": n_k + n_0, "N": n_u + n_k + n_0}


def f_nodal(n: int, seed: int = 0) -> np.ndarray:
    """c2 body force: i.i.d. N(0,1) Q2 nodal values, component-major [fx; fy]
    (BASELINE.json configs[1]: "body force with i.i.d. N(0,1) nodal values from seed 0")."""
    return np.random.default_rng(seed).standard_normal(2 * (2 * n + 1) ** 2)


def random_vector(length: int, seed: int) -> np.ndarray:
    """Seeded N(0,1) vector (c5 sweep inputs and operator-parity inputs)."""
    return np.random.default_rng(seed).standard_normal(length)


def lanczos_start(n_p: int, seed: int = 12345) -> np.ndarray:
    """Start vector of the Lanczos estimate of the Chebyshev-SGS lower bound `a`."""
    return np.random.default_rng(seed).standard_normal(n_p)


def sample_indices(length: int, count: int, seed: int) -> np.ndarray:
    """Sorted seeded sample of distinct indices in [0, length) (solution-sample positions of
    the full-size golden records, tests/golden/c*_*.json)."""
    count = min(count, length)
    return np.sort(np.random.default_rng(seed).choice(length, size=count, replace=False))


# BASELINE.json configs (SURVEY §8 head)
CONFIGS = {
    "c1": {"n": 16, "bc": "lid", "force": None, "pc": "P1"},
    "c2": {"n": 256, "bc": "homogeneous", "force": "random0", "pc": "P2"},
    "c3": {"n": 1024, "bc": "lid", "force": None, "pc": "P2"},
    "c4": {"n": 512, "bc": "lid", "nu": 0.01, "wind": "cavity", "pc": "two-stage"},
}
