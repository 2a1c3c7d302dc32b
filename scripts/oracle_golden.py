#!/usr/bin/env python
"""Write full-length oracle solve records for the full-size configs into tests/golden/.

Imports only `oracle/` and `synth/` (no CUDA path): every stored value comes from the
oracle.  The GPU tests (`tests/test_gpu_golden.py`) compare the CUDA solves with these
records: iteration counts +-2, the whole |eta| / delta / gamma (MINRES) or residual
(GMRES) history, and the O12-normalised solution on a seeded index sample (1e-8).

  c3  Stokes lid cavity n = 1024, MINRES + P2 (a = 0.005), rtol 1e-8    (BASELINE.json configs[2];
      Algorithm 1, stopping rule P:511-514, P2 P:531-535)
  c4  Oseen n = 512, nu = 0.01, cavity wind, two-stage PCD, eta = 1e-6, c = 10, GMRES(50)
      (BASELINE.json configs[3]; Prop 3.3)

  python scripts/oracle_golden.py c3 [--n 1024]   (~1 h single-threaded)
  python scripts/oracle_golden.py c4 [--n 512]
"""
from __future__ import annotations

import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

import synth  # noqa: E402
from oracle import fem, krylov, mg, normalize, oseen, precond  # noqa: E402

N_SAMPLE = 20000


def _sample(x, n_u, s, seed):
    """O12-normalised solution at seeded indices, plus whole-vector norms (velocity, pressure)."""
    g = s.g
    xn = normalize.normalise_solution(x, n_u, s.MQ, fem.null_vector_k(g))
    idx = synth.sample_indices(g.N, N_SAMPLE, seed)
    return {
        "sample_seed": seed, "sample_count": N_SAMPLE,
        "values": [float(v) for v in xn[idx]],
        "max_abs": float(np.abs(xn).max()),
        "norm_u": float(np.linalg.norm(xn[:n_u])),
        "norm_p": float(np.linalg.norm(xn[n_u:])),
    }


def run_c3(n, a, out):
    t0 = time.perf_counter()
    s = fem.assemble_system(n)
    h = mg.Hierarchy(n)
    Pr = precond.StokesP2(s, a, hierarchy=h)
    t1 = time.perf_counter()
    print(f"c3 n={n}: assembly + hierarchy {t1 - t0:.1f} s", flush=True)
    x, rep = krylov.minres(lambda v: s.K @ v, s.b, Pr, rtol=1e-8, maxit=5000)
    t2 = time.perf_counter()
    r = s.b - s.K @ x
    rec = {
        "config": "c3", "n": n, "a": a, "rtol": 1e-8, "maxit": 5000,
        "source": "scripts/oracle_golden.py (oracle.krylov.minres + oracle.precond.StokesP2)",
        "citation": "Algorithm 1 P:343-368; stopping rule P:511-514; P2 P:531-535; readings R5-R9",
        "iterations": int(rep.iterations), "converged": bool(rep.converged),
        "history": [float(v) for v in rep.history],
        "delta": [float(v) for v in rep.delta],
        "gamma": [float(v) for v in rep.gamma],
        "true_rel_res": float(np.linalg.norm(r) / np.linalg.norm(s.b)),
        "solution": _sample(x, s.g.n_u, s, seed=1024),
        "oracle_seconds": t2 - t1,
    }
    json.dump(rec, open(out, "w"))
    print(f"c3: {rep.iterations} iterations in {t2 - t1:.0f} s -> {out}", flush=True)


def run_c4(n, nu, a, out):
    t0 = time.perf_counter()
    s = fem.assemble_system(n, nu=nu)
    hF = oseen.velocity_hierarchy(n, nu, n_coarse=32)
    schur = oseen.PCDSchur(s, nu)
    t1 = time.perf_counter()
    print(f"c4 n={n}: assembly + hierarchies {t1 - t0:.1f} s", flush=True)
    x, (r1, r2), zstar, bound = oseen.two_stage(s, nu, a=a, eta=1e-6, c=10.0, restart=50, maxit=2000,
                                                hF=hF, schur=schur)
    t2 = time.perf_counter()
    r = s.b - s.K @ x
    rec = {
        "config": "c4", "n": n, "nu": nu, "a": a, "eta": 1e-6, "c": 10.0, "restart": 50,
        "coarse_n": 32, "maxit": 2000,
        "source": "scripts/oracle_golden.py (oracle.oseen.two_stage)",
        "citation": "two-stage P:1058-1092; GMRES P:800-814; Prop 3.3 P:1130-1176; readings R9', R11-R16",
        "step1": {"iterations": int(r1.iterations), "converged": bool(r1.converged),
                  "history": [float(v) for v in r1.history]},
        "step2": {"iterations": int(r2.iterations), "converged": bool(r2.converged),
                  "history": [float(v) for v in r2.history]},
        "zstar": float(zstar), "bound": float(bound),
        "true_rel_res": float(np.linalg.norm(r) / np.linalg.norm(s.b)),
        "solution": _sample(x, s.g.n_u, s, seed=512),
        "oracle_seconds": t2 - t1,
    }
    json.dump(rec, open(out, "w"))
    print(f"c4: {r1.iterations} + {r2.iterations} iterations in {t2 - t1:.0f} s -> {out}", flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("config", choices=["c3", "c4"])
    ap.add_argument("--n", type=int, default=None)
    ap.add_argument("--out", default=None)
    args = ap.parse_args()
    gdir = os.path.join(ROOT, "tests", "golden")
    if args.config == "c3":
        n = args.n or 1024
        run_c3(n, 0.005, args.out or os.path.join(gdir, f"c3_minres_p2_n{n}.json"))
    else:
        n = args.n or 512
        run_c4(n, 0.01, 0.005, args.out or os.path.join(gdir, f"c4_two_stage_n{n}.json"))


if __name__ == "__main__":
    main()
