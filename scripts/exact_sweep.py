"""NEXT-2 sweep (Table-1-like): MINRES iterations, EST-MINRES gamma^2, solve time and inner CG
counts with P3 = diag(V-cycle, exact M_Q) and P1_ITER = diag(V-cycle-PCG, exact M_Q), against P2,
for the lid-driven cavity (bc 0) at n = 16 ... nmax.

  python scripts/exact_sweep.py [--nmax 1024] [--kinds p2,p3,p1i]
"""
import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

from paper_2303_10233_b200 import etq  # noqa: E402

DEV = torch.device("cuda:0")
KINDS = {"p2": etq.PC_P2_GMG, "p3": etq.PC_P3, "p1i": etq.PC_P1_ITER}


def run(n, name, maxit=5000):
    kind = KINDS[name]
    P = etq.Problem(n, bc=0)
    t0 = time.perf_counter()
    P.precond_setup(kind, etq.make_params(cheb_sgs_lo=0.005) if name == "p2" else None)
    torch.cuda.synchronize()
    setup = time.perf_counter() - t0
    b = torch.zeros(P.N, dtype=torch.float64, device=DEV)
    P.build_rhs(b)
    x = torch.zeros(P.N, dtype=torch.float64, device=DEV)
    P.minres_solve(kind, b, x, rtol=1e-8, maxit=maxit)     # warm-up (graph capture)
    s0 = [P.inner_stats(0), P.inner_stats(1)] if name != "p2" else None
    reps = []
    for _ in range(3):
        x.zero_()
        reps.append(P.minres_solve(kind, b, x, rtol=1e-8, maxit=maxit))
    r = reps[-1]
    ms = sorted(q["ms_total"] for q in reps)[1]
    y = torch.zeros(P.N, dtype=torch.float64, device=DEV)
    P.apply_saddle(x, y)
    out = {"n": n, "pc": name, "iterations": r["iterations"], "converged": r["converged"],
           "true_rel_res": float(torch.linalg.norm(b - y) / torch.linalg.norm(b)),
           "solve_ms_median_of_3": ms, "ms_per_iteration": ms / r["iterations"], "setup_s": setup,
           "est_minres_gamma2": etq.est_minres(r["delta"], r["gamma"])}
    if s0 is not None:
        s1 = [P.inner_stats(0), P.inner_stats(1)]
        for w, nm in ((0, "mass_cg"), (1, "vel_cg")):
            d_it, d_calls = s1[w][0] - s0[w][0], s1[w][1] - s0[w][1]
            if d_calls > 0:
                out[nm + "_its_per_apply"] = d_it / d_calls
    P.close()
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--nmax", type=int, default=1024)
    ap.add_argument("--kinds", default="p2,p3,p1i")
    args = ap.parse_args()
    rows = []
    n = 16
    while n <= args.nmax:
        for name in args.kinds.split(","):
            rows.append(run(n, name))
            print(json.dumps(rows[-1]), flush=True)
        n *= 2
    print(json.dumps({"gpu": torch.cuda.get_device_name(0), "rows": rows}))


if __name__ == "__main__":
    main()
