"""Per-component device times of the P3 preconditioner at n (default 1024), and one short P3
MINRES solve for launch lists (run under ncu with --maxit small).

  python scripts/profile_p3.py [--n 1024] [--reps 20] [--solve-maxit 0]
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

from paper_2303_10233_b200 import etq  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=1024)
    ap.add_argument("--reps", type=int, default=20)
    ap.add_argument("--solve-maxit", type=int, default=0)
    ap.add_argument("--inner-rtol", type=float, default=0.0)
    args = ap.parse_args()
    P = etq.Problem(args.n)
    P.precond_setup(etq.PC_P3, etq.make_params(inner_rtol=args.inner_rtol))
    if args.solve_maxit > 0:
        b = torch.zeros(P.N, dtype=torch.float64, device="cuda")
        P.build_rhs(b)
        x = torch.zeros(P.N, dtype=torch.float64, device="cuda")
        r = P.minres_solve(etq.PC_P3, b, x, rtol=1e-8, maxit=args.solve_maxit)
        print(json.dumps({"iterations": r["iterations"], "ms": r["ms_total"]}))
        return
    out = {"n": args.n}
    for which, name in ((0, "saddle_spmv"), (2, "q2_vcycle"), (7, "exact_mass"), (8, "sk_vcycle"), (9, "p3_apply")):
        if which == 2:
            P.precond_setup(etq.PC_P2_GMG, etq.make_params(cheb_sgs_lo=0.005))
        ms, by = P.time_kernel(which, args.reps)
        out[name] = {"ms": ms, "bytes": by}
    it0 = P.inner_stats(0)
    out["mass_cg_stats"] = it0
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
