"""A/B of the temporally blocked Chebyshev smoothing (etq_set_option 0): V-cycle output bitwise
equality and device time per V-cycle / P2 apply, then a c3 P2 solve with each.

  python scripts/ab_tile.py [--n 1024]
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import synth  # noqa: E402
from paper_2303_10233_b200 import etq  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=1024)
    ap.add_argument("--solve", action="store_true")
    args = ap.parse_args()
    out = {}
    zs = {}
    for opt in (0, 1):
        etq.set_option(0, opt)
        P = etq.Problem(args.n)
        P.precond_setup(etq.PC_P2_GMG, etq.make_params(cheb_sgs_lo=0.005))
        r = torch.as_tensor(synth.random_vector(P.n_u, seed=3), device="cuda")
        z = torch.zeros(P.n_u, dtype=torch.float64, device="cuda")
        P.apply_vcycle(etq.PC_P2_GMG, r, z)
        torch.cuda.synchronize()
        zs[opt] = z.cpu()
        row = {}
        for which, name in ((2, "vcycle"), (4, "p2_apply")):
            ms, by = P.time_kernel(which, 20)
            row[name + "_ms"] = ms
        if args.solve:
            b = torch.zeros(P.N, dtype=torch.float64, device="cuda")
            P.build_rhs(b)
            x = torch.zeros(P.N, dtype=torch.float64, device="cuda")
            P.minres_solve(etq.PC_P2_GMG, b, x, rtol=1e-8, maxit=5000)
            x.zero_()
            rep = P.minres_solve(etq.PC_P2_GMG, b, x, rtol=1e-8, maxit=5000)
            row.update({"its": rep["iterations"], "solve_ms": rep["ms_total"],
                        "it_per_s": rep["iterations"] / rep["ms_total"] * 1e3})
        out["tile" if opt else "untiled"] = row
        P.close()
    d = (zs[0] - zs[1]).abs().max().item()
    out["vcycle_max_abs_diff"] = d
    out["bitwise_equal"] = bool(torch.equal(zs[0], zs[1]))
    etq.set_option(0, 1)
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
