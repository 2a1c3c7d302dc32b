"""A/B of an etq_set_option switch: V-cycle output bitwise equality and device times of the
V-cycle / P2 apply (and optionally a c3 P2 solve) for each value.

  python scripts/ab_option.py --option 0 --values 0,1 [--n 1024] [--solve]
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

DEFAULTS = {0: 1, 1: 64, 2: 1, 3: 1, 4: 0, 10: 0, 13: 1, 16: 0, 18: 1}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--option", type=int, default=0)
    ap.add_argument("--values", default="0,1")
    ap.add_argument("--n", type=int, default=1024)
    ap.add_argument("--solve", action="store_true")
    args = ap.parse_args()
    out, zs = {}, {}
    for v in [int(x) for x in args.values.split(",")]:
        etq.set_option(args.option, v)
        P = etq.Problem(args.n)
        P.precond_setup(etq.PC_P2_GMG, etq.make_params(cheb_sgs_lo=0.005))
        r = torch.as_tensor(synth.random_vector(P.n_u, seed=3), device="cuda")
        z = torch.zeros(P.n_u, dtype=torch.float64, device="cuda")
        P.apply_vcycle(etq.PC_P2_GMG, r, z)
        torch.cuda.synchronize()
        zs[v] = z.cpu()
        row = {"vcycle_ms": P.time_kernel(2, 30)[0], "p2_apply_ms": P.time_kernel(4, 30)[0]}
        if args.solve:
            b = torch.zeros(P.N, dtype=torch.float64, device="cuda")
            P.build_rhs(b)
            x = torch.zeros(P.N, dtype=torch.float64, device="cuda")
            P.minres_solve(etq.PC_P2_GMG, b, x, rtol=1e-8, maxit=5000)
            x.zero_()
            rep = P.minres_solve(etq.PC_P2_GMG, b, x, rtol=1e-8, maxit=5000)
            row.update({"its": rep["iterations"], "solve_ms": rep["ms_total"],
                        "it_per_s": rep["iterations"] / rep["ms_total"] * 1e3})
        out[v] = row
        P.close()
    etq.set_option(args.option, DEFAULTS[args.option])
    vals = list(zs)
    out["bitwise_equal"] = all(torch.equal(zs[vals[0]], zs[v]) for v in vals[1:])
    out["max_abs_diff"] = max([float((zs[vals[0]] - zs[v]).abs().max()) for v in vals[1:]] + [0.0])
    print(json.dumps(out))


if __name__ == "__main__":
    main()
