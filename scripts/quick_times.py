"""Device times of the hot kernels (etq_time_kernel) and one c3 P2 solve; one JSON line.

  python scripts/quick_times.py [--n 1024] [--no-solve]
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

from paper_2303_10233_b200 import etq  # noqa: E402

NAMES = {0: "saddle", 10: "sgs_step", 11: "cheb_pre", 12: "cheb_post", 2: "vcycle", 3: "pressure", 4: "p2_apply"}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=1024)
    ap.add_argument("--no-solve", action="store_true")
    ap.add_argument("--reps", type=int, default=30)
    ap.add_argument("--opt", action="append", default=[], help="etq_set_option k=v before setup (repeatable)")
    args = ap.parse_args()
    for kv in args.opt:
        k, v = kv.split("=")
        etq.set_option(int(k), int(v))
    P = etq.Problem(args.n)
    P.precond_setup(etq.PC_P2_GMG, etq.make_params(cheb_sgs_lo=0.005))
    row = {"n": args.n, "opts": args.opt}
    for w, name in NAMES.items():
        try:
            row[name + "_us"] = round(P.time_kernel(w, args.reps)[0] * 1e3, 2)
        except Exception as e:  # noqa: BLE001
            row[name + "_us"] = str(e)
    if not args.no_solve:
        b = torch.zeros(P.N, dtype=torch.float64, device="cuda")
        P.build_rhs(b)
        x = torch.zeros(P.N, dtype=torch.float64, device="cuda")
        P.minres_solve(etq.PC_P2_GMG, b, x, rtol=1e-8, maxit=5000)
        ms = []
        for _ in range(3):
            x.zero_()
            rep = P.minres_solve(etq.PC_P2_GMG, b, x, rtol=1e-8, maxit=5000)
            ms.append(rep["ms_total"])
        ms = sorted(ms)[1]
        row.update({"its": rep["iterations"], "solve_ms": round(ms, 2),
                    "it_per_s": round(rep["iterations"] / ms * 1e3, 1), "rel_res": rep["rel_res"]})
    print(json.dumps(row), flush=True)
    P.close()


if __name__ == "__main__":
    main()
