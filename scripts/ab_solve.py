"""Interleaved A/B of etq_debug_set_option switches on the c3 solve (and P2 / pressure apply times):
python scripts/ab_solve.py --option 16 --values 1,2 --rounds 3
python scripts/ab_solve.py --sets 16=1:15=0,16=2:15=1 --rounds 3"""
import argparse, json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2303_10233_b200 import etq

ap = argparse.ArgumentParser()
ap.add_argument("--option", type=int, default=-1)
ap.add_argument("--sets", default="")
ap.add_argument("--values", default="0,1")
ap.add_argument("--rounds", type=int, default=3)
ap.add_argument("--n", type=int, default=1024)
args = ap.parse_args()
if args.sets:
    vals = args.sets.split(",")
else:
    vals = [f"{args.option}={v}" for v in args.values.split(",")]
res = {v: [] for v in vals}
for r in range(args.rounds):
    for v in vals:
        for kv in v.split(":"):
            k, val = kv.split("="); etq.set_option(int(k), int(val))
        P = etq.Problem(args.n)
        P.precond_setup(etq.PC_P2_GMG, etq.make_params(cheb_sgs_lo=0.005))
        b = torch.zeros(P.N, dtype=torch.float64, device="cuda"); P.build_rhs(b)
        x = torch.zeros_like(b)
        P.minres_solve(etq.PC_P2_GMG, b, x, rtol=1e-8, maxit=5000)
        ms = []
        for _ in range(3):
            x.zero_()
            rep = P.minres_solve(etq.PC_P2_GMG, b, x, rtol=1e-8, maxit=5000)
            ms.append(rep["ms_total"])
        res[v].append({"solve_ms": sorted(ms)[1], "its": rep["iterations"],
                       "pressure_us": P.time_kernel(3, 30)[0] * 1e3, "p2_us": P.time_kernel(4, 30)[0] * 1e3})
        P.close()
out = {}
for v in vals:
    s = sorted(q["solve_ms"] for q in res[v])
    out[v] = {"solve_ms_median": s[len(s) // 2], "it_per_s": res[v][0]["its"] / s[len(s) // 2] * 1e3,
              "pressure_us": sorted(q["pressure_us"] for q in res[v])[len(s) // 2],
              "p2_us": sorted(q["p2_us"] for q in res[v])[len(s) // 2], "all_ms": s}
print(json.dumps({"option": args.option, "results": out}))
