"""c4 two-stage timing for an etq_debug_set_option switch: python scripts/c4_ab.py --opt 14=0"""
import argparse, json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2303_10233_b200 import etq

ap = argparse.ArgumentParser()
ap.add_argument("--opt", action="append", default=[])
ap.add_argument("--n", type=int, default=512)
args = ap.parse_args()
for kv in args.opt:
    k, v = kv.split("="); etq.set_option(int(k), int(v))
P = etq.Problem(args.n, bc=0, viscosity=0.01, wind=1)
P.precond_setup(etq.PC_OSEEN_M1)
P.precond_setup(etq.PC_OSEEN_PCD1)
b = torch.zeros(P.N, dtype=torch.float64, device="cuda"); P.build_rhs(b)
x = torch.zeros_like(b)
P.two_stage_solve(b, x, eta=1e-6, c=10.0, restart=50, maxit=2000)
ms = []
for _ in range(3):
    x.zero_()
    out = P.two_stage_solve(b, x, eta=1e-6, c=10.0, restart=50, maxit=2000)
    ms.append(out["step1"]["ms_total"] + out["step2"]["ms_total"])
y = torch.zeros_like(b); P.apply_saddle(x, y)
print(json.dumps({"opts": args.opt, "its": [out["step1"]["iterations"], out["step2"]["iterations"]],
                  "ms_median": sorted(ms)[1], "rel_res": (torch.linalg.norm(b - y) / torch.linalg.norm(b)).item(),
                  "zstar": out["zstar"], "bound": out["bound"]}))
