import sys, json, torch
sys.path.insert(0, "/root/repo")
from paper_2303_10233_b200 import etq
n = 1024
P = etq.Problem(n)
b = torch.zeros(P.N, dtype=torch.float64, device="cuda"); P.build_rhs(b)
for rt in (1e-10, 1e-8, 1e-6, 1e-5, 1e-4, 1e-3):
    P.precond_setup(etq.PC_P3, etq.make_params(inner_rtol=rt))
    x = torch.zeros(P.N, dtype=torch.float64, device="cuda")
    P.minres_solve(etq.PC_P3, b, x, rtol=1e-8, maxit=2000)
    s0 = P.inner_stats(0)
    x.zero_()
    r = P.minres_solve(etq.PC_P3, b, x, rtol=1e-8, maxit=2000)
    s1 = P.inner_stats(0)
    y = torch.zeros_like(x); P.apply_saddle(x, y)
    print(json.dumps({"inner_rtol": rt, "its": r["iterations"], "ms": r["ms_total"], "cg_per_apply": (s1[0]-s0[0])/(s1[1]-s0[1]),
                      "true_rel": float(torch.linalg.norm(b-y)/torch.linalg.norm(b))}), flush=True)
