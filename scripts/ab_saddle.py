import sys, json, torch
sys.path.insert(0, "/root/repo")
import synth
from paper_2303_10233_b200 import etq
out = {}
for n in (16, 64, 1024):
    ys = {}
    for opt in (0, 1):
        etq.set_option(2, opt)
        P = etq.Problem(n)
        P.precond_setup(etq.PC_P2_GMG, etq.make_params(cheb_sgs_lo=0.005))
        x = torch.as_tensor(synth.random_vector(P.N, seed=7), device="cuda")
        for red in (0, 1):
            y = torch.zeros(P.N, dtype=torch.float64, device="cuda")
            P.apply_saddle(x, y, reduced=red) if 'reduced' in P.apply_saddle.__code__.co_varnames else P.apply_saddle(x, y)
            torch.cuda.synchronize()
            ys[(opt, red)] = y.cpu()
        ms, by = P.time_kernel(0, 50)
        out[f"n{n}_opt{opt}_saddle_ms"] = ms
        if n == 1024:
            b = torch.zeros(P.N, dtype=torch.float64, device="cuda"); P.build_rhs(b)
            xx = torch.zeros_like(b); P.minres_solve(etq.PC_P2_GMG, b, xx, rtol=1e-8, maxit=5000); xx.zero_()
            rep = P.minres_solve(etq.PC_P2_GMG, b, xx, rtol=1e-8, maxit=5000)
            out[f"n{n}_opt{opt}_solve"] = [rep["iterations"], rep["ms_total"]]
        P.close()
    out[f"n{n}_bitwise"] = all(torch.equal(ys[(0, r)], ys[(1, r)]) for r in (0, 1))
    out[f"n{n}_maxdiff"] = max(float((ys[(0, r)] - ys[(1, r)]).abs().max()) for r in (0, 1))
etq.set_option(2, 1)
print(json.dumps(out, indent=1))
