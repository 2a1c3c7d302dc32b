#!/usr/bin/env python
"""Measure the GPU-vs-oracle agreement floor of the parity cases whose tolerance is looser than
the north_star bar (applies 1e-12, solutions 1e-8), at several inner / outer tolerances.
Prints one JSON line per case (GPU box; diagnostic only, not a test)."""
from __future__ import annotations

import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import synth  # noqa: E402
from oracle import fem, krylov, normalize, oseen, picard, precond, schur2  # noqa: E402
from paper_2303_10233_b200 import etq  # noqa: E402

DEV = torch.device("cuda:0")
NU = 0.01


def dev(a):
    return torch.as_tensor(np.ascontiguousarray(a), dtype=torch.float64, device=DEV)


def host(t):
    torch.cuda.synchronize()
    return t.detach().cpu().numpy()


def rel(a, b):
    return float(np.abs(a - b).max() / max(np.abs(b).max(), 1e-300))


def out(**kw):
    print(json.dumps(kw), flush=True)


def case_p1_apply():
    for n in (4, 16):
        s = fem.assemble_system(n)
        P = etq.Problem(n)
        P.precond_setup(etq.PC_P1_EXACT)
        Pr = precond.StokesP1(s)
        r = synth.random_vector(P.N, seed=6)
        k = fem.null_vector_k(s.g)
        r[P.n_u:] -= (k @ r[P.n_u:]) / (k @ k) * k
        z = torch.zeros(P.N, dtype=torch.float64, device=DEV)
        P.apply_precond(etq.PC_P1_EXACT, dev(r), z)
        zg, zr = host(z), Pr(r)
        out(case="p1_apply", n=n, all=rel(zg, zr), u=rel(zg[:P.n_u], zr[:P.n_u]), p=rel(zg[P.n_u:], zr[P.n_u:]))


def case_gmres_m1(n=32, nc=16):
    s = fem.assemble_system(n, nu=NU)
    g = s.g
    hF = oseen.velocity_hierarchy(n, NU, n_coarse=nc)
    P = etq.Problem(n, bc=0, viscosity=NU, wind=1)
    for kd in (etq.PC_OSEEN_M1, etq.PC_OSEEN_PCD1):
        P.precond_setup(kd, etq.make_params(coarse_n=nc, cheb_sgs_lo=0.005))
    b = torch.zeros(g.N, dtype=torch.float64, device=DEV)
    P.build_rhs(b)
    k = fem.null_vector_k(g)
    # M1 preconditioner apply alone
    r = synth.random_vector(g.N, seed=3)
    z = torch.zeros(g.N, dtype=torch.float64, device=DEV)
    P.apply_precond(etq.PC_OSEEN_M1, dev(r), z)
    out(case="m1_apply", n=n, err=rel(host(z), oseen.OseenM1(s, hF, NU, 0.005)(r)))
    for maxit, rt in ((60, 1e-12), (400, 1e-10), (800, 1e-12)):
        x = torch.zeros(g.N, dtype=torch.float64, device=DEV)
        rep = P.gmres_solve(etq.PC_OSEEN_M1, b, x, rtol=rt, restart=50, maxit=maxit)
        xo, ro = krylov.gmres(lambda v: s.K @ v, s.b, oseen.OseenM1(s, hF, NU, 0.005),
                              tol_abs=rt * np.linalg.norm(s.b), restart=50, maxit=maxit)
        m = min(len(rep["history"]), len(ro.history))
        hd = float(np.max(np.abs(rep["history"][:m] - ro.history[:m]) / ro.history[:m]))
        xg = normalize.normalise_solution(host(x), g.n_u, s.MQ, k)
        xr = normalize.normalise_solution(xo, g.n_u, s.MQ, k)
        out(case="gmres_m1", n=n, maxit=maxit, rtol=rt, its=[rep["iterations"], ro.iterations],
            hist=hd, sol=rel(xg, xr), sol_u=rel(xg[:g.n_u], xr[:g.n_u]), true=[rep["rel_res"], ro.true_residual / np.linalg.norm(s.b)])
    nr = g.n_u + g.n_k
    Kr = fem.reduced_operator(s)
    for rt in (1e-5, 1e-10):
        x = torch.zeros(g.N, dtype=torch.float64, device=DEV)
        rep = P.gmres_solve(etq.PC_OSEEN_PCD1, b, x, rtol=rt, restart=50, maxit=800, reduced=True)
        xo, ro = krylov.gmres(lambda v: Kr @ v, s.b[:nr], oseen.OseenPCD1(s, hF, oseen.PCDSchur(s, NU)),
                              tol_abs=rt * np.linalg.norm(s.b[:nr]), restart=50, maxit=800)
        xg = host(x)
        p1g = xg[g.n_u:nr] - xg[g.n_u:nr].mean(); p1o = xo[g.n_u:] - xo[g.n_u:].mean()
        m = min(len(rep["history"]), len(ro.history))
        hd = float(np.max(np.abs(rep["history"][:m] - ro.history[:m]) / ro.history[:m]))
        out(case="gmres_pcd1", n=n, rtol=rt, its=[rep["iterations"], ro.iterations], hist=hd,
            u=rel(xg[:g.n_u], xo[:g.n_u]), p1=rel(p1g, p1o))
    for eta in (1e-6, 1e-10):
        x = torch.zeros(g.N, dtype=torch.float64, device=DEV)
        o = P.two_stage_solve(b, x, eta=eta, c=10.0, restart=50, maxit=2000)
        xo, (r1, r2), zs, bd = oseen.two_stage(s, NU, a=0.005, eta=eta, c=10.0, restart=50, maxit=2000, hF=hF)
        xg = normalize.normalise_solution(host(x), g.n_u, s.MQ, k)
        xr = normalize.normalise_solution(xo, g.n_u, s.MQ, k)
        out(case="two_stage", n=n, eta=eta, its=[o["step1"]["iterations"], r1.iterations, o["step2"]["iterations"],
                                                 r2.iterations], sol=rel(xg, xr), u=rel(xg[:g.n_u], xr[:g.n_u]),
            zstar=[o["zstar"], zs], bound=[o["bound"], bd])


def case_p1_iter():
    n = 64
    f = synth.f_nodal(n, 0)
    s = fem.assemble_system(n, bc="homogeneous", f_nodal=f)
    g = s.g
    k = fem.null_vector_k(g)
    xo, ro = krylov.minres(lambda v: s.K @ v, s.b, precond.StokesP1(s), rtol=1e-8, maxit=500)
    xr = normalize.normalise_solution(xo, g.n_u, s.MQ, k)
    for irt in (1e-10, 1e-13):
        P = etq.Problem(n, bc=1)
        P.precond_setup(etq.PC_P1_ITER, etq.make_params(inner_rtol=irt))
        b = torch.zeros(P.N, dtype=torch.float64, device=DEV)
        P.build_rhs(b, dev(f))
        x = torch.zeros(P.N, dtype=torch.float64, device=DEV)
        rep = P.minres_solve(etq.PC_P1_ITER, b, x, rtol=1e-8, maxit=500)
        xg = normalize.normalise_solution(host(x), g.n_u, s.MQ, k)
        out(case="p1_iter_c2force", n=n, inner_rtol=irt, its=[rep["iterations"], ro.iterations], sol=rel(xg, xr))
        P.close()


def case_picard():
    n, steps = 16, 3
    g = fem.Grid(n)
    xs, systems = picard.picard(n, NU, steps=steps)
    for eta in (1e-11, 1e-13):
        P = etq.Problem(n, bc=0, viscosity=NU, wind=2)
        prm = etq.make_params(coarse_n=8)
        P.precond_setup(etq.PC_OSEEN_M1, prm)
        P.precond_setup(etq.PC_OSEEN_PCD1, prm)
        x = torch.zeros(P.N, dtype=torch.float64, device=DEV)
        o = P.picard_solve(x, steps=steps, eta=eta, c=10.0, restart=50, maxit=3000)
        xg, xr = host(x), xs[-1].copy()
        for v in (xg, xr):
            v[g.n_u:g.n_u + g.n_k] -= v[g.n_u:g.n_u + g.n_k].mean()
            v[g.n_u + g.n_k:] -= v[g.n_u + g.n_k:].mean()
        s = systems[-1]
        out(case="picard", n=n, eta=eta, status=o["status"], res=[float(v) for v in o["rel_res"]],
            u=rel(xg[:g.n_u], xr[:g.n_u]), p=rel(xg[g.n_u:], xr[g.n_u:]),
            gpu_res=float(np.linalg.norm(s.K @ xg - s.b) / np.linalg.norm(s.b)),
            orc_res=float(np.linalg.norm(s.K @ xr - s.b) / np.linalg.norm(s.b)))
        P.close()


def case_schur2():
    for kind in (etq.PC_OSEEN_M2, etq.PC_OSEEN_LSC):
        for n in (8, 32):
            s = fem.assemble_system(n, nu=NU)
            g = s.g
            x, y = g.node_xy()
            wx, wy = fem.cavity_wind(x, y)
            hF = oseen.velocity_hierarchy(n, NU)
            if kind == etq.PC_OSEEN_M2:
                S = schur2.TwoFieldPCD(s, NU, fem.pcd_f1(g, NU), schur2.f0_jump(g, NU, wx, wy))
            else:
                S = schur2.LSCSchur(s)
            Mo = schur2.OseenBlockTriangular(s, hF, S)
            r = synth.random_vector(g.N, seed=41)
            zr = Mo(r)
            for irt in (1e-13, 1e-15, 1e-16):
                P = etq.Problem(n, bc=0, viscosity=NU, wind=1)
                P.precond_setup(kind, etq.make_params(inner_rtol=irt, inner_maxit=1000))
                z = torch.zeros(g.N, dtype=torch.float64, device=DEV)
                P.apply_precond(kind, dev(r), z)
                zg = host(z)
                out(case="schur2_apply", kind=kind, n=n, inner_rtol=irt, all=rel(zg, zr),
                    p=rel(zg[g.n_u:], zr[g.n_u:]))
                P.close()


def case_exact_mass():
    from oracle import mass
    for n in (16, 128):
        g = fem.Grid(n)
        s = fem.assemble_system(n)
        k = fem.null_vector_k(g)
        ref = mass.SparseAugmentedMassSolver(s.MQ, k)
        r = synth.random_vector(g.n_p, seed=3)
        zr = ref.solve(r)
        for irt in (1e-10, 1e-13, 1e-14, 1e-15):
            P = etq.Problem(n)
            P.precond_setup(etq.PC_P3, etq.make_params(inner_rtol=irt, inner_maxit=400))
            z = torch.zeros(g.n_p, dtype=torch.float64, device=DEV)
            its = P.apply_mass_exact(dev(r), z)
            out(case="exact_mass", n=n, inner_rtol=irt, its=its, err=rel(host(z), zr))
            P.close()


def main():
    which = sys.argv[1:] or ["p1", "m1", "p1iter", "picard", "schur2", "exact"]
    for w in which:
        try:
            {"p1": case_p1_apply, "m1": case_gmres_m1, "p1iter": case_p1_iter, "picard": case_picard,
             "schur2": case_schur2, "exact": case_exact_mass}[w]()
        except Exception as e:   # keep measuring the other cases
            out(case=w, error=repr(e))


if __name__ == "__main__":
    main()
