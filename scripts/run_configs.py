"""Run the BASELINE.json configurations c1-c5 on the GPU and print one JSON document.

  python scripts/run_configs.py [--only c1,c2,c3,c4,c5] [--c5-max 2048]

c1: n=16 lid, P1 MINRES; c2: n=256 homogeneous BC + N(0,1) nodal force (seed 0), P2 MINRES;
c3: n=1024 lid, P2 MINRES (also bench.py's headline); c4: n=512 Oseen nu=0.01 cavity wind,
two-stage PCD with GMRES(50), eta=1e-6, c=10; c4p (NEXT-3): the Picard loop at n=512, nu=0.01,
5 Oseen solves with the previous iterate as wind; c5: fused saddle SpMV and one V-cycle for
n = 64 ... c5-max (fp64), GB/s of algorithmic bytes against the measured HBM peak.
"""
import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import synth  # noqa: E402
from paper_2303_10233_b200 import etq  # noqa: E402

DEV = torch.device("cuda:0")


def peak():
    try:
        return float(json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"])
    except Exception:
        return 6650.0


def zeros(n):
    return torch.zeros(n, dtype=torch.float64, device=DEV)


def minres_case(n, bc, force, kind, maxit):
    t0 = time.perf_counter()
    P = etq.Problem(n, bc=bc)
    P.precond_setup(kind)
    torch.cuda.synchronize()
    setup = time.perf_counter() - t0
    b = zeros(P.N)
    P.build_rhs(b, torch.as_tensor(synth.f_nodal(n, 0), device=DEV) if force else None)
    x = zeros(P.N)
    P.minres_solve(kind, b, x, rtol=1e-8, maxit=maxit)   # warm-up (graph capture)
    reps = []
    for _ in range(3):
        x.zero_()
        reps.append(P.minres_solve(kind, b, x, rtol=1e-8, maxit=maxit))
    ms = sorted(r["ms_total"] for r in reps)[1]
    r = reps[-1]
    out = {"n": n, "N": P.N, "iterations": r["iterations"], "converged": r["converged"], "rel_res": r["rel_res"],
           "solve_ms_median_of_3": ms, "iters_per_s": r["iterations"] / (ms / 1e3), "setup_s": setup}
    if kind == etq.PC_P2_GMG:
        out["cheb_sgs_lo"] = P.get_cheb_sgs_lo()
    P.close()
    return out


def c4_case(n=512):
    t0 = time.perf_counter()
    P = etq.Problem(n, bc=0, viscosity=0.01, wind=1)
    P.precond_setup(etq.PC_OSEEN_M1)
    P.precond_setup(etq.PC_OSEEN_PCD1)
    torch.cuda.synchronize()
    setup = time.perf_counter() - t0
    b = zeros(P.N)
    P.build_rhs(b)
    x = zeros(P.N)
    t0 = time.perf_counter()
    out = P.two_stage_solve(b, x, eta=1e-6, c=10.0, restart=50, maxit=2000)
    torch.cuda.synchronize()
    wall = time.perf_counter() - t0
    # true final residual through the saddle apply
    y = zeros(P.N)
    P.apply_saddle(x, y)
    rel = (torch.linalg.norm(b - y) / torch.linalg.norm(b)).item()
    res = {"n": n, "N": P.N, "setup_s": setup, "wall_s": wall,
           "step1": {k: out["step1"][k] for k in ("iterations", "converged", "abs_res", "rel_res", "ms_total")},
           "step2": {k: out["step2"][k] for k in ("iterations", "converged", "abs_res", "rel_res", "ms_total")},
           "zstar": out["zstar"], "prop33_bound": out["bound"], "final_rel_res": rel,
           "step1_history_head": out["step1"]["history"][:5].tolist(),
           "step2_history_head": out["step2"]["history"][:5].tolist()}
    P.close()
    return res


def c4p_case(n=512, steps=5):
    """NEXT-3: the Picard loop of the cavity at nu = 0.01: Stokes start +
    `steps` Oseen solves with the previous iterate as wind, two-stage PCD with GMRES(50), eta 1e-6."""
    t0 = time.perf_counter()
    P = etq.Problem(n, bc=0, viscosity=0.01, wind=2)
    P.precond_setup(etq.PC_OSEEN_M1)
    P.precond_setup(etq.PC_OSEEN_PCD1)
    torch.cuda.synchronize()
    setup = time.perf_counter() - t0
    x = zeros(P.N)
    t0 = time.perf_counter()
    out = P.picard_solve(x, steps=steps, eta=1e-6, c=10.0, restart=50, maxit=3000)
    torch.cuda.synchronize()
    wall = time.perf_counter() - t0
    res = {"n": n, "N": P.N, "steps": steps, "setup_s": setup, "wall_s": wall, "device_ms": out["ms_total"],
           "status": out["status"], "step1_its": out["step1_its"].tolist(), "step2_its": out["step2_its"].tolist(),
           "true_rel_res": out["rel_res"].tolist()}
    P.close()
    return res


def c4s_case(n=512, maxit=400):
    """NEXT-4: c4's Oseen system with GMRES(50) and the one-stage Schur approximations M2 (two-field
    PCD) and M3 (LSC), against M1, from x = 0 to ||r|| <= 1e-6 ||b||."""
    out = {"n": n}
    for name, kind in (("M1", etq.PC_OSEEN_M1), ("M2", etq.PC_OSEEN_M2), ("LSC", etq.PC_OSEEN_LSC)):
        P = etq.Problem(n, bc=0, viscosity=0.01, wind=1)
        t0 = time.perf_counter()
        P.precond_setup(kind)
        torch.cuda.synchronize()
        setup = time.perf_counter() - t0
        b = zeros(P.N)
        P.build_rhs(b)
        x = zeros(P.N)
        r = P.gmres_solve(kind, b, x, rtol=1e-6, restart=50, maxit=maxit)
        h = r["history"]
        out[name] = {"iterations": r["iterations"], "converged": r["converged"], "ms_total": r["ms_total"],
                     "setup_s": setup, "rel_res_true": r["abs_res"] / float(torch.linalg.norm(b)),
                     "history_every_25": [float(h[k] / h[0]) for k in range(0, len(h), 25)]}
        P.close()
    return out


def c5_case(nmax, storage=0):
    pk = peak()
    rows = []
    n = 64
    while n <= nmax:
        P = etq.Problem(n, bc=0, storage=storage)
        P.precond_setup(etq.PC_P2_GMG, etq.make_params(cheb_sgs_lo=0.005))
        row = {"n": n, "N": P.N}
        for which, name in ((0, "spmv"), (1, "cheb_step"), (2, "vcycle"), (5, "spmv_f32"), (6, "vcycle_f32")):
            ms, by = P.time_kernel(which, 100)
            gbs = by / (ms * 1e-3) / 1e9
            row[name] = {"ms": ms, "bytes": by, "GB_per_s": gbs, "frac_of_measured_peak": gbs / pk,
                         "l2_resident": by < 100e6}
        rows.append(row)
        P.close()
        n *= 2
    return {"peak_GBps": pk, "dtype": "f64 (spmv, cheb_step, vcycle) and f32 values+vectors (*_f32)", "reps": 100,
            "storage": {0: "compressed (implicit indices + value dictionary)", 2: "explicit SELL"}[storage],
            "rows": rows}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--only", default="c1,c2,c3,c4,c4p,c4s,c5")
    ap.add_argument("--c5-max", type=int, default=2048)
    args = ap.parse_args()
    which = set(args.only.split(","))
    res = {"gpu": torch.cuda.get_device_name(0)}
    if "c1" in which:
        res["c1"] = minres_case(16, 0, False, etq.PC_P1_EXACT, 200)
    if "c2" in which:
        res["c2"] = minres_case(256, 1, True, etq.PC_P2_GMG, 2000)
    if "c3" in which:
        res["c3"] = minres_case(1024, 0, False, etq.PC_P2_GMG, 5000)
    if "c4" in which:
        res["c4"] = c4_case(512)
    if "c4p" in which:
        res["c4p"] = c4p_case(512)
    if "c4s" in which:
        res["c4s"] = c4s_case(512)
    if "c5" in which:
        res["c5"] = c5_case(args.c5_max)
        res["c5_explicit_sell"] = c5_case(args.c5_max, storage=2)
    print(json.dumps(res, indent=1))


if __name__ == "__main__":
    main()
