"""Small end-to-end exercise of every kernel family for compute-sanitizer (n = 8 / 16)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2303_10233_b200 import etq

dev = torch.device("cuda:0")
z = lambda n: torch.zeros(n, dtype=torch.float64, device=dev)
# Stokes: P1 and P2 MINRES
for kind in (etq.PC_P1_EXACT, etq.PC_P2_GMG):
    P = etq.Problem(8)
    P.precond_setup(kind)
    b = z(P.N); P.build_rhs(b); x = z(P.N)
    r = P.minres_solve(kind, b, x, rtol=1e-8, maxit=200)
    print("stokes", kind, r["iterations"], r["converged"])
P = etq.Problem(16)
P.precond_setup(etq.PC_P2_GMG)
ms, by = P.time_kernel(5, 2); ms, by = P.time_kernel(6, 2)
y = torch.zeros(P.N, dtype=torch.float32, device=dev)
P.apply_saddle_f32(torch.ones(P.N, dtype=torch.float32, device=dev), y)
# Oseen: two-stage
P = etq.Problem(16, bc=0, viscosity=0.01, wind=1)
P.precond_setup(etq.PC_OSEEN_M1, etq.make_params(coarse_n=8))
P.precond_setup(etq.PC_OSEEN_PCD1, etq.make_params(coarse_n=8))
b = z(P.N); P.build_rhs(b); x = z(P.N)
out = P.two_stage_solve(b, x, eta=1e-6, c=10.0, restart=20, maxit=400)
print("oseen", out["step1"]["iterations"], out["step2"]["iterations"], out["zstar"] <= out["bound"])
# interior tiles of every tiled kernel (k_cheb_tile3 n >= 64, k_sgs_tile both geometries,
# k_saddle_tile, k_cheb_step_os, k_prolong_tile) and a few MINRES / GMRES iterations through the graphs
P = etq.Problem(128)
P.precond_setup(etq.PC_P2_GMG, etq.make_params(cheb_sgs_lo=0.005))
b = z(P.N); P.build_rhs(b); x = z(P.N)
r = P.minres_solve(etq.PC_P2_GMG, b, x, rtol=1e-8, maxit=4)
for win in (1, 2, 3):
    etq.set_option(16, win)
    w = z(P.n_p); P.apply_mass_pc(b[P.n_u:].contiguous(), w)
etq.set_option(16, 0)
print("stokes n=128", r["iterations"])
P = etq.Problem(64, bc=0, viscosity=0.01, wind=1)
P.precond_setup(etq.PC_OSEEN_M1, etq.make_params(coarse_n=16))
b = z(P.N); P.build_rhs(b); x = z(P.N)
rep = P.gmres_solve(etq.PC_OSEEN_M1, b, x, rtol=1e-6, restart=10, maxit=12)
print("oseen n=64 M1 GMRES", rep["iterations"])
torch.cuda.synchronize()
print("sanitize smoke ok")
