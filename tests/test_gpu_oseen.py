"""GPU parity for the Oseen rows (a3 on F, a7 PCD, a8 GMRES, a9 two-stage) against the oracle.

Same tolerances as tests/test_gpu_parity.py: applies 1e-12 relative, assembled entries 1e-13,
solutions 1e-8 relative (after normalising the pressure null space), iterations +-2.
"""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

from oracle import fem, krylov, mass, normalize, oseen  # noqa: E402
from paper_2303_10233_b200 import etq  # noqa: E402
import synth  # noqa: E402

DEV = torch.device("cuda:0")
NU = 0.01
APPLY_TOL = 1e-12
SOL_TOL = 1e-8      # north_star: final solutions within 1e-8 relative (measured floor ~2e-14 at n = 32)


def dev(a):
    return torch.as_tensor(np.ascontiguousarray(a), dtype=torch.float64, device=DEV)


def host(t):
    torch.cuda.synchronize()
    return t.detach().cpu().numpy()


def rel_err(a, b):
    return np.abs(a - b).max() / max(np.abs(b).max(), 1e-300)


def sp_rel_diff(A, B):
    D = (A - B).tocsr()
    return (np.abs(D.data).max() if D.nnz else 0.0) / np.abs(B.data).max()


_cache = {}


def system(n):
    if n not in _cache:
        _cache[n] = fem.assemble_system(n, nu=NU)
    return _cache[n]


def gpu_problem(n, coarse_n, kinds=(etq.PC_OSEEN_M1, etq.PC_OSEEN_PCD1), a=0.005):
    P = etq.Problem(n, bc=0, viscosity=NU, wind=1)
    for k in kinds:
        P.precond_setup(k, etq.make_params(coarse_n=coarse_n, cheb_sgs_lo=a))
    return P


@pytest.mark.parametrize("n,nc", [(8, 2), (16, 4), (64, 32)])
def test_f_vcycle(n, nc):
    h = oseen.velocity_hierarchy(n, NU, n_coarse=nc)
    P = gpu_problem(n, nc, kinds=(etq.PC_OSEEN_M1,))
    r = synth.random_vector(P.n_u, seed=21)
    z = torch.zeros(P.n_u, dtype=torch.float64, device=DEV)
    P.apply_vcycle(etq.PC_OSEEN_M1, dev(r), z)
    assert rel_err(host(z), h.apply_velocity(r)) < APPLY_TOL
    for lvl in range(1, len(h.levels)):
        assert sp_rel_diff(P.export_operator(0, level=lvl), h.levels[lvl]["A"]) < 1e-13


@pytest.mark.parametrize("n", [4, 16])
def test_pcd_operators_entrywise(n):
    s = system(n)
    P = gpu_problem(n, 2, kinds=(etq.PC_OSEEN_PCD1,))
    assert sp_rel_diff(P.export_operator(4), fem.pcd_f1(s.g, NU)) < 1e-13
    H = oseen.ApHierarchy(n)
    for lvl, lev in enumerate(H.levels):
        assert sp_rel_diff(P.export_operator(3, level=lvl), lev["A"]) < 1e-13


@pytest.mark.parametrize("n", [8, 32])
def test_pcd_schur_apply(n):
    s = system(n)
    P = gpu_problem(n, min(32, n), kinds=(etq.PC_OSEEN_PCD1,))
    S = oseen.PCDSchur(s, NU)
    r = synth.random_vector(s.g.n_k, seed=22)
    z = torch.zeros(s.g.n_k, dtype=torch.float64, device=DEV)
    P.apply_pcd_schur(dev(r), z)
    assert rel_err(host(z), S(r)) < APPLY_TOL


@pytest.mark.parametrize("n,nc", [(8, 2), (16, 4)])
def test_block_triangular_applies(n, nc):
    s = system(n)
    g = s.g
    P = gpu_problem(n, nc)
    hF = oseen.velocity_hierarchy(n, NU, n_coarse=nc)
    r = synth.random_vector(g.N, seed=23)
    z = torch.zeros(g.N, dtype=torch.float64, device=DEV)
    P.apply_precond(etq.PC_OSEEN_M1, dev(r), z)
    M1 = oseen.OseenM1(s, hF, NU, 0.005)
    assert rel_err(host(z), M1(r)) < APPLY_TOL
    nr = g.n_u + g.n_k
    rr = r.copy(); rr[nr:] = 0.0
    P.apply_precond(etq.PC_OSEEN_PCD1, dev(rr), z)
    M_I = oseen.OseenPCD1(s, hF, oseen.PCDSchur(s, NU))
    zz = host(z)
    assert rel_err(zz[:nr], M_I(r[:nr])) < APPLY_TOL
    assert np.all(zz[nr:] == 0.0)


@pytest.mark.parametrize("n,nc", [(32, 16)])
def test_gmres_parity(n, nc):
    s = system(n)
    g = s.g
    P = gpu_problem(n, nc)
    hF = oseen.velocity_hierarchy(n, NU, n_coarse=nc)
    b = torch.zeros(g.N, dtype=torch.float64, device=DEV)
    P.build_rhs(b)
    assert rel_err(host(b), s.b) < APPLY_TOL
    # full system, M1, a fixed 60 iterations (one restart at 50): same residual path and iterate
    x = torch.zeros(g.N, dtype=torch.float64, device=DEV)
    rep = P.gmres_solve(etq.PC_OSEEN_M1, b, x, rtol=1e-12, restart=50, maxit=60)
    xo, ro = krylov.gmres(lambda v: s.K @ v, s.b, oseen.OseenM1(s, hF, NU, 0.005),
                          tol_abs=1e-12 * np.linalg.norm(s.b), restart=50, maxit=60)
    assert rep["iterations"] == ro.iterations == 60 and rep["restarts"] == ro.restarts == 2
    np.testing.assert_allclose(rep["history"], ro.history, rtol=1e-9)
    assert rep["abs_res"] == pytest.approx(ro.true_residual, rel=1e-9)
    k = fem.null_vector_k(g)
    assert rel_err(normalize.normalise_solution(host(x), g.n_u, s.MQ, k),
                   normalize.normalise_solution(xo, g.n_u, s.MQ, k)) < SOL_TOL
    # reduced system, PCD, to convergence
    nr = g.n_u + g.n_k
    x = torch.zeros(g.N, dtype=torch.float64, device=DEV)
    rep = P.gmres_solve(etq.PC_OSEEN_PCD1, b, x, rtol=1e-5, restart=50, maxit=400, reduced=True)
    Kr = fem.reduced_operator(s)
    xo, ro = krylov.gmres(lambda v: Kr @ v, s.b[:nr], oseen.OseenPCD1(s, hF, oseen.PCDSchur(s, NU)),
                          tol_abs=1e-5 * np.linalg.norm(s.b[:nr]), restart=50, maxit=400)
    assert rep["converged"] and ro.converged
    assert abs(rep["iterations"] - ro.iterations) <= 2
    xg = host(x)
    # reduced solution is unique up to a constant Q1 pressure: compare velocity and the mean-free p1
    np.testing.assert_allclose(xg[:g.n_u], xo[:g.n_u], rtol=0, atol=SOL_TOL * np.abs(xo[:g.n_u]).max())
    p1g = xg[g.n_u:nr] - xg[g.n_u:nr].mean(); p1o = xo[g.n_u:] - xo[g.n_u:].mean()
    assert rel_err(p1g, p1o) < SOL_TOL
    assert np.all(xg[nr:] == 0.0)


@pytest.mark.parametrize("n,nc", [(32, 16)])
def test_two_stage_parity(n, nc):
    s = system(n)
    g = s.g
    P = gpu_problem(n, nc)
    hF = oseen.velocity_hierarchy(n, NU, n_coarse=nc)
    b = torch.zeros(g.N, dtype=torch.float64, device=DEV)
    P.build_rhs(b)
    x = torch.zeros(g.N, dtype=torch.float64, device=DEV)
    out = P.two_stage_solve(b, x, eta=1e-6, c=10.0, restart=50, maxit=600)
    xo, (r1, r2), zstar, bound = oseen.two_stage(s, NU, a=0.005, eta=1e-6, c=10.0, restart=50, maxit=600,
                                                 hF=hF)
    assert out["step1"]["converged"] and out["step2"]["converged"]
    assert abs(out["step1"]["iterations"] - r1.iterations) <= 2
    assert abs(out["step2"]["iterations"] - r2.iterations) <= 2
    assert out["zstar"] == pytest.approx(zstar, rel=1e-9)
    assert out["bound"] == pytest.approx(bound, rel=1e-9)
    assert out["zstar"] <= out["bound"] * (1 + 1e-9)          # Prop 3.3
    k = fem.null_vector_k(g)
    xg = normalize.normalise_solution(host(x), g.n_u, s.MQ, k)
    xr = normalize.normalise_solution(xo, g.n_u, s.MQ, k)
    assert rel_err(xg, xr) < SOL_TOL
    assert np.linalg.norm(s.b - s.K @ host(x)) <= 1e-6 * np.linalg.norm(s.b) * (1 + 1e-6)
