"""Edge cases and full-size sampled parity (BASELINE.json sizes, bench launch configuration)."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

from oracle import fem, krylov, mg, normalize, oseen, precond  # noqa: E402
from paper_2303_10233_b200 import etq  # noqa: E402
import synth  # noqa: E402

DEV = torch.device("cuda:0")


def dev(a):
    return torch.as_tensor(np.ascontiguousarray(a), dtype=torch.float64, device=DEV)


def host(t):
    torch.cuda.synchronize()
    return t.detach().cpu().numpy()


def zeros(n):
    return torch.zeros(n, dtype=torch.float64, device=DEV)


def test_invalid_arguments():
    with pytest.raises(etq.EtqError) as e:
        etq.Problem(1)
    assert e.value.status == -1
    with pytest.raises(etq.EtqError):
        etq.Problem(8, bc=0, viscosity=-1.0, wind=1)
    P = etq.Problem(6)                                    # not a power of two: no multigrid
    with pytest.raises(etq.EtqError):
        P.precond_setup(etq.PC_P2_GMG)
    P = etq.Problem(8)
    b = zeros(P.N); x = zeros(P.N)
    with pytest.raises(etq.EtqError) as e:                # not set up
        P.minres_solve(etq.PC_P2_GMG, b, x)
    assert e.value.status == -6
    with pytest.raises(etq.EtqError):                     # Oseen kinds on a Stokes problem
        P.precond_setup(etq.PC_OSEEN_M1)


def test_zero_rhs_and_maxit_status():
    P = etq.Problem(8)
    P.precond_setup(etq.PC_P2_GMG, etq.make_params(cheb_sgs_lo=0.005))
    b = zeros(P.N); x = zeros(P.N)
    rep = P.minres_solve(etq.PC_P2_GMG, b, x, rtol=1e-8, maxit=50)
    assert rep["iterations"] == 0 and rep["converged"] and float(x.abs().max()) == 0.0
    P.build_rhs(b)
    rep = P.minres_solve(etq.PC_P2_GMG, b, x, rtol=1e-8, maxit=3)
    assert rep["iterations"] == 3 and not rep["converged"] and rep["status"] == etq.ETQ_NOT_CONVERGED


@pytest.mark.parametrize("kind", [etq.PC_P1_EXACT, etq.PC_P2_GMG])
def test_minres_n2_and_warm_start(kind):
    """Smallest grid (n = 2: one interior Q2 node per element row) and a non-zero initial guess."""
    for n in (2, 8):
        s = fem.assemble_system(n)
        g = s.g
        P = etq.Problem(n)
        if kind == etq.PC_P1_EXACT:
            P.precond_setup(kind); Pr = precond.StokesP1(s)
        else:
            P.precond_setup(kind, etq.make_params(cheb_sgs_lo=0.03)); Pr = precond.StokesP2(s, 0.03)
        b = zeros(P.N); P.build_rhs(b)
        x0 = synth.random_vector(P.N, seed=41)
        x = dev(x0)
        rep = P.minres_solve(kind, b, x, rtol=1e-10, maxit=300)
        xo, ro = krylov.minres(lambda v: s.K @ v, s.b, Pr, rtol=1e-10, maxit=300, x0=x0)
        assert rep["converged"] and ro.converged and abs(rep["iterations"] - ro.iterations) <= 2
        k = fem.null_vector_k(g)
        xg = normalize.normalise_solution(host(x), g.n_u, s.MQ, k)
        xr = normalize.normalise_solution(xo, g.n_u, s.MQ, k)
        assert np.abs(xg - xr).max() <= 1e-8 * np.abs(xr).max()


def test_c3_full_size_sampled_parity():
    """c3 (n = 1024, the bench configuration): the first MINRES iterations match the oracle's
    |eta_j|, delta_j, gamma_j; the complete GPU solve meets rtol and its true residual is small."""
    n = 1024
    a = 0.005
    s = fem.assemble_system(n)
    h = mg.Hierarchy(n)
    Pr = precond.StokesP2(s, a, hierarchy=h)
    _, ro = krylov.minres(lambda v: s.K @ v, s.b, Pr, rtol=0.0, maxit=3)
    P = etq.Problem(n)
    P.precond_setup(etq.PC_P2_GMG, etq.make_params(cheb_sgs_lo=a))
    b = zeros(P.N); P.build_rhs(b)
    x = zeros(P.N)
    rep = P.minres_solve(etq.PC_P2_GMG, b, x, rtol=1e-8, maxit=5000)
    np.testing.assert_allclose(rep["history"][:3], ro.history[1:4], rtol=1e-9)
    np.testing.assert_allclose(rep["delta"][:3], ro.delta[:3], rtol=1e-9)
    np.testing.assert_allclose(rep["gamma"][:3], ro.gamma[1:4], rtol=1e-9)
    assert rep["converged"] and rep["rel_res"] < 1e-8
    y = zeros(P.N); P.apply_saddle(x, y)
    # preconditioned residual 1e-8 ~ Euclidean residual a few orders larger at most
    assert float(torch.linalg.norm(b - y) / torch.linalg.norm(b)) < 1e-5
    # local mass conservation of the GPU solution
    g0 = s.b[s.g.n_u + s.g.n_k:]
    assert np.abs(s.B0 @ host(x)[:s.g.n_u] - g0).max() <= 10 * 1e-8 * np.linalg.norm(s.b)


def test_c4_full_size_sampled_parity():
    """c4 (n = 512 Oseen, two-stage): the first Step-I GMRES residual estimates match the oracle;
    the full GPU two-stage solve meets eta = 1e-6 and Prop 3.3."""
    n, nu = 512, 0.01
    s = fem.assemble_system(n, nu=nu)
    hF = oseen.velocity_hierarchy(n, nu, n_coarse=32)
    nr = s.g.n_u + s.g.n_k
    Kr = fem.reduced_operator(s)
    _, ro = krylov.gmres(lambda v: Kr @ v, s.b[:nr], oseen.OseenPCD1(s, hF, oseen.PCDSchur(s, nu)),
                         tol_abs=0.0, restart=50, maxit=3)
    P = etq.Problem(n, bc=0, viscosity=nu, wind=1)
    P.precond_setup(etq.PC_OSEEN_M1); P.precond_setup(etq.PC_OSEEN_PCD1)
    b = zeros(P.N); P.build_rhs(b)
    x = zeros(P.N)
    rep = P.gmres_solve(etq.PC_OSEEN_PCD1, b, x, rtol=1e-30, restart=50, maxit=3, reduced=True)
    np.testing.assert_allclose(rep["history"][:4], ro.history[:4], rtol=1e-9)
    x.zero_()
    out = P.two_stage_solve(b, x, eta=1e-6, c=10.0, restart=50, maxit=2000)
    assert out["step1"]["converged"] and out["step2"]["converged"]
    assert out["zstar"] <= out["bound"] * (1 + 1e-9)
    y = zeros(P.N); P.apply_saddle(x, y)
    assert float(torch.linalg.norm(b - y) / torch.linalg.norm(b)) <= 1e-6 * (1 + 1e-6)


@pytest.mark.gpu
def test_gmres_restart_above_limit_rejected():
    """GMRES restart lengths above ETQ_MAX_RESTART (63) are rejected, not run past the Krylov
    bookkeeping (include/etq.h)."""
    P = etq.Problem(4, viscosity=0.01, wind=1)
    P.precond_setup(etq.PC_OSEEN_M1, etq.make_params(cheb_sgs_lo=0.01, coarse_n=2))
    b = torch.zeros(P.N, dtype=torch.float64, device="cuda")
    P.build_rhs(b)
    x = torch.zeros_like(b)
    with pytest.raises(etq.EtqError):
        P.gmres_solve(etq.PC_OSEEN_M1, b, x, rtol=1e-6, restart=64, maxit=10)
    rep = P.gmres_solve(etq.PC_OSEEN_M1, b, x, rtol=1e-6, restart=63, maxit=10)
    assert rep["iterations"] >= 1
    P.close()


def test_cached_graphs_follow_history_reallocation():
    """A solve with a larger maxit reallocates the device history buffer; the cached MINRES /
    Arnoldi graphs (which capture that buffer) must be rebuilt, so the reported |eta|, delta,
    gamma and GMRES histories equal those of a fresh problem (solvers.cu / oseen.cu)."""
    n = 8
    P = etq.Problem(n)
    P.precond_setup(etq.PC_P2_GMG, etq.make_params(cheb_sgs_lo=0.01))
    b = zeros(P.N); P.build_rhs(b)
    x = zeros(P.N)
    P.minres_solve(etq.PC_P2_GMG, b, x, rtol=1e-8, maxit=3)
    x.zero_()
    rep = P.minres_solve(etq.PC_P2_GMG, b, x, rtol=1e-10, maxit=400)
    F = etq.Problem(n)
    F.precond_setup(etq.PC_P2_GMG, etq.make_params(cheb_sgs_lo=0.01))
    xf = zeros(F.N)
    ref = F.minres_solve(etq.PC_P2_GMG, b, xf, rtol=1e-10, maxit=400)
    assert rep["iterations"] == ref["iterations"] > 3
    for key in ("history", "delta", "gamma"):
        np.testing.assert_array_equal(rep[key], ref[key])
    np.testing.assert_array_equal(host(x), host(xf))
    # GMRES: a short reduced solve, then the two-stage driver on the same problem
    Q = etq.Problem(16, bc=0, viscosity=0.01, wind=1)
    G = etq.Problem(16, bc=0, viscosity=0.01, wind=1)
    for p in (Q, G):
        p.precond_setup(etq.PC_OSEEN_M1, etq.make_params(coarse_n=4, cheb_sgs_lo=0.005))
        p.precond_setup(etq.PC_OSEEN_PCD1, etq.make_params(coarse_n=4))
    bq = zeros(Q.N); Q.build_rhs(bq)
    xq = zeros(Q.N)
    Q.gmres_solve(etq.PC_OSEEN_PCD1, bq, xq, rtol=1e-6, restart=50, maxit=3, reduced=True)
    xq.zero_()
    o1 = Q.two_stage_solve(bq, xq, eta=1e-6, c=10.0, restart=50, maxit=2000)
    xg = zeros(G.N)
    o2 = G.two_stage_solve(bq, xg, eta=1e-6, c=10.0, restart=50, maxit=2000)
    for st in ("step1", "step2"):
        assert o1[st]["iterations"] == o2[st]["iterations"]
        np.testing.assert_array_equal(o1[st]["history"], o2[st]["history"])


def test_binding_rejects_wrong_lengths():
    """The C ABI takes no lengths; the binding checks every tensor against the problem's sizes."""
    P = etq.Problem(4)
    with pytest.raises(ValueError):
        P.apply_saddle(zeros(P.N - 1), zeros(P.N))
    with pytest.raises(ValueError):
        P.apply_mass(zeros(P.n_p + 1), zeros(P.n_p))
    with pytest.raises(ValueError):
        P.minres_solve_host(etq.PC_P2_GMG, np.zeros(P.N - 1), np.zeros(P.N))
    with pytest.raises(ValueError):
        P.minres_solve_host(etq.PC_P2_GMG, np.zeros(P.N, dtype=np.float32), np.zeros(P.N))


def test_nan_input_reports_enan():
    """A NaN in the right-hand side reaches the scalar recurrences: MINRES (Algorithm 1 line 3) and
    GMRES return ETQ_ENAN (-7) instead of iterating on garbage."""
    P = etq.Problem(8)
    P.precond_setup(etq.PC_P2_GMG, etq.make_params(cheb_sgs_lo=0.01))
    b = zeros(P.N); P.build_rhs(b)
    b[5] = float("nan")
    x = zeros(P.N)
    with pytest.raises(etq.EtqError) as e:
        P.minres_solve(etq.PC_P2_GMG, b, x, rtol=1e-8, maxit=50)
    assert e.value.status == -7
    Q = etq.Problem(8, bc=0, viscosity=0.01, wind=1)
    Q.precond_setup(etq.PC_OSEEN_M1, etq.make_params(coarse_n=2, cheb_sgs_lo=0.01))
    bq = zeros(Q.N); Q.build_rhs(bq)
    bq[Q.n_u + 3] = float("nan")
    xq = zeros(Q.N)
    with pytest.raises(etq.EtqError) as e:
        Q.gmres_solve(etq.PC_OSEEN_M1, bq, xq, rtol=1e-6, restart=20, maxit=40)
    assert e.value.status == -7


@pytest.mark.parametrize("devloop", [1, 0])
def test_minres_iterate_after_every_small_iteration_count(devloop):
    """Algorithm 1 lines 16-17: x^{(j)} after exactly j = 1 ... 7 iterations equals the oracle's
    (the x update of an odd iteration is deferred to the next call or to the tail; the loop may
    stop inside the two-iteration graph body), in the device loop and in the host loop."""
    n, a = 16, 0.005
    s = fem.assemble_system(n)
    Pr = precond.StokesP2(s, a)
    P = etq.Problem(n)
    etq.set_option(3, devloop)
    try:
        P.precond_setup(etq.PC_P2_GMG, etq.make_params(cheb_sgs_lo=a))
        b = zeros(P.N); P.build_rhs(b)
        scale = None
        for j in range(1, 8):
            xo, ro = krylov.minres(lambda v: s.K @ v, s.b, Pr, rtol=0.0, maxit=j)
            x = zeros(P.N)
            rep = P.minres_solve(etq.PC_P2_GMG, b, x, rtol=1e-30, maxit=j)
            assert rep["iterations"] == j == ro.iterations
            xg = host(x)
            scale = np.abs(xo).max()
            assert np.abs(xg - xo).max() <= 1e-10 * scale, (j, np.abs(xg - xo).max() / scale)
    finally:
        etq.set_option(3, 1)
        P.close()


def test_indefinite_preconditioner_is_reported():
    """Algorithm 1 needs <z, v> >= 0 (lines 3 / 10): a V-cycle whose Chebyshev interval ends far
    below lambda_max(D^-1 A) amplifies the rough modes and is indefinite; MINRES stops with
    ETQ_EINDEFINITE (-4) instead of taking the square root of a negative number."""
    P = etq.Problem(32)
    P.precond_setup(etq.PC_P2_GMG, etq.make_params(cheb_sgs_lo=0.005, smooth_lo=0.05, smooth_hi=0.3))
    b = zeros(P.N); P.build_rhs(b)
    x = zeros(P.N)
    with pytest.raises(etq.EtqError) as e:
        P.minres_solve(etq.PC_P2_GMG, b, x, rtol=1e-8, maxit=200)
    assert e.value.status == -4
    assert np.isfinite(host(x)).all()
    P.close()
