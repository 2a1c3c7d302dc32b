"""GPU parity: the CUDA path (through the C ABI) against the CPU oracle on identical seeded inputs.

Tolerances (BASELINE.json north_star): per-operator applies within 1e-12 relative (max-norm,
relative to the oracle output's max-norm), final solutions within 1e-8 relative after the
null-space normalisation O12, iteration counts within +-2.  Assembled matrices are compared
entry by entry (1e-14 relative): the CUDA side builds them from closed-form 1D tables, the
oracle from a 2D Gauss-quadrature element loop.
"""
import numpy as np
import pytest
import scipy.sparse as sp

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

from oracle import fem, mass, mg, krylov, normalize, precond  # noqa: E402
from paper_2303_10233_b200 import etq  # noqa: E402
import synth  # noqa: E402

DEV = torch.device("cuda:0")
APPLY_TOL = 1e-12


def dev(a):
    return torch.as_tensor(np.ascontiguousarray(a), dtype=torch.float64, device=DEV)


def host(t):
    torch.cuda.synchronize()
    return t.detach().cpu().numpy()


def rel_err(a, b):
    return np.abs(a - b).max() / max(np.abs(b).max(), 1e-300)


_sys_cache = {}


def oracle_system(n, bc="lid", nu=None, f=None):
    key = (n, bc, nu, None if f is None else "f")
    if key not in _sys_cache:
        _sys_cache[key] = fem.assemble_system(n, bc=bc, nu=nu, f_nodal=f)
    return _sys_cache[key]


def sp_rel_diff(A, B):
    D = (A - B).tocsr()
    return (np.abs(D.data).max() if D.nnz else 0.0) / np.abs(B.data).max()


@pytest.mark.parametrize("n", [2, 4, 8, 16, 32])
def test_assembly_entrywise(n):
    s = oracle_system(n)
    P = etq.Problem(n, bc=0)
    L = P.export_operator(0)
    B = P.export_operator(1)
    BT = P.export_operator(2)
    assert sp_rel_diff(L, s.Ls) < 1e-14
    assert sp_rel_diff(B, s.B) < 1e-14
    assert sp_rel_diff(BT, s.B.T.tocsr()) < 1e-14
    # stored pattern = exact nnz formulas (cancelled entries dropped)
    if n >= 8:
        assert L.nnz == 60 * n * n - 128 * n + 81
        assert B.nnz == (24 * n * n - 20 * n + 4) + (12 * n * n - 20 * n + 8)
    # B^T is exactly the transpose of B (symmetric saddle operator)
    assert (B.T - BT).nnz == 0 or np.abs((B.T - BT).data).max() == 0.0


@pytest.mark.parametrize("n", [4, 16])
def test_oseen_assembly_entrywise(n):
    s = oracle_system(n, nu=0.01)
    P = etq.Problem(n, bc=0, viscosity=0.01, wind=1)
    F = P.export_operator(0)
    assert sp_rel_diff(F, s.Ls) < 1e-13


@pytest.mark.parametrize("n,bc,force", [(4, 0, False), (16, 0, False), (16, 1, True), (64, 0, True)])
def test_rhs(n, bc, force):
    f = synth.f_nodal(n, seed=0) if force else None
    s = oracle_system(n, bc="lid" if bc == 0 else "homogeneous", f=f)
    P = etq.Problem(n, bc=bc)
    b = torch.zeros(P.N, dtype=torch.float64, device=DEV)
    P.build_rhs(b, dev(f) if force else None)
    assert rel_err(host(b), s.b) < APPLY_TOL


@pytest.mark.parametrize("n", [2, 4, 16, 64, 256])
def test_apply_saddle(n):
    s = oracle_system(n)
    P = etq.Problem(n)
    x = synth.random_vector(P.N, seed=n)
    y = torch.zeros(P.N, dtype=torch.float64, device=DEV)
    P.apply_saddle(dev(x), y)
    assert rel_err(host(y), s.K @ x) < APPLY_TOL
    # reduced Taylor-Hood operator [A B1^T; B1 0] on [u; p1]
    K1 = fem.reduced_operator(s)
    nr = P.n_u + P.n_k
    yr = torch.zeros(P.N, dtype=torch.float64, device=DEV)
    xr = x.copy(); xr[nr:] = 0.0
    P.apply_saddle(dev(xr), yr, reduced=True)
    yr = host(yr)
    assert rel_err(yr[:nr], K1 @ x[:nr]) < APPLY_TOL
    assert np.all(yr[nr:] == 0.0)


@pytest.mark.parametrize("n", [2, 8, 64, 129, 200])     # 129, 200: interior and ragged SGS tiles
def test_mass_and_sgs(n):
    s = oracle_system(n)
    P = etq.Problem(n)
    col = mass.colours(s.g)
    x = synth.random_vector(P.n_p, seed=1)
    r = synth.random_vector(P.n_p, seed=2)
    y = torch.zeros(P.n_p, dtype=torch.float64, device=DEV)
    P.apply_mass(dev(x), y)
    assert rel_err(host(y), s.MQ @ x) < APPLY_TOL
    z = torch.zeros(P.n_p, dtype=torch.float64, device=DEV)
    P.sgs_sweep(dev(r), dev(x), z)
    assert rel_err(host(z), mass.sgs_sweep(s.MQ, r, x, col)) < APPLY_TOL
    P.sgs_sweep(dev(r), None, z)
    assert rel_err(host(z), mass.sgs_sweep(s.MQ, r, np.zeros(P.n_p), col)) < APPLY_TOL


def _p2(P, a):
    P.precond_setup(etq.PC_P2_GMG, etq.make_params(cheb_sgs_lo=a))


@pytest.mark.parametrize("n", [2, 4, 16, 64])
def test_vcycle(n):
    h = mg.Hierarchy(n)
    P = etq.Problem(n)
    _p2(P, 0.01)
    r = synth.random_vector(P.n_u, seed=3)
    z = torch.zeros(P.n_u, dtype=torch.float64, device=DEV)
    P.apply_vcycle(etq.PC_P2_GMG, dev(r), z)
    assert rel_err(host(z), h.apply_velocity(r)) < APPLY_TOL
    for lvl in range(1, len(h.levels)):
        A = P.export_operator(0, level=lvl)
        assert sp_rel_diff(A, h.levels[lvl]["A"]) < 1e-14


@pytest.mark.parametrize("n", [4, 16, 64])
def test_mass_pc(n):
    s = oracle_system(n)
    P = etq.Problem(n)
    a = 0.01 if n > 4 else 0.03
    _p2(P, a)
    assert P.get_cheb_sgs_lo() == a
    r = synth.random_vector(P.n_p, seed=4)
    z = torch.zeros(P.n_p, dtype=torch.float64, device=DEV)
    P.apply_mass_pc(dev(r), z)
    ref = mass.pi_c_pi(s.MQ, r, a, 20, mass.colours(s.g), fem.null_vector_k(s.g))
    assert rel_err(host(z), ref) < APPLY_TOL
    k = fem.null_vector_k(s.g)
    assert abs(k @ host(z)) < 1e-12 * np.abs(host(z)).sum()


@pytest.mark.parametrize("n", [8, 32])
def test_full_precond_p2(n):
    s = oracle_system(n)
    P = etq.Problem(n)
    _p2(P, 0.01)
    Pr = precond.StokesP2(s, 0.01)
    r = synth.random_vector(P.N, seed=5)
    z = torch.zeros(P.N, dtype=torch.float64, device=DEV)
    P.apply_precond(etq.PC_P2_GMG, dev(r), z)
    assert rel_err(host(z), Pr(r)) < APPLY_TOL


@pytest.mark.parametrize("n", [4, 16])
def test_full_precond_p1(n):
    s = oracle_system(n)
    P = etq.Problem(n)
    P.precond_setup(etq.PC_P1_EXACT)
    Pr = precond.StokesP1(s)
    r = synth.random_vector(P.N, seed=6)
    # consistent pressure residual (k^T r_p = 0) as inside MINRES
    k = fem.null_vector_k(s.g)
    r[P.n_u:] -= (k @ r[P.n_u:]) / (k @ k) * k
    z = torch.zeros(P.N, dtype=torch.float64, device=DEV)
    P.apply_precond(etq.PC_P1_EXACT, dev(r), z)
    assert rel_err(host(z), Pr(r)) < APPLY_TOL


@pytest.mark.parametrize("n", [8, 32])
def test_lanczos_estimate(n):
    s = oracle_system(n)
    P = etq.Problem(n)
    v0 = synth.lanczos_start(P.n_p)
    est = P.estimate_sgs_lo(dev(v0), 30)
    ref = mass.estimate_cheb_lo(s.MQ, v0, 30, mass.colours(s.g))
    assert est == pytest.approx(ref, rel=1e-8)


def _solve_parity(n, kind, a=None, rtol=1e-8, maxit=500, bc="lid", force=False):
    f = synth.f_nodal(n, 0) if force else None
    s = oracle_system(n, bc=bc, f=f)
    g = s.g
    P = etq.Problem(n, bc=0 if bc == "lid" else 1)
    if kind == etq.PC_P1_EXACT:
        P.precond_setup(kind)
        Pr = precond.StokesP1(s)
    else:
        _p2(P, a)
        Pr = precond.StokesP2(s, a)
    b = torch.zeros(P.N, dtype=torch.float64, device=DEV)
    P.build_rhs(b, dev(f) if force else None)
    x = torch.zeros(P.N, dtype=torch.float64, device=DEV)
    rep = P.minres_solve(kind, b, x, rtol=rtol, maxit=maxit)
    xo, ro = krylov.minres(lambda v: s.K @ v, s.b, Pr, rtol=rtol, maxit=maxit)
    k = fem.null_vector_k(g)
    xg = normalize.normalise_solution(host(x), g.n_u, s.MQ, k)
    xr = normalize.normalise_solution(xo, g.n_u, s.MQ, k)
    return rep, ro, xg, xr, s


def test_minres_c1_p1():
    """Config c1: n = 16, lid, P1 (BASELINE.json configs[0])."""
    rep, ro, xg, xr, s = _solve_parity(16, etq.PC_P1_EXACT)
    assert rep["converged"] and ro.converged
    assert abs(rep["iterations"] - ro.iterations) <= 2
    assert rel_err(xg, xr) < 1e-8
    n = min(len(rep["delta"]), len(ro.delta))
    np.testing.assert_allclose(rep["delta"][:n], ro.delta[:n], rtol=1e-8, atol=1e-12)
    # |eta| non-increasing
    assert np.all(np.diff(rep["history"]) <= 1e-14 * rep["history"][0])
    # local mass conservation of the GPU solution
    g = s.g
    g0 = s.b[g.n_u + g.n_k:]
    assert np.abs(s.B0 @ xg[:g.n_u] - g0).max() <= 10 * 1e-8 * np.linalg.norm(s.b)


@pytest.mark.parametrize("n", [8, 32, 64])
def test_minres_p2(n):
    rep, ro, xg, xr, s = _solve_parity(n, etq.PC_P2_GMG, a=0.005)
    assert rep["converged"] and ro.converged
    assert abs(rep["iterations"] - ro.iterations) <= 2
    assert rel_err(xg, xr) < 1e-8


def test_minres_c2_p2():
    """Config c2: n = 256, homogeneous BC, N(0,1) nodal body force from seed 0, P2."""
    rep, ro, xg, xr, s = _solve_parity(256, etq.PC_P2_GMG, a=0.005, bc="homogeneous", force=True, maxit=1000)
    assert rep["converged"] and ro.converged
    assert abs(rep["iterations"] - ro.iterations) <= 2
    assert rel_err(xg, xr) < 1e-8


def test_minres_host_entry_matches_device_entry():
    n = 16
    P = etq.Problem(n)
    _p2(P, 0.005)
    b = torch.zeros(P.N, dtype=torch.float64, device=DEV)
    P.build_rhs(b)
    x = torch.zeros(P.N, dtype=torch.float64, device=DEV)
    rep = P.minres_solve(etq.PC_P2_GMG, b, x, rtol=1e-8, maxit=500)
    bh = host(b).copy()
    xh = np.zeros(P.N)
    rep2 = P.minres_solve_host(etq.PC_P2_GMG, bh, xh, rtol=1e-8, maxit=500)
    assert rep2["iterations"] == rep["iterations"]
    np.testing.assert_array_equal(xh, host(x))


def test_solve_is_deterministic():
    n = 32
    P = etq.Problem(n)
    _p2(P, 0.005)
    b = torch.zeros(P.N, dtype=torch.float64, device=DEV)
    P.build_rhs(b)
    xs = []
    for _ in range(2):
        x = torch.zeros(P.N, dtype=torch.float64, device=DEV)
        P.minres_solve(etq.PC_P2_GMG, b, x, rtol=1e-8, maxit=500)
        xs.append(host(x))
    np.testing.assert_array_equal(xs[0], xs[1])


def test_full_size_properties_c3():
    """At the c3 size (n = 1024, the bench's launch configuration) the oracle is too slow for a
    full comparison: check properties that hold at any size and sampled rows."""
    n = 1024
    P = etq.Problem(n)
    N = P.N
    x = dev(synth.random_vector(N, seed=11))
    y = dev(synth.random_vector(N, seed=12))
    Kx = torch.zeros(N, dtype=torch.float64, device=DEV)
    Ky = torch.zeros(N, dtype=torch.float64, device=DEV)
    P.apply_saddle(x, Kx)
    P.apply_saddle(y, Ky)
    lhs = torch.dot(Kx, y).item(); rhs = torch.dot(x, Ky).item()
    assert abs(lhs - rhs) < 1e-12 * abs(lhs) * 100
    # K [0; k] = 0 (Remark 2.2)
    w = torch.zeros(N, dtype=torch.float64, device=DEV)
    w[P.n_u:P.n_u + P.n_k] = 1.0; w[P.n_u + P.n_k:] = -1.0
    P.apply_saddle(w, Kx)
    assert Kx.abs().max().item() < 1e-15
    # sampled rows: compare with the oracle on a 16x16 patch? -> use translation invariance:
    # interior rows of the scalar operator equal the n = 1024 closed form computed by the oracle
    # on a small grid with the same h is impossible (h differs), so check scaling instead:
    # L is h-independent in 2D, so an interior row of L at n=1024 equals an interior row at n=16.
    L = P.export_operator(0)
    s16 = oracle_system(16)
    m16, m = 33, 2 * n + 1
    for (i, j) in [(10, 12), (11, 12), (10, 13), (11, 13)]:
        r16 = s16.Ls.getrow(i + m16 * j)
        rb = L.getrow(500 + i + m * (500 + j))
        v16 = sorted(r16.data.tolist()); vb = sorted(rb.data.tolist())
        np.testing.assert_allclose(vb, v16, rtol=1e-13, atol=1e-15)


def test_est_minres_c1():
    """EST-MINRES (NEXT-1): the GPU MINRES Lanczos scalars give the same gamma^2 as the oracle's,
    and both approximate the deflated generalised eigenvalue of Eq. (7)."""
    n = 8
    s = oracle_system(n)
    P = etq.Problem(n)
    P.precond_setup(etq.PC_P1_EXACT)
    b = torch.zeros(P.N, dtype=torch.float64, device=DEV)
    P.build_rhs(b)
    x = torch.zeros(P.N, dtype=torch.float64, device=DEV)
    rep = P.minres_solve(etq.PC_P1_EXACT, b, x, rtol=1e-12, maxit=400)
    g2 = etq.est_minres(rep["delta"], rep["gamma"])
    xo, ro = krylov.minres(lambda v: s.K @ v, s.b, precond.StokesP1(s), rtol=1e-12, maxit=400)
    assert g2 == pytest.approx(krylov.est_minres_gamma2(ro.delta, ro.gamma), rel=1e-8)
    from tests.test_oracle_estminres import deflated_infsup
    assert g2 == pytest.approx(deflated_infsup(s), rel=1e-3)


@pytest.mark.parametrize("n", [16, 64])
def test_fp32_sweep_variants(n):
    """c5 fp32-value variants (BASELINE.json configs[4]) against the fp64 oracle at 1e-5."""
    s = oracle_system(n)
    P = etq.Problem(n)
    _p2(P, 0.01)
    x = synth.random_vector(P.N, seed=31)
    y = torch.zeros(P.N, dtype=torch.float32, device=DEV)
    P.apply_saddle_f32(torch.as_tensor(x, dtype=torch.float32, device=DEV), y)
    assert rel_err(host(y).astype(np.float64), s.K @ x) < 1e-5
    h = mg.Hierarchy(n)
    r = synth.random_vector(P.n_u, seed=32)
    z = torch.zeros(P.n_u, dtype=torch.float32, device=DEV)
    P.apply_vcycle_f32(torch.as_tensor(r, dtype=torch.float32, device=DEV), z)
    assert rel_err(host(z).astype(np.float64), h.apply_velocity(r)) < 1e-5


@pytest.mark.parametrize("storage", [0, 1, 2])
def test_storage_modes_bitwise_identical(storage):
    """The compressed storage modes change what is streamed, not what is computed."""
    n = 32
    ref = etq.Problem(n, storage=2)
    P = etq.Problem(n, storage=storage)
    for Q in (ref, P):
        _p2(Q, 0.005)
    x = dev(synth.random_vector(P.N, seed=51))
    y0 = torch.zeros(P.N, dtype=torch.float64, device=DEV); y1 = torch.zeros_like(y0)
    ref.apply_saddle(x, y0); P.apply_saddle(x, y1)
    # velocity rows bitwise; storage 0's tiled kernel sums the pressure rows' u_x and u_y parts
    # separately (rounding-level difference from the interleaved stored-row order)
    assert torch.equal(y0[:P.n_u], y1[:P.n_u])
    assert (y0[P.n_u:] - y1[P.n_u:]).abs().max().item() <= 1e-14 * y0[P.n_u:].abs().max().item()
    z0 = torch.zeros(P.N, dtype=torch.float64, device=DEV); z1 = torch.zeros_like(z0)
    ref.apply_precond(etq.PC_P2_GMG, x, z0); P.apply_precond(etq.PC_P2_GMG, x, z1)
    assert torch.equal(z0, z1)
