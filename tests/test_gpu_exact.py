"""GPU parity of SURVEY §8(f) NEXT-2: the exact augmented M_Q solve at scale through the Schur
complement S_k (reading R21) and the preconditioners built on it (P3, P1_ITER).

The oracle side is the definition: the bordered system [[M_Q, k], [k^T, 0]] solved by sparse LU
(oracle.mass.SparseAugmentedMassSolver) and P1 = diag(A^{-1}, exact M_Q) with a sparse
direct A^{-1}.  The CUDA side solves S_k zhat = g by Q1-GMG-preconditioned CG inside a
CUDA-graph while loop; with the inner tolerance at 1e-13 the two agree to ~1e-10 relative, and
with the default 1e-10 the outer MINRES iteration counts agree within the north-star +-2.
"""
import numpy as np
import pytest
import scipy.sparse as sp

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

from oracle import fem, mass, krylov, normalize, precond  # noqa: E402
from paper_2303_10233_b200 import etq  # noqa: E402
import synth  # noqa: E402

DEV = torch.device("cuda:0")


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


def _setup(P, kind=etq.PC_P3, **kw):
    P.precond_setup(kind, etq.make_params(**kw))


@pytest.mark.parametrize("n", [2, 8, 32])
def test_sk_levels_entrywise(n):
    """Every level of the S_k hierarchy equals the oracle's Schur complement on that grid, scaled
    by 4^-l (reading R21), entry by entry."""
    P = etq.Problem(n)
    _setup(P)
    l, m = 0, n
    while True:
        S = P.export_operator(5, l)
        ref = mass.schur_mass(fem.Grid(m)) * 4.0 ** (-l)
        assert S.shape == ref.shape
        assert sp_rel_diff(S, ref) < 1e-13
        if m <= min(n, 16):
            break
        l, m = l + 1, m // 2
    P.close()


@pytest.mark.parametrize("n", [2, 4, 16, 64, 128])
def test_exact_mass_solve_matches_bordered_lu(n):
    """z = exact augmented M_Q solve against the oracle's sparse LU of the bordered
    matrix, at a tight inner tolerance; k^T z = 0 and M_Q z + lambda k = r hold."""
    g = fem.Grid(n)
    s = fem.assemble_system(n)
    k = fem.null_vector_k(g)
    ref = mass.SparseAugmentedMassSolver(s.MQ, k)
    P = etq.Problem(n)
    _setup(P, inner_rtol=1e-13)
    for seed in (3, 4):
        r = synth.random_vector(g.n_p, seed=seed)
        z = torch.zeros(g.n_p, dtype=torch.float64, device=DEV)
        its = P.apply_mass_exact(dev(r), z)
        zg = host(z)
        zr = ref.solve(r)
        # floor: the oracle's own sparse LU of the bordered matrix is accurate to ~cond * eps
        # (measured GPU-oracle difference 1.6e-12 at n = 128 for every inner tolerance <= 1e-10)
        assert rel_err(zg, zr) < 1e-11, (n, seed)
        assert 1 <= its <= 40
        assert abs(k @ zg) <= 1e-10 * np.abs(zg).sum()
        lam = (k @ r) / (g.n_k + g.n_0)   # lambda = k^T r / 1^T a (reading R21)
        res = s.MQ @ zg + lam * k - r
        assert np.abs(res).max() <= 1e-9 * np.abs(r).max()
    P.close()


def test_exact_mass_inner_iterations_mesh_independent():
    """Q1-GMG-preconditioned CG on S_k converges in a mesh-independent number of iterations."""
    its = []
    for n in (32, 128, 512):
        P = etq.Problem(n)
        _setup(P)
        g = fem.Grid(n)
        r = dev(synth.random_vector(g.n_p, seed=5))
        z = torch.zeros(g.n_p, dtype=torch.float64, device=DEV)
        its.append(P.apply_mass_exact(r, z))
        P.close()
    assert max(its) <= 15 and max(its) - min(its) <= 3, its


def test_exact_mass_zero_rhs_and_graph_modes():
    """r = 0 gives z = 0 with no CG iteration; graph-captured (inside MINRES) and eager applies
    agree bitwise."""
    n = 16
    P = etq.Problem(n)
    _setup(P)
    g = fem.Grid(n)
    z = torch.ones(g.n_p, dtype=torch.float64, device=DEV)
    its = P.apply_mass_exact(torch.zeros(g.n_p, dtype=torch.float64, device=DEV), z)
    assert its == 0 and float(z.abs().max()) == 0.0
    b = torch.zeros(P.N, dtype=torch.float64, device=DEV)
    P.build_rhs(b)
    xs = []
    for graphs in (1, 0):
        _setup(P, use_graphs=graphs)
        x = torch.zeros(P.N, dtype=torch.float64, device=DEV)
        P.minres_solve(etq.PC_P3, b, x, rtol=1e-8, maxit=300)
        xs.append(host(x))
    np.testing.assert_array_equal(xs[0], xs[1])
    P.close()


def _minres_parity(n, kind, Pr_factory, bc="lid", force=False, rtol=1e-8, maxit=500, **kw):
    f = synth.f_nodal(n, 0) if force else None
    s = fem.assemble_system(n, bc=bc, f_nodal=f)
    g = s.g
    P = etq.Problem(n, bc=0 if bc == "lid" else 1)
    _setup(P, kind, **kw)
    b = torch.zeros(P.N, dtype=torch.float64, device=DEV)
    P.build_rhs(b, dev(f) if force else None)
    x = torch.zeros(P.N, dtype=torch.float64, device=DEV)
    rep = P.minres_solve(kind, b, x, rtol=rtol, maxit=maxit)
    xo, ro = krylov.minres(lambda v: s.K @ v, s.b, Pr_factory(s), rtol=rtol, maxit=maxit)
    k = fem.null_vector_k(g)
    xg = normalize.normalise_solution(host(x), g.n_u, s.MQ, k)
    xr = normalize.normalise_solution(xo, g.n_u, s.MQ, k)
    P.close()
    return rep, ro, xg, xr, s


@pytest.mark.parametrize("n", [8, 32])
def test_minres_p3_parity(n):
    rep, ro, xg, xr, s = _minres_parity(n, etq.PC_P3, lambda s: precond.StokesP3(s), inner_rtol=1e-13)
    assert rep["converged"] and ro.converged
    assert abs(rep["iterations"] - ro.iterations) <= 2
    assert rel_err(xg, xr) < 1e-8
    m = min(len(rep["delta"]), len(ro.delta))
    np.testing.assert_allclose(rep["delta"][:m], ro.delta[:m], rtol=1e-9, atol=1e-12)


@pytest.mark.parametrize("n", [16, 32])
def test_minres_p1_iter_matches_exact_p1(n):
    """P1 at scale (A^{-1} by V-cycle-PCG, exact M_Q through S_k) reproduces the oracle's P1
    (sparse direct A^{-1}, bordered M_Q solve): same iteration count (c1 at n = 16) and solution."""
    rep, ro, xg, xr, s = _minres_parity(n, etq.PC_P1_ITER, lambda s: precond.StokesP1(s), inner_rtol=1e-13)
    assert rep["converged"] and ro.converged
    assert abs(rep["iterations"] - ro.iterations) <= 1
    assert rel_err(xg, xr) < 1e-8
    m = min(len(rep["delta"]), len(ro.delta))
    np.testing.assert_allclose(rep["delta"][:m], ro.delta[:m], rtol=1e-9, atol=1e-12)


def test_minres_p1_iter_c2_force():
    """Homogeneous BC with the N(0,1) nodal force (c2's right-hand side) at n = 64."""
    rep, ro, xg, xr, s = _minres_parity(64, etq.PC_P1_ITER, lambda s: precond.StokesP1(s), bc="homogeneous",
                                        force=True)
    assert rep["converged"] and ro.converged
    assert abs(rep["iterations"] - ro.iterations) <= 2
    assert rel_err(xg, xr) < 1e-8


def test_p3_iterations_mesh_independent():
    """With the exact M_Q block the MINRES count stops growing with n (Table-1 behaviour,
    P:578-580), unlike P2 (Table 2)."""
    its = {}
    for n in (64, 256, 1024):
        P = etq.Problem(n)
        _setup(P)
        b = torch.zeros(P.N, dtype=torch.float64, device=DEV)
        P.build_rhs(b)
        x = torch.zeros(P.N, dtype=torch.float64, device=DEV)
        rep = P.minres_solve(etq.PC_P3, b, x, rtol=1e-8, maxit=1000)
        assert rep["converged"]
        its[n] = rep["iterations"]
        # true residual of the returned iterate
        y = torch.zeros(P.N, dtype=torch.float64, device=DEV)
        P.apply_saddle(x, y)
        assert float(torch.linalg.norm(b - y) / torch.linalg.norm(b)) < 1e-6
        P.close()
    assert its[1024] <= its[64] + 10, its
