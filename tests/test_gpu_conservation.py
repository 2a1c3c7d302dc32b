"""GPU local mass conservation, the paper's headline property of Q2-Q1* (P:196-202): the converged
enriched solution satisfies B0 u = g0 element by element, while plain Taylor-Hood Q2-Q1 on the
same mesh (etq_grid.enriched = 0) violates it by orders of magnitude.  The plain GPU path is
checked against the oracle's plain MINRES (iterations +-2, mean-free solution 1e-8)."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

from oracle import fem, krylov, precond  # noqa: E402
from paper_2303_10233_b200 import etq  # noqa: E402

DEV = torch.device("cuda:0")


def zeros(n):
    return torch.zeros(n, dtype=torch.float64, device=DEV)


def host(t):
    torch.cuda.synchronize()
    return t.cpu().numpy()


def _solve(n, enriched, rtol):
    P = etq.Problem(n, enriched=enriched)
    P.precond_setup(etq.PC_P2_GMG, etq.make_params(cheb_sgs_lo=0.005))
    b = zeros(P.N); P.build_rhs(b)
    x = zeros(P.N)
    rep = P.minres_solve(etq.PC_P2_GMG, b, x, rtol=rtol, maxit=2000)
    return P, b, x, rep


@pytest.mark.parametrize("n", [16, 64])
def test_plain_q2q1_matches_oracle(n):
    s = fem.assemble_system(n)
    g = s.g
    P, b, x, rep = _solve(n, False, 1e-10)
    nr = g.n_u + g.n_k
    bh = host(b)
    K, bo = precond.plain_system(s)
    assert np.abs(bh[:nr] - bo).max() <= 1e-12 * np.abs(bo).max() and np.all(bh[nr:] == 0.0)
    xo, ro = krylov.minres(lambda v: K @ v, bo, precond.StokesP2Plain(s), rtol=1e-10, maxit=2000)
    assert rep["converged"] and ro.converged and abs(rep["iterations"] - ro.iterations) <= 2
    xg = host(x)
    assert np.all(xg[nr:] == 0.0)
    xg = xg[:nr].copy()
    for v in (xg, xo):
        v[g.n_u:] -= v[g.n_u:].mean()
    assert np.abs(xg - xo).max() <= 1e-8 * np.abs(xo).max()
    # the plain saddle apply is the reduced operator
    y = zeros(P.N)
    P.apply_saddle(x, y)
    assert np.abs(host(y)[:nr] - K @ host(x)[:nr]).max() <= 1e-12 * np.abs(K @ host(x)[:nr]).max()


@pytest.mark.parametrize("n", [16, 128])
def test_local_conservation_contrast(n):
    """max_T |(B0 u - g0)_T| <= 10 rtol ||b|| for Q2-Q1* and >= 100x larger for plain Q2-Q1."""
    s = fem.assemble_system(n)
    g = s.g
    g0 = s.b[g.n_u + g.n_k:]
    rtol = 1e-10
    _, _, xs, rs = _solve(n, True, rtol)
    _, _, xp, rp = _solve(n, False, rtol)
    assert rs["converged"] and rp["converged"]
    star = np.abs(s.B0 @ host(xs)[:g.n_u] - g0).max()
    plain = np.abs(s.B0 @ host(xp)[:g.n_u] - g0).max()
    assert star <= 10 * rtol * np.linalg.norm(s.b)
    assert plain >= 100 * star, (plain, star)


def test_plain_rejects_other_preconditioners_and_oseen():
    P = etq.Problem(8, enriched=False)
    with pytest.raises(etq.EtqError):
        P.precond_setup(etq.PC_P1_EXACT)
    with pytest.raises(etq.EtqError):
        etq.Problem(8, viscosity=0.01, wind=1, enriched=False)
