"""GPU parity of SURVEY §8(f) NEXT-3: Oseen operators with a nodal Q2 wind (the Picard wind) and the
Picard loop, against oracle.picard (4 x 4 Gauss element assembly, exact bordered solves)."""
import numpy as np
import pytest
import scipy.sparse as sp

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

from oracle import fem, mg, normalize, picard  # noqa: E402
from paper_2303_10233_b200 import etq  # noqa: E402
import synth  # noqa: E402

DEV = torch.device("cuda:0")
NU = 0.01


def dev(a):
    return torch.as_tensor(np.ascontiguousarray(a), dtype=torch.float64, device=DEV)


def host(t):
    torch.cuda.synchronize()
    return t.detach().cpu().numpy()


def sp_rel_diff(A, B):
    D = (A - B).tocsr()
    return (np.abs(D.data).max() if D.nnz else 0.0) / np.abs(B.data).max()


def _wind(n, seed):
    g = fem.Grid(n)
    w = synth.random_vector(g.n_u, seed=seed)
    return g, w


def test_cavity_wind_as_nodal_wind_matches_kind1():
    """The c4 wind lies in Q2: set as a nodal wind it reproduces the analytic-wind problem."""
    n = 16
    g = fem.Grid(n)
    x, y = g.node_xy()
    wx, wy = fem.cavity_wind(x, y)
    P2 = etq.Problem(n, bc=0, viscosity=NU, wind=2)
    P2.set_wind(dev(np.concatenate([wx, wy])))
    P1 = etq.Problem(n, bc=0, viscosity=NU, wind=1, storage=2)
    assert sp_rel_diff(P2.export_operator(0), P1.export_operator(0)) < 1e-13
    b1 = torch.zeros(P1.N, dtype=torch.float64, device=DEV)
    b2 = torch.zeros(P2.N, dtype=torch.float64, device=DEV)
    P1.build_rhs(b1)
    P2.build_rhs(b2)
    np.testing.assert_allclose(host(b2), host(b1), rtol=0, atol=1e-13 * float(b1.abs().max()))


@pytest.mark.parametrize("n", [4, 16])
def test_nodal_wind_operators_entrywise(n):
    """F = nu L + N(w) on every MG level (coarse winds injected), F1 and the lifted RHS against the
    oracle's 4 x 4 Gauss element assembly, entry by entry."""
    g, w = _wind(n, 31)
    P = etq.Problem(n, bc=0, viscosity=NU, wind=2)
    P.set_wind(dev(w))
    P.precond_setup(etq.PC_OSEEN_M1, etq.make_params(coarse_n=2))
    P.precond_setup(etq.PC_OSEEN_PCD1, etq.make_params(coarse_n=2))
    s = picard.oseen_system(n, NU, w[:g.nq], w[g.nq:])
    assert sp_rel_diff(P.export_operator(0), s.Ls) < 1e-13
    # coarser levels: rediscretised with the injected wind, identity Dirichlet rows
    m, wl, l = n, w, 0
    while m > 2:
        gf = fem.Grid(m)
        mc = m // 2
        gc = fem.Grid(mc)
        I, J = np.meshgrid(np.arange(gc.m), np.arange(gc.m), indexing="xy")
        fine = (2 * I + gf.m * 2 * J).ravel()
        wl = np.concatenate([wl[:gf.nq][fine], wl[gf.nq:][fine]])
        l += 1
        ref = mg.dirichlet_scalar((NU * fem.laplacian(gc) + picard.convection_nodal(gc, wl[:gc.nq], wl[gc.nq:])).tocsr(), gc)
        assert sp_rel_diff(P.export_operator(0, l), ref) < 1e-13, l
        m = mc
    F1 = picard.pcd_f1_nodal(g, NU, w[:g.nq], w[g.nq:])
    assert sp_rel_diff(P.export_operator(4), F1) < 1e-13
    b = torch.zeros(P.N, dtype=torch.float64, device=DEV)
    P.build_rhs(b)
    np.testing.assert_allclose(host(b), s.b, rtol=0, atol=1e-13 * np.abs(s.b).max())


def test_picard_iterates_match_oracle():
    """Three Picard steps from the Stokes start with tight inner solves: the GPU's
    last iterate equals the oracle's exact Picard iterate (normalised pressures, reading R19)."""
    n, steps = 16, 3
    g = fem.Grid(n)
    P = etq.Problem(n, bc=0, viscosity=NU, wind=2)
    prm = etq.make_params(coarse_n=8)
    P.precond_setup(etq.PC_OSEEN_M1, prm)
    P.precond_setup(etq.PC_OSEEN_PCD1, prm)
    x = torch.zeros(P.N, dtype=torch.float64, device=DEV)
    out = P.picard_solve(x, steps=steps, eta=1e-11, c=10.0, restart=50, maxit=3000)
    assert out["status"] == 0
    assert np.all(out["rel_res"] < 1e-9)
    xs, systems = picard.picard(n, NU, steps=steps)
    xg, xr = host(x), xs[-1]
    assert np.abs(xg[:g.n_u] - xr[:g.n_u]).max() <= 1e-8 * np.abs(xr[:g.n_u]).max()
    # pressures: both satisfy the same system; compare after removing the 2-D null space
    s = systems[-1]
    for v in (xg, xr):
        v[g.n_u:g.n_u + g.n_k] -= v[g.n_u:g.n_u + g.n_k].mean()
        v[g.n_u + g.n_k:] -= v[g.n_u + g.n_k:].mean()
    assert np.abs(xg[g.n_u:] - xr[g.n_u:]).max() <= 1e-8 * np.abs(xr[g.n_u:]).max()
    assert np.linalg.norm(s.K @ xg - s.b) <= 1e-8 * np.linalg.norm(s.b)


def test_set_wind_rejects_other_kinds():
    P = etq.Problem(8, bc=0, viscosity=NU, wind=1)
    with pytest.raises(etq.EtqError):
        P.set_wind(torch.zeros(P.n_u, dtype=torch.float64, device=DEV))
