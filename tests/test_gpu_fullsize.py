"""Full-size parity at BASELINE.json's sizes, in the launch configuration bench.py times.

* c3 (n = 1024, Stokes lid cavity, P2): every operator apply of the path — the saddle SpMV
  (P:127-142), one V-cycle on both velocity components (reading R9), the Pi C Pi
  Chebyshev-SGS pressure apply (readings R6/R7) and the whole P2 apply —
  compared with the oracle ELEMENT BY ELEMENT at 1e-12 relative; then the whole 397-iteration
  MINRES solve (Algorithm 1) against the oracle's full-length record
  (tests/golden/c3_minres_p2_n1024.json, written by scripts/oracle_golden.py, which imports only
  oracle/ and synth/): iteration count +-2, the complete |eta_j|, delta_j, gamma_j histories,
  and the O12-normalised solution at 20000 seeded positions within 1e-8.
* c4 (n = 512, Oseen nu = 0.01, two-stage PCD): the M1 and PCD1 preconditioner applies
   element by element at 1e-12, then the two-stage solve
   against tests/golden/c4_two_stage_n512.json: Step I / II iterations +-2 and
  residual histories, ||z*|| and the Prop 3.3 bound, the sampled solution within 1e-8.
"""
import json
import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

from oracle import fem, mg, normalize, oseen, precond  # noqa: E402
from paper_2303_10233_b200 import etq  # noqa: E402
import synth  # noqa: E402

DEV = torch.device("cuda:0")
GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")
APPLY_TOL = 1e-12
SOL_TOL = 1e-8
A_C3 = 0.005


def dev(a):
    return torch.as_tensor(np.ascontiguousarray(a), dtype=torch.float64, device=DEV)


def host(t):
    torch.cuda.synchronize()
    return t.detach().cpu().numpy()


def rel_err(a, b):
    return float(np.abs(a - b).max() / max(np.abs(b).max(), 1e-300))


def golden(name):
    path = os.path.join(GOLDEN, name)
    if not os.path.exists(path):
        pytest.fail(f"missing golden record {path} (run scripts/oracle_golden.py)")
    return json.load(open(path))


def sampled_solution_check(xg, rec, s):
    """O12-normalised GPU solution vs the oracle's stored sample (1e-8 relative to max|x|)."""
    g = s.g
    xn = normalize.normalise_solution(xg, g.n_u, s.MQ, fem.null_vector_k(g))
    sol = rec["solution"]
    idx = synth.sample_indices(g.N, sol["sample_count"], sol["sample_seed"])
    ref = np.asarray(sol["values"])
    err = float(np.abs(xn[idx] - ref).max() / sol["max_abs"])
    assert err < SOL_TOL, err
    assert abs(np.abs(xn).max() - sol["max_abs"]) <= SOL_TOL * sol["max_abs"]
    assert abs(np.linalg.norm(xn[:g.n_u]) - sol["norm_u"]) <= SOL_TOL * sol["norm_u"]
    assert abs(np.linalg.norm(xn[g.n_u:]) - sol["norm_p"]) <= SOL_TOL * sol["norm_p"]
    return err


@pytest.fixture(scope="module")
def c3():
    n = 1024
    s = fem.assemble_system(n)
    Pr = precond.StokesP2(s, A_C3, hierarchy=mg.Hierarchy(n))
    P = etq.Problem(n)
    P.precond_setup(etq.PC_P2_GMG, etq.make_params(cheb_sgs_lo=A_C3))
    yield s, Pr, P
    P.close()


def test_c3_applies_elementwise(c3):
    s, Pr, P = c3
    g = s.g
    x = synth.random_vector(g.N, seed=1031)
    xd = dev(x)
    y = torch.zeros(g.N, dtype=torch.float64, device=DEV)
    P.apply_saddle(xd, y)
    assert rel_err(host(y), s.K @ x) < APPLY_TOL
    zu = torch.zeros(g.n_u, dtype=torch.float64, device=DEV)
    P.apply_vcycle(etq.PC_P2_GMG, dev(x[:g.n_u]), zu)
    zu_ref = Pr.velocity(x[:g.n_u])
    assert rel_err(host(zu), zu_ref) < APPLY_TOL
    zp = torch.zeros(g.n_p, dtype=torch.float64, device=DEV)
    P.apply_mass_pc(dev(x[g.n_u:]), zp)
    zp_ref = Pr.pressure(x[g.n_u:])
    assert rel_err(host(zp), zp_ref) < APPLY_TOL
    z = torch.zeros(g.N, dtype=torch.float64, device=DEV)
    P.apply_precond(etq.PC_P2_GMG, xd, z)
    zh = host(z)
    assert rel_err(zh[:g.n_u], zu_ref) < APPLY_TOL and rel_err(zh[g.n_u:], zp_ref) < APPLY_TOL


def test_c3_minres_full_length_vs_golden(c3):
    s, _, P = c3
    rec = golden("c3_minres_p2_n1024.json")
    assert rec["n"] == 1024 and rec["a"] == A_C3 and rec["converged"]
    b = torch.zeros(P.N, dtype=torch.float64, device=DEV)
    P.build_rhs(b)
    assert rel_err(host(b), s.b) < APPLY_TOL
    x = torch.zeros(P.N, dtype=torch.float64, device=DEV)
    rep = P.minres_solve(etq.PC_P2_GMG, b, x, rtol=rec["rtol"], maxit=rec["maxit"])
    assert rep["converged"]
    assert abs(rep["iterations"] - rec["iterations"]) <= 2, (rep["iterations"], rec["iterations"])
    k = min(rep["iterations"], rec["iterations"])
    hist_o = np.asarray(rec["history"])        # |eta_0| = gamma_1, |eta_1|, ...
    # relative drift of the recurrences over the whole solve (rounding-order differences only)
    np.testing.assert_allclose(rep["delta"][:k], np.asarray(rec["delta"])[:k], rtol=1e-6)
    np.testing.assert_allclose(rep["gamma"][:k], np.asarray(rec["gamma"])[1:k + 1], rtol=1e-6)
    np.testing.assert_allclose(rep["history"][:k], hist_o[1:k + 1], rtol=1e-6)
    sampled_solution_check(host(x), rec, s)


@pytest.fixture(scope="module")
def c4():
    n, nu = 512, 0.01
    s = fem.assemble_system(n, nu=nu)
    hF = oseen.velocity_hierarchy(n, nu, n_coarse=32)
    schur = oseen.PCDSchur(s, nu)
    P = etq.Problem(n, bc=0, viscosity=nu, wind=1)
    P.precond_setup(etq.PC_OSEEN_M1, etq.make_params(cheb_sgs_lo=0.005))
    P.precond_setup(etq.PC_OSEEN_PCD1)
    yield s, hF, schur, P
    P.close()


def test_c4_applies_elementwise(c4):
    s, hF, schur, P = c4
    g = s.g
    r = synth.random_vector(g.N, seed=513)
    z = torch.zeros(g.N, dtype=torch.float64, device=DEV)
    P.apply_precond(etq.PC_OSEEN_M1, dev(r), z)
    assert rel_err(host(z), oseen.OseenM1(s, hF, 0.01, 0.005)(r)) < APPLY_TOL
    nr = g.n_u + g.n_k
    rr = r.copy(); rr[nr:] = 0.0
    P.apply_precond(etq.PC_OSEEN_PCD1, dev(rr), z)
    zo = oseen.OseenPCD1(s, hF, schur)(r[:nr])
    assert rel_err(host(z)[:nr], zo) < APPLY_TOL
    y = torch.zeros(g.N, dtype=torch.float64, device=DEV)
    P.apply_saddle(dev(r), y)
    assert rel_err(host(y), s.K @ r) < APPLY_TOL


def test_c4_two_stage_vs_golden(c4):
    s, _, _, P = c4
    rec = golden("c4_two_stage_n512.json")
    b = torch.zeros(P.N, dtype=torch.float64, device=DEV)
    P.build_rhs(b)
    x = torch.zeros(P.N, dtype=torch.float64, device=DEV)
    out = P.two_stage_solve(b, x, eta=rec["eta"], c=rec["c"], restart=rec["restart"], maxit=rec["maxit"])
    for st in ("step1", "step2"):
        assert out[st]["converged"] and rec[st]["converged"]
        assert abs(out[st]["iterations"] - rec[st]["iterations"]) <= 2, (st, out[st]["iterations"],
                                                                        rec[st]["iterations"])
        k = min(len(out[st]["history"]), len(rec[st]["history"]))
        np.testing.assert_allclose(out[st]["history"][:k], np.asarray(rec[st]["history"])[:k], rtol=1e-6)
    assert out["zstar"] == pytest.approx(rec["zstar"], rel=1e-9)
    assert out["bound"] == pytest.approx(rec["bound"], rel=1e-9)
    assert out["zstar"] <= out["bound"] * (1 + 1e-12)          # Prop 3.3
    sampled_solution_check(host(x), rec, s)
