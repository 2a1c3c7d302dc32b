"""Out-of-bounds write guards for the caller-owned vectors (compute-sanitizer is closed on this GPU
pool, so the library's user-facing writes are checked with our own canaries instead).

Every caller vector handed to the C ABI is a view into a larger buffer whose leading and trailing
guard zones hold a signalling bit pattern; after each apply / solve the guards must be untouched and
the outputs finite.  Sizes cover interior and ragged last tiles of every tiled kernel (the smoother
tiles are 56 wide, the saddle tiles 64, the Chebyshev-SGS tiles 50 x 26 / 50 x 58), both SGS
geometries and the Oseen path with its matrix-free F rows.
"""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

from paper_2303_10233_b200 import etq  # noqa: E402
import synth  # noqa: E402

G = 4099                                     # guard elements on each side (odd: misaligned views)
CANARY = np.frombuffer(np.uint64(0x7FF4DEADBEEF0001).tobytes(), dtype=np.float64)[0]   # a NaN payload


class Guarded:
    """A length-n float64 CUDA view with guard zones before and after it."""

    def __init__(self, n, init=None):
        self.n = n
        self.buf = torch.full((n + 2 * G,), float(CANARY), dtype=torch.float64, device="cuda")
        self.v = self.buf[G:G + n]
        if init is None:
            self.v.zero_()
        else:
            self.v.copy_(torch.as_tensor(init, device="cuda"))

    def check(self, what):
        torch.cuda.synchronize()
        raw = self.buf.view(torch.int64).cpu().numpy()
        pat = np.int64(np.uint64(0x7FF4DEADBEEF0001).astype(np.int64))
        assert np.all(raw[:G] == pat), f"{what}: write before the vector"
        assert np.all(raw[G + self.n:] == pat), f"{what}: write after the vector"
        assert torch.isfinite(self.v).all().item(), f"{what}: non-finite output"


@pytest.mark.parametrize("n", [64, 128, 512])
def test_stokes_applies_and_solve_stay_in_bounds(n):
    P = etq.Problem(n)
    P.precond_setup(etq.PC_P2_GMG, etq.make_params(cheb_sgs_lo=0.005))
    x = Guarded(P.N, synth.random_vector(P.N, seed=n))
    y = Guarded(P.N)
    P.apply_saddle(x.v, y.v)
    x.check("saddle input"); y.check("saddle")
    z = Guarded(P.N)
    P.apply_precond(etq.PC_P2_GMG, x.v, z.v)
    z.check("P2 apply")
    zu = Guarded(P.n_u)
    P.apply_vcycle(etq.PC_P2_GMG, x.v[:P.n_u], zu.v)
    zu.check("V-cycle")
    for win in (1, 2, 3):
        etq.set_option(16, win)
        try:
            zp = Guarded(P.n_p)
            P.apply_mass_pc(x.v[P.n_u:], zp.v)
            zp.check(f"Pi C Pi (SGS geometry {win})")
        finally:
            etq.set_option(16, 0)
    b = Guarded(P.N)
    P.build_rhs(b.v)
    b.check("rhs")
    xs = Guarded(P.N)
    rep = P.minres_solve(etq.PC_P2_GMG, b.v, xs.v, rtol=1e-6, maxit=60)
    xs.check("MINRES solution")
    assert rep["iterations"] > 0
    P.close()


def test_oseen_two_stage_stays_in_bounds():
    n = 128
    P = etq.Problem(n, bc=0, viscosity=0.01, wind=1)
    P.precond_setup(etq.PC_OSEEN_M1, etq.make_params(cheb_sgs_lo=0.005))
    P.precond_setup(etq.PC_OSEEN_PCD1)
    r = Guarded(P.N, synth.random_vector(P.N, seed=3))
    for kind in (etq.PC_OSEEN_M1, etq.PC_OSEEN_PCD1):
        z = Guarded(P.N)
        if kind == etq.PC_OSEEN_PCD1:
            rr = Guarded(P.N, synth.random_vector(P.N, seed=3))
            rr.v[P.n_u + P.n_k:] = 0.0
            P.apply_precond(kind, rr.v, z.v)
        else:
            P.apply_precond(kind, r.v, z.v)
        z.check(f"Oseen preconditioner {kind}")
    b = Guarded(P.N)
    P.build_rhs(b.v)
    x = Guarded(P.N)
    out = P.two_stage_solve(b.v, x.v, eta=1e-6, c=10.0, restart=50, maxit=400)
    x.check("two-stage solution")
    assert out["step2"]["converged"]
    P.close()
