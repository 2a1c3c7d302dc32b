"""The temporally blocked Chebyshev smoother (one kernel per pre/post-smoothing pass on the
Stokes interior-stencil levels) against the one-kernel-per-step path: bitwise-identical V-cycles
(same per-row arithmetic and summation order, reading R2's eliminated Dirichlet columns) and the
oracle V-cycle within the apply tolerance."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

from oracle import mg  # noqa: E402
from paper_2303_10233_b200 import etq  # noqa: E402
import synth  # noqa: E402


def _vcycle(n, tile, bc=0, min_n=32, tile2=1, tile3=0):
    etq.set_option(0, 1 if tile else 0)
    etq.set_option(1, min_n)
    etq.set_option(11, tile2)
    etq.set_option(12, tile3)
    try:
        P = etq.Problem(n, bc=bc)
        P.precond_setup(etq.PC_P2_GMG, etq.make_params(cheb_sgs_lo=0.005))
        r = torch.as_tensor(synth.random_vector(P.n_u, seed=21), device="cuda")
        z = torch.zeros(P.n_u, dtype=torch.float64, device="cuda")
        P.apply_vcycle(etq.PC_P2_GMG, r, z)
        torch.cuda.synchronize()
        out = z.cpu().numpy()
        P.close()
        return out
    finally:
        etq.set_option(0, 1)
        etq.set_option(1, 64)
        etq.set_option(11, 1)
        etq.set_option(12, 1)


@pytest.mark.parametrize("n,bc", [(32, 0), (64, 1), (128, 0), (512, 0)])
def test_tiled_smoother_bitwise_equal(n, bc):
    """k_cheb_tile (stored-row summation order) is bitwise the per-step path; k_cheb_tile2 sums the
    mirrored taps first (grouped weights), so it agrees to rounding."""
    a = _vcycle(n, True, bc, tile2=0)
    b = _vcycle(n, False, bc)
    np.testing.assert_array_equal(a, b)
    c = _vcycle(n, True, bc, tile2=1)
    assert np.abs(c - b).max() <= 1e-14 * np.abs(b).max()


@pytest.mark.parametrize("n,bc", [(32, 0), (64, 1), (128, 0), (256, 1), (512, 0), (1024, 1)])
def test_tile3_smoother_bitwise_equal_tile2(n, bc):
    """k_cheb_tile3 (residual in registers, one output map for the three steps, outputs written from
    the last step) performs k_cheb_tile2's arithmetic in the same order: bitwise-identical V-cycles
    (ragged last tiles at every n; n = 1024: the c3 finest level)."""
    a = _vcycle(n, True, bc, tile2=1, tile3=0)
    b = _vcycle(n, True, bc, tile2=1, tile3=1)
    np.testing.assert_array_equal(a, b)


def _minres_tile3(n, tile3):
    etq.set_option(12, tile3)
    try:
        P = etq.Problem(n)
        P.precond_setup(etq.PC_P2_GMG, etq.make_params(cheb_sgs_lo=0.005))
        b = torch.zeros(P.N, dtype=torch.float64, device="cuda")
        P.build_rhs(b)
        x = torch.zeros_like(b)
        rep = P.minres_solve(etq.PC_P2_GMG, b, x, rtol=1e-8, maxit=500)
        out = x.cpu().numpy(), rep["iterations"]
        P.close()
        return out
    finally:
        etq.set_option(12, 1)


def test_tile3_minres_bitwise_equal_tile2():
    """The finest post pass of k_cheb_tile3 also writes z = x + d2 and the <z, v> partials inside the
    MINRES graph.  z is bitwise k_cheb_tile2's (test above); the <z, v> partials are summed per thread
    over a different set of outputs (one output map for all steps), so gamma_j differs in the last
    bits (deterministic either way): same iterations, solutions equal to rounding."""
    x0, i0 = _minres_tile3(256, 0)
    x1, i1 = _minres_tile3(256, 1)
    assert i0 == i1
    assert np.abs(x1 - x0).max() <= 1e-12 * np.abs(x0).max()


def test_tiled_vcycle_matches_oracle():
    n = 64
    z = _vcycle(n, True)
    h = mg.Hierarchy(n)
    r = synth.random_vector(2 * (2 * n + 1) ** 2, seed=21)
    ref = h.apply_velocity(r)
    assert np.abs(z - ref).max() <= 1e-12 * np.abs(ref).max()


def test_set_option_rejects_unknown():
    with pytest.raises(etq.EtqError):
        etq.set_option(99, 1)
    with pytest.raises(etq.EtqError):
        etq.set_option(1, 0)


@pytest.mark.parametrize("tiled", [0, 1])
@pytest.mark.parametrize("n", [15, 16, 64, 130, 256])
def test_matrix_free_saddle_bitwise_equal(n, tiled):
    """The matrix-free Stokes saddle apply (class stencils of L, B^T and B) equals the stored-row
    apply, full and reduced: the velocity rows bitwise; the pressure rows bitwise for the gather
    kernel and to rounding for the tiled kernel, which sums each component's B u terms from the
    velocity walk's register window separately (u_x part + u_y part instead of interleaved)."""
    ys = {}
    x = None
    etq.set_option(6, tiled)
    for opt in (0, 1):
        etq.set_option(2, opt)
        try:
            P = etq.Problem(n)
            x = torch.as_tensor(synth.random_vector(P.N, seed=7), device="cuda")
            for red in (False, True):
                y = torch.zeros(P.N, dtype=torch.float64, device="cuda")
                P.apply_saddle(x, y, reduced=red)
                torch.cuda.synchronize()
                ys[(opt, red)] = y.cpu().numpy()
            P.close()
        finally:
            etq.set_option(2, 1)
    etq.set_option(6, 1)
    n_u = 2 * (2 * n + 1) ** 2
    for red in (False, True):
        np.testing.assert_array_equal(ys[(0, red)][:n_u], ys[(1, red)][:n_u])
        if tiled:
            scale = np.abs(ys[(0, red)][n_u:]).max()
            assert np.abs(ys[(0, red)][n_u:] - ys[(1, red)][n_u:]).max() <= 1e-14 * scale
        else:
            np.testing.assert_array_equal(ys[(0, red)][n_u:], ys[(1, red)][n_u:])


@pytest.mark.parametrize("n", [64, 256])
def test_saddle_apply_any_output_alignment(n):
    """The tiled saddle apply stores aligned 16-byte pairs; an output vector that is only 8-byte
    aligned (a view at element offset 1) and one at offset 2 get bitwise the same values."""
    P = etq.Problem(n)
    x = torch.as_tensor(synth.random_vector(P.N, seed=8), device="cuda")
    buf = torch.zeros(P.N + 2, dtype=torch.float64, device="cuda")
    outs = []
    for off in (1, 2):
        buf.zero_()
        y = buf[off:off + P.N]
        P.apply_saddle(x, y)
        torch.cuda.synchronize()
        outs.append(y.cpu().numpy().copy())
        assert buf[:off].abs().sum().item() == 0.0 and buf[off + P.N:].abs().sum().item() == 0.0
    P.close()
    np.testing.assert_array_equal(outs[0], outs[1])


@pytest.mark.parametrize("n", [64, 512, 1024])
def test_sgs_window_heights_agree(n):
    """Chebyshev-SGS with 64 x 64 windows (512 threads), 64 x 32 windows with 256 threads (two plane
    rows per thread) and with 512 threads (one row): every halo is the exact dependency cone, so one
    symmetric sweep is bitwise the same; the Pi C Pi apply agrees to rounding (its k^T y reduction
    runs over a different tile grid)."""
    P = etq.Problem(n)
    P.precond_setup(etq.PC_P2_GMG, etq.make_params(cheb_sgs_lo=0.005))
    r = torch.as_tensor(synth.random_vector(P.n_p, seed=31), device="cuda")
    y = torch.as_tensor(synth.random_vector(P.n_p, seed=32), device="cuda")
    outs = {}
    try:
        for win in (1, 2, 3):
            etq.set_option(16, win)
            z = torch.zeros(P.n_p, dtype=torch.float64, device="cuda")
            P.sgs_sweep(r, y, z)
            w = torch.zeros(P.n_p, dtype=torch.float64, device="cuda")
            P.apply_mass_pc(r, w)
            torch.cuda.synchronize()
            outs[win] = (z.cpu().numpy(), w.cpu().numpy())
    finally:
        etq.set_option(16, 0)
    P.close()
    for win in (2, 3):
        np.testing.assert_array_equal(outs[1][0], outs[win][0])
        assert np.abs(outs[1][1] - outs[win][1]).max() <= 1e-14 * np.abs(outs[1][1]).max()


@pytest.mark.parametrize("n", [16, 64, 256])
def test_oseen_matrix_free_rows_match_stored_rows(n):
    """Cavity-wind Oseen problem (storage 0): the matrix-free F (nu L class stencils + 1D convection
    tables), B^T and B of the saddle apply (full and reduced), the matrix-free B^T of M1 and the
    matrix-free interior rows of the F V-cycle levels agree with the stored SELL rows to rounding
    (debug option 14 switches all of them)."""
    out = {}
    try:
        for opt in (0, 1):
            etq.set_option(14, opt)
            P = etq.Problem(n, bc=0, viscosity=0.01, wind=1)
            P.precond_setup(etq.PC_OSEEN_M1, etq.make_params(cheb_sgs_lo=0.005, coarse_n=8))
            x = torch.as_tensor(synth.random_vector(P.N, seed=41), device="cuda")
            res = []
            for red in (False, True):
                y = torch.zeros(P.N, dtype=torch.float64, device="cuda")
                P.apply_saddle(x, y, reduced=red)
                res.append(y.cpu().numpy())
            z = torch.zeros(P.N, dtype=torch.float64, device="cuda")
            P.apply_precond(etq.PC_OSEEN_M1, x, z)
            torch.cuda.synchronize()
            res.append(z.cpu().numpy())
            out[opt] = res
            P.close()
    finally:
        etq.set_option(14, 1)
    for a, b in zip(out[0], out[1]):
        assert np.abs(a - b).max() <= 1e-13 * np.abs(a).max()


@pytest.mark.parametrize("kind", [etq.PC_P2_GMG, etq.PC_P3])
def test_device_minres_loop_matches_host_loop(kind):
    """MINRES as one CUDA graph with a while node (no host round trip per iteration) gives the same
    iterates as one graph launch plus one flag read-back per iteration."""
    n = 32
    xs, its = [], []
    for opt in (0, 1):
        etq.set_option(3, opt)
        try:
            P = etq.Problem(n)
            P.precond_setup(kind, etq.make_params(cheb_sgs_lo=0.005))
            b = torch.zeros(P.N, dtype=torch.float64, device="cuda")
            P.build_rhs(b)
            x = torch.zeros(P.N, dtype=torch.float64, device="cuda")
            rep = P.minres_solve(kind, b, x, rtol=1e-8, maxit=500)
            xs.append(x.cpu().numpy()); its.append(rep["iterations"])
            P.close()
        finally:
            etq.set_option(3, 1)
    assert its[0] == its[1]
    np.testing.assert_array_equal(xs[0], xs[1])


@pytest.mark.parametrize("option", [5, 9])
@pytest.mark.parametrize("n", [32, 64, 256])
def test_vcycle_fusions_bitwise_equal(n, option):
    """Option 5: the coarse-level tail run in shared memory with the class stencils; option 9: the
    tiled prolongation.  Either way the V-cycle output is the same, bit for bit, as with the
    global-memory kernels."""
    zs = {}
    for opt in (0, 1):
        etq.set_option(option, opt)
        try:
            P = etq.Problem(n)
            P.precond_setup(etq.PC_P2_GMG, etq.make_params(cheb_sgs_lo=0.005))
            r = torch.as_tensor(synth.random_vector(P.n_u, seed=11), device="cuda")
            z = torch.zeros(P.n_u, dtype=torch.float64, device="cuda")
            P.apply_vcycle(etq.PC_P2_GMG, r, z)
            torch.cuda.synchronize()
            zs[opt] = z.cpu().numpy()
            P.close()
        finally:
            etq.set_option(option, 1)
    np.testing.assert_array_equal(zs[0], zs[1])


@pytest.mark.parametrize("option,kind", [(7, etq.PC_P2_GMG), (8, etq.PC_P3)])
def test_programmatic_dependent_launches_bitwise_equal(option, kind):
    """Programmatic dependent launches (option 7: between the Chebyshev-SGS steps; option 8: between
    the V-cycle kernels, used by P3) change only when the next kernel's CTAs launch: the MINRES
    iterates are bit for bit the same with them off."""
    n = 64
    xs, its = [], []
    for opt in (0, 1):
        etq.set_option(option, opt)
        try:
            P = etq.Problem(n)
            P.precond_setup(kind, etq.make_params(cheb_sgs_lo=0.005))
            b = torch.zeros(P.N, dtype=torch.float64, device="cuda")
            P.build_rhs(b)
            x = torch.zeros(P.N, dtype=torch.float64, device="cuda")
            rep = P.minres_solve(kind, b, x, rtol=1e-8, maxit=500)
            xs.append(x.cpu().numpy()); its.append(rep["iterations"])
            P.close()
        finally:
            etq.set_option(option, 1)
    assert its[0] == its[1]
    np.testing.assert_array_equal(xs[0], xs[1])


def _mass_pc(n, planar, seed=77, m=20, oseen=False):
    etq.set_option(10, 1 if planar else 0)
    try:
        if oseen:
            P = etq.Problem(n, bc=0, viscosity=0.01, wind=1)
            P.precond_setup(etq.PC_OSEEN_M1, etq.make_params(cheb_sgs_lo=0.005, cheb_sgs_steps=m, coarse_n=2))
            r = torch.as_tensor(synth.random_vector(P.N, seed=seed), device="cuda")
            z = torch.zeros(P.N, dtype=torch.float64, device="cuda")
            P.apply_precond(etq.PC_OSEEN_M1, r, z)
        else:
            P = etq.Problem(n)
            P.precond_setup(etq.PC_P2_GMG, etq.make_params(cheb_sgs_lo=0.005, cheb_sgs_steps=m))
            r = torch.as_tensor(synth.random_vector(P.n_p, seed=seed), device="cuda")
            z = torch.zeros(P.n_p, dtype=torch.float64, device="cuda")
            P.apply_mass_pc(r, z)
        torch.cuda.synchronize()
        out = z.cpu().numpy()
        P.close()
        return out
    finally:
        etq.set_option(10, 0)


@pytest.mark.parametrize("n,m", [(2, 20), (4, 3), (16, 20), (64, 1), (128, 20), (1024, 20)])
def test_planar_sgs_chain_equals_lexicographic(n, m):
    """Chebyshev-SGS on parity planes with TMA windows (k_sgs_plane) against the lexicographic
    k_sgs_tile chain: the same colour updates and combinations, so the outputs agree to rounding of
    the final k-projection coefficient (k^T y summed in another order)."""
    a = _mass_pc(n, True, m=m)
    b = _mass_pc(n, False, m=m)
    assert np.abs(a - b).max() <= 1e-14 * np.abs(b).max()


def test_planar_sgs_chain_oseen_m1():
    a = _mass_pc(64, True, oseen=True)
    b = _mass_pc(64, False, oseen=True)
    assert np.abs(a - b).max() <= 1e-14 * np.abs(b).max()
