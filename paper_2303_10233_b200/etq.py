"""Thin ctypes binding of libetq (include/etq.h): argument marshalling only.

Every step of the hot path runs in the CUDA kernels of libetq.so; this module only turns
torch tensors into device pointers, passes torch's current CUDA stream, and raises on a
negative etq_status.  There is no CPU fallback: if libetq.so is missing the import fails.
Function names mirror the C ABI (etq_<name> -> <name>).
"""
from __future__ import annotations

import ctypes as C
import os
import re

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("ETQ_LIB", os.path.join(_HERE, "libetq.so"))
HEADER = os.path.join(os.path.dirname(_HERE), "include", "etq.h")
DEBUG_HEADER = os.path.join(os.path.dirname(_HERE), "include", "etq_debug.h")

ETQ_OK, ETQ_NOT_CONVERGED = 0, 1
PC_P1_EXACT, PC_P2_GMG, PC_OSEEN_M1, PC_OSEEN_PCD1, PC_P1_ITER, PC_P3, PC_OSEEN_M2, PC_OSEEN_LSC = 0, 1, 2, 3, 4, 5, 6, 7


class EtqError(RuntimeError):
    def __init__(self, status, what):
        super().__init__(f"{what}: etq status {status} ({status_string(status)})")
        self.status = status


class Grid(C.Structure):
    _fields_ = [("n", C.c_int32), ("bc", C.c_int32), ("storage", C.c_int32), ("enriched", C.c_int32)]


class Wind(C.Structure):
    _fields_ = [("kind", C.c_int32)]


class PcParams(C.Structure):
    _fields_ = [("cheb_sgs_steps", C.c_int32), ("cheb_sgs_lo", C.c_double), ("lanczos_steps", C.c_int32),
                ("smooth_degree", C.c_int32), ("smooth_hi", C.c_double), ("smooth_lo", C.c_double),
                ("coarse_n", C.c_int32), ("mass_cheb_steps", C.c_int32), ("use_graphs", C.c_int32),
                ("inner_rtol", C.c_double), ("inner_maxit", C.c_int32), ("inner_coarse_n", C.c_int32)]


class Report(C.Structure):
    _fields_ = [("iterations", C.c_int32), ("converged", C.c_int32), ("restarts", C.c_int32),
                ("status", C.c_int32), ("rel_res", C.c_double), ("abs_res", C.c_double),
                ("ms_total", C.c_double), ("history", C.POINTER(C.c_double)), ("history_cap", C.c_int32),
                ("lanczos_delta", C.POINTER(C.c_double)), ("lanczos_gamma", C.POINTER(C.c_double)),
                ("lanczos_cap", C.c_int32)]


def load_library(path: str = LIB_PATH) -> C.CDLL:
    if not os.path.exists(path):
        raise ImportError(f"libetq.so not built at {path}; run __graft_entry__.build()")
    lib = C.CDLL(path)
    P, I32, I64, D, VP = C.c_void_p, C.c_int32, C.c_int64, C.c_double, C.c_void_p
    sig = {
        "etq_assemble": ([C.POINTER(Grid), D, C.POINTER(Wind), VP, C.POINTER(P)], I32),
        "etq_sizes": ([P, C.POINTER(I64), C.POINTER(I64), C.POINTER(I64)], I32),
        "etq_build_rhs": ([P, VP, VP], I32),
        "etq_apply_saddle": ([P, I32, VP, VP], I32),
        "etq_precond_setup": ([P, I32, C.POINTER(PcParams)], I32),
        "etq_apply_precond": ([P, I32, VP, VP], I32),
        "etq_apply_vcycle": ([P, I32, VP, VP], I32),
        "etq_apply_mass_pc": ([P, VP, VP], I32),
        "etq_apply_mass": ([P, VP, VP], I32),
        "etq_apply_mass_exact": ([P, VP, VP, C.POINTER(I32)], I32),
        "etq_inner_stats": ([P, I32, C.POINTER(D), C.POINTER(D)], I32),
        "etq_sgs_sweep": ([P, VP, VP, VP], I32),
        "etq_estimate_sgs_lo": ([P, VP, I32, C.POINTER(D)], I32),
        "etq_get_cheb_sgs_lo": ([P, C.POINTER(D)], I32),
        "etq_minres_solve": ([P, I32, VP, VP, D, I32, C.POINTER(Report)], I32),
        "etq_minres_solve_host": ([P, I32, VP, VP, D, I32, C.POINTER(Report)], I32),
        "etq_export_operator": ([P, I32, I32, C.POINTER(I64), C.POINTER(I64), VP, VP, VP], I32),
        "etq_launch_count": ([C.POINTER(I64)], I32),
        "etq_gmres_solve": ([P, I32, I32, VP, VP, D, I32, I32, C.POINTER(Report)], I32),
        "etq_two_stage_solve": ([P, VP, VP, D, D, I32, I32, C.POINTER(Report), C.POINTER(Report),
                                 C.POINTER(D)], I32),
        "etq_apply_pcd_schur": ([P, VP, VP], I32),
        "etq_set_wind": ([P, VP], I32),
        "etq_picard_solve": ([P, I32, D, D, I32, I32, VP, VP, VP, C.POINTER(D)], I32),
        "etq_est_minres": ([VP, VP, I32, C.POINTER(D)], I32),
        "etq_apply_saddle_f32": ([P, I32, VP, VP], I32),
        "etq_apply_vcycle_f32": ([P, VP, VP], I32),
        "etq_time_kernel": ([P, I32, I32, C.POINTER(D), C.POINTER(D)], I32),
        "etq_debug_set_option": ([I32, I32], I32),
        "etq_status_string": ([I32], C.c_char_p),
        "etq_destroy": ([P], None),
    }
    for name, (args, res) in sig.items():
        f = getattr(lib, name)
        f.argtypes = args
        f.restype = res
    return lib


_lib = None


def lib() -> C.CDLL:
    global _lib
    if _lib is None:
        _lib = load_library()
    return _lib


def header_functions(path: str = HEADER):
    """Names of the functions declared in include/etq.h."""
    txt = open(path).read()
    return sorted(set(re.findall(r"^\s*(?:[\w\*]+\s+)+\**(etq_\w+)\s*\(", txt, flags=re.M)))


def launch_count() -> int:
    """libetq kernel launches so far in this process (graph kernel nodes included)."""
    c = C.c_int64()
    lib().etq_launch_count(C.byref(c))
    return c.value


def est_minres(delta, gamma):
    """EST-MINRES gamma^2 from a MINRES report's delta/gamma arrays (etq_est_minres)."""
    import numpy as np
    d = np.ascontiguousarray(delta, dtype=np.float64)
    g = np.ascontiguousarray(gamma, dtype=np.float64)
    out = C.c_double()
    _check(lib().etq_est_minres(C.c_void_p(d.ctypes.data), C.c_void_p(g.ctypes.data), len(d), C.byref(out)),
           "etq_est_minres")
    return out.value


def set_option(option: int, value: int):
    """Process-wide A/B switch for tests and measurements (etq_debug_set_option, include/etq_debug.h)."""
    _check(lib().etq_debug_set_option(option, value), "etq_debug_set_option")


def status_string(s: int) -> str:
    return lib().etq_status_string(int(s)).decode()


def _check(s, what):
    if s < 0:
        raise EtqError(s, what)
    return s


def _ptr(t, n):
    """Device pointer of a contiguous float64 CUDA tensor of exactly n elements (the C ABI takes
    no lengths: a shorter tensor would be read or written out of bounds)."""
    if t is None:
        return None
    import torch
    if not (t.is_cuda and t.dtype == torch.float64 and t.is_contiguous()):
        raise ValueError("expected a contiguous float64 CUDA tensor")
    if t.numel() != n:
        raise ValueError(f"expected {n} elements, got {t.numel()}")
    return C.c_void_p(t.data_ptr())


def _fptr(t, n):
    import torch
    if not (t.is_cuda and t.dtype == torch.float32 and t.is_contiguous()):
        raise ValueError("expected a contiguous float32 CUDA tensor")
    if t.numel() != n:
        raise ValueError(f"expected {n} elements, got {t.numel()}")
    return C.c_void_p(t.data_ptr())


def _hptr(a, n):
    """Host pointer of a contiguous float64 CPU tensor or numpy array of exactly n elements."""
    import numpy as np
    if hasattr(a, "data_ptr"):
        import torch
        if a.is_cuda or a.dtype != torch.float64 or not a.is_contiguous():
            raise ValueError("expected a contiguous float64 CPU tensor")
        size, ptr = a.numel(), a.data_ptr()
    else:
        if not (isinstance(a, np.ndarray) and a.dtype == np.float64 and a.flags["C_CONTIGUOUS"]):
            raise ValueError("expected a C-contiguous float64 numpy array")
        size, ptr = a.size, a.ctypes.data
    if size != n:
        raise ValueError(f"expected {n} elements, got {size}")
    return C.c_void_p(ptr)


def _stream():
    import torch
    return C.c_void_p(torch.cuda.current_stream().cuda_stream)


def make_params(**kw) -> PcParams:
    p = PcParams()
    p.use_graphs = 1
    for k, v in kw.items():
        setattr(p, k, v)
    return p


class Problem:
    """Owns an etq_problem (device matrices and workspaces)."""

    def __init__(self, n: int, bc: int = 0, viscosity: float = 1.0, wind: int = 0, storage: int = 0,
                 enriched: bool = True):
        """enriched=False: plain Taylor-Hood Q2-Q1 on the same mesh (etq_grid.enriched = 0)."""
        h = C.c_void_p()
        g = Grid(n, bc, storage, 1 if enriched else 0)
        w = Wind(wind)
        _check(lib().etq_assemble(C.byref(g), viscosity, C.byref(w), _stream(), C.byref(h)), "etq_assemble")
        self.h = h
        self.n = n
        n_u, n_k, n_0 = C.c_int64(), C.c_int64(), C.c_int64()
        _check(lib().etq_sizes(h, C.byref(n_u), C.byref(n_k), C.byref(n_0)), "etq_sizes")
        self.n_u, self.n_k, self.n_0 = n_u.value, n_k.value, n_0.value
        self.n_p = self.n_k + self.n_0
        self.N = self.n_u + self.n_p
        self.nq = self.n_u // 2

    def close(self):
        if self.h:
            lib().etq_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # ---- C-ABI mirrors
    def build_rhs(self, b, f_nodal=None):
        _check(lib().etq_build_rhs(self.h, _ptr(f_nodal, self.n_u), _ptr(b, self.N)), "etq_build_rhs")
        return b

    def apply_saddle(self, x, y, reduced=False):
        _check(lib().etq_apply_saddle(self.h, int(reduced), _ptr(x, self.N), _ptr(y, self.N)), "etq_apply_saddle")
        return y

    def precond_setup(self, kind, params: PcParams | None = None):
        _check(lib().etq_precond_setup(self.h, kind, C.byref(params) if params is not None else None),
               "etq_precond_setup")

    def apply_precond(self, kind, r, z):
        _check(lib().etq_apply_precond(self.h, kind, _ptr(r, self.N), _ptr(z, self.N)), "etq_apply_precond")
        return z

    def apply_vcycle(self, kind, r_u, z_u):
        _check(lib().etq_apply_vcycle(self.h, kind, _ptr(r_u, self.n_u), _ptr(z_u, self.n_u)), "etq_apply_vcycle")
        return z_u

    def apply_mass_pc(self, r_p, z_p):
        _check(lib().etq_apply_mass_pc(self.h, _ptr(r_p, self.n_p), _ptr(z_p, self.n_p)), "etq_apply_mass_pc")
        return z_p

    def apply_mass_exact(self, r_p, z_p):
        """Exact augmented M_Q solve through S_k (P3 / P1_ITER set up); returns the CG iterations."""
        it = C.c_int32()
        _check(lib().etq_apply_mass_exact(self.h, _ptr(r_p, self.n_p), _ptr(z_p, self.n_p), C.byref(it)), "etq_apply_mass_exact")
        return it.value

    def inner_stats(self, which=0):
        """(total inner CG iterations, solves) since setup; which 0 = M_Q, 1 = velocity."""
        it, calls = C.c_double(), C.c_double()
        _check(lib().etq_inner_stats(self.h, which, C.byref(it), C.byref(calls)), "etq_inner_stats")
        return it.value, calls.value

    def apply_mass(self, x_p, y_p):
        _check(lib().etq_apply_mass(self.h, _ptr(x_p, self.n_p), _ptr(y_p, self.n_p)), "etq_apply_mass")
        return y_p

    def sgs_sweep(self, r_p, y_p, z_p):
        _check(lib().etq_sgs_sweep(self.h, _ptr(r_p, self.n_p), _ptr(y_p, self.n_p), _ptr(z_p, self.n_p)), "etq_sgs_sweep")
        return z_p

    def estimate_sgs_lo(self, v0, steps):
        lam = C.c_double()
        _check(lib().etq_estimate_sgs_lo(self.h, _ptr(v0, self.n_p), steps, C.byref(lam)), "etq_estimate_sgs_lo")
        return lam.value

    def get_cheb_sgs_lo(self):
        a = C.c_double()
        _check(lib().etq_get_cheb_sgs_lo(self.h, C.byref(a)), "etq_get_cheb_sgs_lo")
        return a.value

    def time_kernel(self, which, reps=20):
        """(ms per launch, algorithmic bytes per launch) of hot kernel `which` (etq_time_kernel)."""
        ms, by = C.c_double(), C.c_double()
        _check(lib().etq_time_kernel(self.h, which, reps, C.byref(ms), C.byref(by)), "etq_time_kernel")
        return ms.value, by.value

    def _report(self, cap):
        import numpy as np
        rep = Report()
        hist = np.zeros(cap); dl = np.zeros(cap); gm = np.zeros(cap)
        rep.history = hist.ctypes.data_as(C.POINTER(C.c_double)); rep.history_cap = cap
        rep.lanczos_delta = dl.ctypes.data_as(C.POINTER(C.c_double))
        rep.lanczos_gamma = gm.ctypes.data_as(C.POINTER(C.c_double)); rep.lanczos_cap = cap
        return rep, hist, dl, gm

    @staticmethod
    def _report_dict(rep, hist, dl, gm, status):
        k = rep.iterations
        return {"status": status, "iterations": k, "converged": bool(rep.converged), "rel_res": rep.rel_res,
                "abs_res": rep.abs_res, "ms_total": rep.ms_total, "history": hist[:k].copy(),
                "delta": dl[:k].copy(), "gamma": gm[:k].copy()}

    def minres_solve(self, kind, b, x, rtol=1e-8, maxit=1000):
        rep, hist, dl, gm = self._report(maxit + 1)
        s = _check(lib().etq_minres_solve(self.h, kind, _ptr(b, self.N), _ptr(x, self.N), rtol, maxit,
                                               C.byref(rep)), "etq_minres_solve")
        return self._report_dict(rep, hist, dl, gm, s)

    def minres_solve_host(self, kind, b_host, x_host, rtol=1e-8, maxit=1000):
        """b_host, x_host: contiguous float64 CPU tensors or numpy arrays (x in/out)."""
        rep, hist, dl, gm = self._report(maxit + 1)
        pb = _hptr(b_host, self.N)
        px = _hptr(x_host, self.N)
        s = _check(lib().etq_minres_solve_host(self.h, kind, pb, px, rtol, maxit, C.byref(rep)),
                   "etq_minres_solve_host")
        return self._report_dict(rep, hist, dl, gm, s)

    def apply_saddle_f32(self, x, y, reduced=False):
        _check(lib().etq_apply_saddle_f32(self.h, int(reduced), _fptr(x, self.N), _fptr(y, self.N)), "etq_apply_saddle_f32")
        return y

    def apply_vcycle_f32(self, r_u, z_u):
        _check(lib().etq_apply_vcycle_f32(self.h, _fptr(r_u, self.n_u), _fptr(z_u, self.n_u)), "etq_apply_vcycle_f32")
        return z_u

    def apply_pcd_schur(self, r_p1, z_p1):
        _check(lib().etq_apply_pcd_schur(self.h, _ptr(r_p1, self.n_k), _ptr(z_p1, self.n_k)), "etq_apply_pcd_schur")
        return z_p1

    def gmres_solve(self, kind, b, x, rtol=1e-6, restart=50, maxit=1000, reduced=False):
        rep, hist, dl, gm = self._report(maxit + 2)
        s = _check(lib().etq_gmres_solve(self.h, int(reduced), kind, _ptr(b, self.N), _ptr(x, self.N), rtol, restart, maxit,
                                         C.byref(rep)), "etq_gmres_solve")
        d = self._report_dict(rep, hist, dl, gm, s)
        d["history"] = hist[:rep.iterations + 1].copy()
        d["restarts"] = rep.restarts
        return d

    def two_stage_solve(self, b, x, eta=1e-6, c=10.0, restart=50, maxit=2000):
        r1, h1, d1, g1 = self._report(maxit + 2)
        r2, h2, d2, g2 = self._report(maxit + 2)
        bound = (C.c_double * 2)()
        s = _check(lib().etq_two_stage_solve(self.h, _ptr(b, self.N), _ptr(x, self.N), eta, c, restart, maxit, C.byref(r1),
                                             C.byref(r2), bound), "etq_two_stage_solve")
        st1 = self._report_dict(r1, h1, d1, g1, s); st1["history"] = h1[:r1.iterations + 1].copy()
        st2 = self._report_dict(r2, h2, d2, g2, s); st2["history"] = h2[:r2.iterations + 1].copy()
        return {"status": s, "step1": st1, "step2": st2, "zstar": bound[0], "bound": bound[1]}

    def set_wind(self, w):
        """Nodal Q2 wind [w_x | w_y] (device tensor, length n_u) of a wind-kind-2 problem."""
        _check(lib().etq_set_wind(self.h, _ptr(w, self.n_u)), "etq_set_wind")

    def picard_solve(self, x, steps=5, eta=1e-6, c=10.0, restart=50, maxit=2000):
        """Picard loop (etq_picard_solve); x receives the last iterate."""
        import numpy as np
        its = np.zeros(2 * (steps + 1), dtype=np.int32)
        res = np.zeros(steps + 1)
        ms = C.c_double()
        s = _check(lib().etq_picard_solve(self.h, steps, eta, c, restart, maxit, _ptr(x, self.N),
                                          C.c_void_p(its.ctypes.data), C.c_void_p(res.ctypes.data),
                                          C.byref(ms)), "etq_picard_solve")
        return {"status": s, "step1_its": its[0::2].copy(), "step2_its": its[1::2].copy(), "rel_res": res,
                "ms_total": ms.value}

    def export_operator(self, which, level=0):
        """Assembled operator as a scipy CSR matrix (host copy; tests only)."""
        import numpy as np
        import scipy.sparse as sp
        nr, nz = C.c_int64(), C.c_int64()
        _check(lib().etq_export_operator(self.h, which, level, C.byref(nr), C.byref(nz), None, None, None),
               "etq_export_operator")
        rp = np.zeros(nr.value + 1, dtype=np.int64)
        col = np.zeros(max(nz.value, 1), dtype=np.int32)
        val = np.zeros(max(nz.value, 1))
        _check(lib().etq_export_operator(self.h, which, level, C.byref(nr), C.byref(nz),
                                         C.c_void_p(rp.ctypes.data), C.c_void_p(col.ctypes.data),
                                         C.c_void_p(val.ctypes.data)), "etq_export_operator")
        ncol = {0: nr.value, 1: self.n_u, 2: self.n_p, 3: nr.value, 4: nr.value, 5: nr.value, 6: nr.value}[which]
        return sp.csr_matrix((val[:nz.value], col[:nz.value], rp), shape=(nr.value, ncol))
