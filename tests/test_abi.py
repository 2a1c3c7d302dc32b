"""CPU-side checks of the C-ABI library: it loads without a GPU and exports every function
that include/etq.h declares; the Python binding mirrors the same names."""
import os

import pytest

from paper_2303_10233_b200 import etq


def test_library_exports_every_header_symbol():
    lib = etq.lib()
    names = etq.header_functions() + etq.header_functions(etq.DEBUG_HEADER)
    assert len(names) >= 15
    missing = [n for n in names if not hasattr(lib, n)]
    assert not missing, missing


def test_ab_switches_are_not_in_the_product_header():
    assert "etq_set_option" not in etq.header_functions()
    assert etq.header_functions(etq.DEBUG_HEADER) == ["etq_debug_set_option"]


def test_binding_mirrors_header_names():
    methods = set(dir(etq.Problem)) | {"assemble", "status_string", "destroy", "sizes", "launch_count", "est_minres",
                                        "set_option"}
    assert callable(etq.set_option)
    for n in etq.header_functions():
        short = n[len("etq_"):]
        assert short in methods or short == "status_string", short


def test_status_strings():
    assert etq.status_string(0) == "ok"
    assert "indefinite" in etq.status_string(-4)


def test_product_path_never_imports_oracle():
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    pkg = os.path.join(root, "paper_2303_10233_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".h")):
                txt = open(os.path.join(dirpath, f)).read()
                assert "import oracle" not in txt and "from oracle" not in txt, f


def test_est_minres_host_matches_oracle():
    """etq_est_minres is host-side: check it against oracle.krylov.est_minres_gamma2 on CPU."""
    import numpy as np
    from oracle import krylov
    rng = np.random.default_rng(3)
    for k in (1, 2, 5, 30):
        d = rng.standard_normal(k)
        g = np.abs(rng.standard_normal(k)) + 0.1          # gamma_2 .. gamma_{k+1}
        ref = krylov.est_minres_gamma2(d, np.concatenate([[1.0], g]))
        got = etq.est_minres(d, g)
        if np.isnan(ref):
            assert np.isnan(got)
        else:
            assert abs(got - ref) <= 1e-10 * max(1.0, abs(ref))


def test_nvtx_ranges_compiled_in():
    """Solver phases and kernel families carry NVTX ranges (SURVEY §5 tracing)."""
    blob = open(etq.LIB_PATH, "rb").read()
    for name in (b"minres (Algorithm 1)", b"V-cycle", b"Pi C Pi (Chebyshev-SGS)", b"saddle apply", b"gmres (CGS2)",
                 b"two-stage PCD", b"exact M_Q solve", b"etq_precond_setup"):
        assert name in blob, name
