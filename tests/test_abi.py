"""CPU-side checks of the C-ABI library: it loads without a GPU and exports every function
that include/etq.h declares; the Python binding mirrors the same names."""
import os

import pytest

from paper_2303_10233_b200 import etq


def test_library_exports_every_header_symbol():
    lib = etq.lib()
    names = etq.header_functions()
    assert len(names) >= 15
    missing = [n for n in names if not hasattr(lib, n)]
    assert not missing, missing


def test_binding_mirrors_header_names():
    methods = set(dir(etq.Problem)) | {"assemble", "status_string", "destroy", "sizes", "launch_count"}
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
