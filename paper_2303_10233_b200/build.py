"""Build libetq.so in-tree for sm_100a (nvcc cross-compiles without a GPU)."""
from __future__ import annotations

import os
import subprocess

HERE = os.path.dirname(os.path.abspath(__file__))
SOURCES = ["assemble.cu", "ops.cu", "solvers.cu", "oseen.cu", "sweep32.cu", "exact.cu", "picard.cu", "api.cu"]
OUT = os.path.join(HERE, "libetq.so")


def nvcc_cmd(out=OUT, extra=()):
    return ["nvcc", "-shared", "-Xcompiler", "-fPIC", "-gencode", "arch=compute_100a,code=sm_100a",
            "-lineinfo", "-O3", "-std=c++17", *extra, "-o", out] + [os.path.join(HERE, "csrc", s) for s in SOURCES]


def build(force: bool = False, verbose: bool = True) -> str:
    srcs = [os.path.join(HERE, "csrc", s) for s in SOURCES] + \
        [os.path.join(HERE, "csrc", "etq_internal.cuh"), os.path.join(HERE, "csrc", "device_common.cuh"), os.path.join(os.path.dirname(HERE), "include", "etq.h"), os.path.join(os.path.dirname(HERE), "include", "etq_debug.h")]
    if not force and os.path.exists(OUT) and os.path.getmtime(OUT) >= max(os.path.getmtime(s) for s in srcs):
        return OUT
    cmd = nvcc_cmd()
    if verbose:
        print(" ".join(cmd), flush=True)
    subprocess.run(cmd, check=True)
    return OUT


def build_variant(out, defines):
    """A/B variant of the library with extra -D flags (experiments; ETQ_LIB=<out> selects it)."""
    cmd = nvcc_cmd(out, ["-D" + d for d in defines])
    subprocess.run(cmd, check=True)
    return out


if __name__ == "__main__":
    import sys
    if len(sys.argv) > 2:          # python build.py <out.so> DEF1=.. DEF2=..
        build_variant(sys.argv[1], sys.argv[2:])
    else:
        build(force=True)
