"""paper_2303_10233_b200 — B200-native (sm_100a) Krylov hot path for enriched Taylor-Hood
Q2-Q1* saddle-point systems (arXiv 2303.10233).

The product is libetq.so (CUDA kernels + C ABI, include/etq.h); `etq` is its ctypes binding.
"""
from . import etq  # noqa: F401
from .etq import Problem, PC_P1_EXACT, PC_P2_GMG, PC_OSEEN_M1, PC_OSEEN_PCD1, EtqError  # noqa: F401
