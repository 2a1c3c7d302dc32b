"""Chebyshev-SGS step time against the tile count (wave quantisation): which = 10 at n = 256 ... 2048."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2303_10233_b200 import etq
for n in (256, 512, 1024, 2048):
    P = etq.Problem(n)
    P.precond_setup(etq.PC_P2_GMG, etq.make_params(cheb_sgs_lo=0.005))
    ms, by = P.time_kernel(10, 200)
    ms3, by3 = P.time_kernel(3, 50)
    tx = (n + 1 + 49) // 50
    t32 = tx * ((n + 1 + 25) // 26)
    print(f"n={n:5d} tiles32={t32:5d} waves(592)={t32/592:5.2f} step={ms*1e3:7.2f}us  {by/ms/1e6:7.0f} GB/s  PiCPi={ms3*1e3:7.1f}us", flush=True)
    P.close()
