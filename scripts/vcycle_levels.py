"""V-cycle time for n = 2 ... 1024 (each level's incremental cost = V(n) - V(n/2))."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2303_10233_b200 import etq
prev = 0.0
n = 4
while n <= 1024:
    P = etq.Problem(n)
    P.precond_setup(etq.PC_P2_GMG, etq.make_params(cheb_sgs_lo=0.005))
    ms, by = P.time_kernel(2, 50)
    msp, _ = P.time_kernel(3, 50)
    msa, _ = P.time_kernel(0, 50)
    print(f"n={n:5d} vcycle={ms*1e3:8.1f}us  incr={(ms-prev)*1e3:8.1f}us  bytes={by/1e6:9.1f}MB  pressure={msp*1e3:7.1f}us  saddle={msa*1e3:7.1f}us", flush=True)
    prev = ms
    P.close()
    n *= 2
