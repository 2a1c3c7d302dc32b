"""Locate k_cheb_tile3 vs k_cheb_tile2 V-cycle differences (debug)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np
from tests.test_gpu_tile import _vcycle

for n, bc in [(128, 0), (256, 1), (512, 0), (1024, 0)]:
    a = _vcycle(n, True, bc, tile2=1, tile3=0)
    b = _vcycle(n, True, bc, tile2=1, tile3=1)
    m = 2 * n + 1
    d = np.nonzero(a != b)[0]
    print(n, bc, "ndiff", d.size, "maxrel", np.abs(a - b).max() / np.abs(a).max(), flush=True)
    if d.size:
        c = d // (m * m); q = d % (m * m)
        print("   first", [(int(cc), int(qq % m), int(qq // m)) for cc, qq in zip(c[:16], q[:16])], flush=True)
        print("   i hist", np.bincount((q % m) % 56, minlength=56).tolist(), flush=True)
        print("   j hist", np.bincount((q // m) % 56, minlength=56).tolist(), flush=True)
