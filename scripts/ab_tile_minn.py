"""V-cycle / P2-apply device time at n = 1024 for several etq_set_option(1) thresholds."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
from paper_2303_10233_b200 import etq  # noqa: E402
out = {}
for mn in (64, 128, 256, 512, 1024, 100000):
    etq.set_option(1, mn)
    P = etq.Problem(1024)
    P.precond_setup(etq.PC_P2_GMG, etq.make_params(cheb_sgs_lo=0.005))
    out[mn] = {"vcycle_ms": P.time_kernel(2, 30)[0], "p2_apply_ms": P.time_kernel(4, 30)[0]}
    P.close()
print(json.dumps(out, indent=1))
