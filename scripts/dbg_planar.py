import sys, torch, numpy as np
sys.path.insert(0, '/root/repo')
from paper_2303_10233_b200 import etq
import synth
n, m, pdl = int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3])
etq.set_option(7, pdl)
P = etq.Problem(n)
P.precond_setup(etq.PC_P2_GMG, etq.make_params(cheb_sgs_lo=0.005, cheb_sgs_steps=m))
r = torch.as_tensor(synth.random_vector(P.n_p, seed=1), device="cuda")
z = torch.zeros(P.n_p, dtype=torch.float64, device="cuda")
try:
    P.apply_mass_pc(r, z); torch.cuda.synchronize(); print("OK", n, m, pdl)
except Exception as e:
    print("FAIL", n, m, pdl, repr(e)[:100])
