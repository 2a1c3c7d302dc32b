"""Run one hot kernel of libetq repeatedly (for ncu captures): python scripts/profile_kernel.py --n 1024 --which 3"""
import argparse, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2303_10233_b200 import etq

ap = argparse.ArgumentParser()
ap.add_argument("--n", type=int, default=1024)
ap.add_argument("--which", type=int, default=1)
ap.add_argument("--reps", type=int, default=3)
args = ap.parse_args()
P = etq.Problem(args.n)
P.precond_setup(etq.PC_P2_GMG, etq.make_params(cheb_sgs_lo=0.005))
ms, by = P.time_kernel(args.which, args.reps)
print(f"which={args.which} n={args.n} ms={ms:.4f} bytes={by:.4g} GB/s={by/ms/1e6 if by else 0:.1f}")
