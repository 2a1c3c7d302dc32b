"""A/B of a debug option on the kernel timers: python scripts/ab_kernels.py --option 18 --values 0,1 [--which 11,12,2,4]"""
import argparse, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2303_10233_b200 import etq
ap = argparse.ArgumentParser()
ap.add_argument("--option", type=int, required=True)
ap.add_argument("--values", default="0,1")
ap.add_argument("--which", default="11,12,2,4")
ap.add_argument("--n", type=int, default=1024)
ap.add_argument("--rounds", type=int, default=2)
args = ap.parse_args()
for r in range(args.rounds):
    for v in [int(x) for x in args.values.split(",")]:
        etq.set_option(args.option, v)
        P = etq.Problem(args.n)
        P.precond_setup(etq.PC_P2_GMG, etq.make_params(cheb_sgs_lo=0.005))
        row = {w: round(P.time_kernel(int(w), 200)[0] * 1e3, 2) for w in args.which.split(",")}
        print(f"option {args.option} = {v}: us {row}", flush=True)
        P.close()
