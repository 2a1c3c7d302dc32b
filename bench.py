#!/usr/bin/env python
"""bench.py — headline benchmark of the Q2-Q1* Krylov hot path (BASELINE.json metric).

Workload (BASELINE.json configs[2], "c3"): Stokes lid-driven cavity on [-1,1]^2, 1024x1024
Q2-Q1* grid (N = 10,496,003 dofs), fp64, MINRES (Algorithm 1) with the P2
block-diagonal preconditioner (one Q2 GMG V-cycle + 20-step Chebyshev-SGS on the singular
M_Q with the Pi C Pi k-projection), rtol 1e-8.  A "step" is one full MINRES solve from x0 = 0
(all §8(a) rows a2-a6 of SURVEY.md; assembly a1 and the preconditioner setup are outside the
timed region and reported separately).  value = MINRES iterations / second over all ranks.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

Multi-GPU: the path is not partitioned across GPUs in this build (BASELINE.json fixes 1 GPU;
SURVEY §8(e)); --gpus N runs N independent replicas, one per rank ("replicas only",
scaling "weak"), timed as the max over ranks.  Without torchrun, --gpus N > 1 re-launches
itself under `torch.distributed.run --nproc-per-node N` (127.0.0.1 rendezvous).
--impl reference times the CPU oracle (oracle/, plain NumPy/SciPy, single thread) on a
bounded sample of the same workload (one MINRES iteration per step).
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "Stokes MINRES solve time & iters/s, Q2-Q1* 1024²; SpMV/V-cycle HBM GB/s vs peak"
UNIT = "MINRES iterations/s"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--grid-n", dest="n", type=int, default=1024,
                    help="elements per side (the driver passes no value: c3, n = 1024)")
    ap.add_argument("--rtol", type=float, default=1e-8)
    ap.add_argument("--maxit", type=int, default=5000)
    ap.add_argument("--cpu-baseline-iters", type=int, default=1,
                    help="oracle MINRES iterations timed for cpu_baseline (0 = skip)")
    ap.add_argument("--kernel-reps", type=int, default=100)
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-p3", action="store_true", help="skip the P3 (exact M_Q) time-to-solution block")
    ap.add_argument("--clock-ms", type=int, default=1000, help="nvidia-smi sampling period during the timed region")
    ap.add_argument("--host-loop", action="store_true",
                    help="MINRES as one graph launch per iteration instead of one graph with a device while node "
                         "(ncu cannot profile kernels inside graphs with conditional nodes; same iterates)")
    return ap.parse_args()


def workload_name(n):
    return (f"c3: Stokes lid-driven cavity [-1,1]^2, Q2-Q1* {n}x{n} (frame Q1+P0 pressure), "
            f"fp64, MINRES + P2 (1 Q2-GMG V-cycle, Chebyshev-3 smoother; 20-step Chebyshev-SGS "
            f"on singular M_Q with Pi C Pi), rtol 1e-8, x0 = 0")


def load_peak():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        d = json.load(open(p))
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs, torch copy)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md: 6.65 TB/s)"


# ------------------------------------------------------------------ clocks
class ClockSampler:
    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index, period_ms=1000):
        self.idx = gpu_index
        self.period = max(int(period_ms), 100)
        self.proc = None

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.idx), f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", str(self.period)], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except Exception:
            self.proc = None

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        time.sleep(0.25)
        self.proc.terminate()
        try:
            out, _ = self.proc.communicate(timeout=5)
        except Exception:
            self.proc.kill()
            out = ""
        sm, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in out.strip().splitlines():
            f = [x.strip() for x in line.split(",")]
            if len(f) < 9:
                continue
            try:
                sm.append(float(f[1])); mx = float(f[2])
            except ValueError:
                continue
            for nm, v in zip(names, f[5:9]):
                if v.lower().startswith("active"):
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": mx,
                "reasons": sorted(reasons), "samples": len(sm)}


# ------------------------------------------------------------------ oracle (CPU)
def _oracle_setup(n, a):
    from oracle import fem, mg, precond
    t0 = time.perf_counter()
    s = fem.assemble_system(n, bc="lid")
    h = mg.Hierarchy(n)
    P = precond.StokesP2(s, a, hierarchy=h)
    return s, P, time.perf_counter() - t0


def _oracle_iteration_time(s, P, iters):
    """Time `iters` MINRES iterations of the oracle; the initial preconditioner apply of
    Algorithm 1 line 3 is timed separately and excluded."""
    from oracle import krylov
    first = {}

    def Pinv(v):
        t = time.perf_counter()
        z = P(v)
        if "t" not in first:
            first["t"] = time.perf_counter() - t
        return z

    t0 = time.perf_counter()
    krylov.minres(lambda v: s.K @ v, s.b, Pinv, rtol=0.0, maxit=iters)
    total = time.perf_counter() - t0
    return max(total - first["t"], 1e-9)


def cpu_threads_guard():
    try:
        from threadpoolctl import threadpool_limits
        return threadpool_limits(limits=1)
    except Exception:
        import contextlib
        return contextlib.nullcontext()


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    n = args.n
    a = 2.0 / 400.0   # the GPU arm's automatic a at n >= 16 (reading R7: max(Lanczos, 2/m^2))
    with cpu_threads_guard():
        s, P, setup_s = _oracle_setup(n, a)
        for _ in range(args.warmup):
            _oracle_iteration_time(s, P, 1)
        times = [_oracle_iteration_time(s, P, 1) for _ in range(args.steps)]
    tot = sum(times)
    value = args.steps / tot
    sample = (f"{args.steps} steps x 1 oracle MINRES iteration on the c3 system (n={n}); oracle assembly "
              f"+ hierarchy {setup_s:.1f}s excluded; first preconditioner apply excluded")
    world = int(os.environ.get("WORLD_SIZE", "1"))
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1000 * tot / args.steps,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic", "config": {"workload": workload_name(n), "n": n, "cheb_sgs_lo": a},
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": 1, "kind": "oracle", "sample": sample},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)
    return 0


# ------------------------------------------------------------------ multi-rank timing
def aggregate(ms, its, world, device=None):
    """Max of the per-rank timed region and sum of the per-rank MINRES iterations (contract:
    value = units all ranks processed / max-over-ranks time).  Works with nccl or gloo."""
    if world == 1:
        return float(ms), float(its)
    import torch
    import torch.distributed as dist
    t_ms = torch.tensor([float(ms)], dtype=torch.float64, device=device)
    t_it = torch.tensor([float(its)], dtype=torch.float64, device=device)
    dist.all_reduce(t_ms, op=dist.ReduceOp.MAX)
    dist.all_reduce(t_it, op=dist.ReduceOp.SUM)
    return t_ms.item(), t_it.item()


# ------------------------------------------------------------------ ours (GPU)
def run_ours(args):
    import numpy as np
    import torch
    import torch.distributed as dist
    from paper_2303_10233_b200 import etq

    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)

    def barrier():
        if world > 1:
            dist.barrier()

    n = args.n
    if args.host_loop:
        etq.set_option(3, 0)
    t0 = time.perf_counter()
    P = etq.Problem(n, bc=0)
    torch.cuda.synchronize()
    assemble_s = time.perf_counter() - t0
    t0 = time.perf_counter()
    P.precond_setup(etq.PC_P2_GMG)          # automatic a (reading R7)
    torch.cuda.synchronize()
    setup_s = time.perf_counter() - t0
    a = P.get_cheb_sgs_lo()
    b = torch.zeros(P.N, dtype=torch.float64, device=dev)
    P.build_rhs(b)
    x = torch.zeros(P.N, dtype=torch.float64, device=dev)
    for _ in range(max(args.warmup, 0)):
        x.zero_()
        P.minres_solve(etq.PC_P2_GMG, b, x, rtol=args.rtol, maxit=args.maxit)

    clocks = ClockSampler(local, args.clock_ms)
    clocks.start()
    time.sleep(0.3)
    L0 = etq.launch_count()
    barrier()
    torch.cuda.synchronize()
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    e0.record()
    its = 0
    reps = []
    for _ in range(args.steps):
        x.zero_()
        rep = P.minres_solve(etq.PC_P2_GMG, b, x, rtol=args.rtol, maxit=args.maxit)
        its += rep["iterations"]
        reps.append(rep)
    e1.record()
    torch.cuda.synchronize()
    barrier()
    L1 = etq.launch_count()
    ms = e0.elapsed_time(e1)
    clk = clocks.stop()
    ms_max, its_all = aggregate(ms, its, world, dev)
    value = its_all / (ms_max / 1000.0)
    last = reps[-1]

    # ---- end to end through the public C ABI with host buffers (copies inside the timed region)
    e2e = None
    if not args.no_e2e:
        bh = b.cpu().pin_memory()
        xh = torch.zeros(P.N, dtype=torch.float64).pin_memory()
        xh.zero_()
        P.minres_solve_host(etq.PC_P2_GMG, bh, xh, rtol=args.rtol, maxit=args.maxit)   # warm
        barrier(); torch.cuda.synchronize()
        t0 = time.perf_counter()
        e_its = 0
        for _ in range(args.steps):
            xh.zero_()
            r = P.minres_solve_host(etq.PC_P2_GMG, bh, xh, rtol=args.rtol, maxit=args.maxit)
            e_its += r["iterations"]
        torch.cuda.synchronize()
        el = time.perf_counter() - t0
        barrier()
        el_max, e_all = aggregate(el, e_its, world, dev)
        e2e = {"value": e_all / el_max, "unit": UNIT, "h2d_bytes_per_step": 2 * 8 * P.N,
               "d2h_bytes_per_step": 8 * P.N,
               "note": "etq_minres_solve_host: b and x0 copied H2D, x copied D2H each step (pinned host)"}

    # ---- kernel timings (CUDA events on the library stream, etq_time_kernel)
    peak, peak_src = load_peak()
    kern = {}
    names = {0: "fused saddle SpMV [A B^T; B 0] (k_saddle)",
             10: "Chebyshev-SGS step on M_Q (k_sgs_tile)",
             11: "finest-level pre-smoothing pass, 3 fused Chebyshev steps (k_cheb_tile<0>)",
             12: "finest-level post-smoothing pass, residual + 2 fused steps (k_cheb_tile<1>)",
             2: "Q2 GMG V-cycle (both components)", 3: "Pi C Pi Chebyshev-SGS pressure apply (20 steps)",
             4: "P2 preconditioner apply (both branches concurrently)"}
    for w in (0, 10, 11, 12, 2, 3, 4):
        k_ms, k_bytes = P.time_kernel(w, args.kernel_reps)
        kern[names[w]] = {"ms": k_ms, "algorithmic_bytes": k_bytes,
                          "GB_per_s": (k_bytes / (k_ms * 1e-3) / 1e9) if k_bytes > 0 else None,
                          "frac_of_peak": (k_bytes / (k_ms * 1e-3) / 1e9 / peak) if k_bytes > 0 else None}
    # one whole MINRES iteration (the step / its iteration count): saddle apply (16 N), P2 apply (both
    # branches), the <z, v> dot inputs read by the P2 epilogues (8 N), lines 8 and 16-17 of Algorithm 1
    # (k_minres_v: q, v, v_prev in, v_prev out = 32 N; k_minres_wx: z, w, w_prev in, w_prev out = 32 N,
    # plus x in and out every other iteration = 8 N on average).  Algorithmic bytes (each kernel's
    # vectors once); the pressure vectors are L2-sized
    it_bytes = 16.0 * P.N + kern[names[4]]["algorithmic_bytes"] + 8.0 * P.N + 72.0 * P.N
    it_ms = ms / its if its else float("nan")
    kern["whole MINRES iteration (solve time / iterations)"] = {
        "ms": it_ms, "algorithmic_bytes": it_bytes, "GB_per_s": it_bytes / (it_ms * 1e-3) / 1e9,
        "frac_of_peak": it_bytes / (it_ms * 1e-3) / 1e9 / peak}
    # the saddle apply is matrix-free (class stencils): its algorithmic bytes are x in + y out; the
    # stored-operator (CSR model) bytes it replaces are reported beside them
    nnz = 192 * n * n - 336 * n + 186
    stored = 12.0 * nnz + 4.0 * (P.N + 1) + 16.0 * P.N
    s0 = kern[names[0]]
    s0["csr_model_bytes"] = stored
    s0["csr_equivalent_GB_per_s"] = stored / (s0["ms"] * 1e-3) / 1e9
    # dominant kernel of the step by the committed ncu launch-list share (profiles/r02_launches_summary.txt)
    dom_name = names[10]
    dom = kern[dom_name]
    traffic = None
    tp = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    if os.path.exists(tp):
        try:
            traffic = json.load(open(tp)).get("dram_bytes_per_launch")
        except Exception:
            traffic = None
    roofline = {"bound": "hbm", "kernel": dom_name, "achieved": dom["GB_per_s"], "peak": peak, "unit": "GB/s",
                "frac": dom["frac_of_peak"], "traffic": traffic, "peak_source": peak_src,
                "bytes_per_launch": dom["algorithmic_bytes"], "ms_per_launch": dom["ms"],
                "note": ("largest share of the step in the ncu launch list; latency-bound (9 dependent colour "
                         "steps per launch), its 4 pressure vectors (67 MB) are partly L2-resident")}

    # ---- NEXT-2: the same c3 solve with P3 = diag(V-cycle, exact M_Q through S_k) (time to solution;
    #      untimed by the headline, which stays the paper's P2 path)
    p3 = None
    if not args.no_p3:
        t0 = time.perf_counter()
        P.precond_setup(etq.PC_P3)
        torch.cuda.synchronize()
        p3_setup = time.perf_counter() - t0
        x.zero_()
        P.minres_solve(etq.PC_P3, b, x, rtol=args.rtol, maxit=args.maxit)   # warm-up (graph capture)
        s0 = P.inner_stats(0)
        rs = []
        for _ in range(3):
            x.zero_()
            rs.append(P.minres_solve(etq.PC_P3, b, x, rtol=args.rtol, maxit=args.maxit))
        s1 = P.inner_stats(0)
        r3 = rs[-1]
        ms3 = sorted(q["ms_total"] for q in rs)[1]
        y = torch.zeros_like(x)
        P.apply_saddle(x, y)
        p3 = {"preconditioner": "P3 = diag(one Q2-GMG V-cycle, exact augmented M_Q solve via S_k + Q1-GMG-PCG)",
              "iterations": r3["iterations"], "converged": bool(r3["converged"]), "solve_ms_median_of_3": ms3,
              "speedup_vs_p2_solve": (ms_max / args.steps) / ms3,
              "true_rel_res": float(torch.linalg.norm(b - y) / torch.linalg.norm(b)),
              "inner_cg_per_apply": (s1[0] - s0[0]) / max(s1[1] - s0[1], 1.0), "inner_rtol": 1e-10,
              "est_minres_gamma2": etq.est_minres(r3["delta"], r3["gamma"]), "setup_s": p3_setup}

    # ---- CPU baseline: the oracle on this host, rank 0, N = 1 only, bounded sample
    cpu = None
    if rank == 0 and world == 1 and args.cpu_baseline_iters > 0:
        with cpu_threads_guard():
            s, Po, osetup = _oracle_setup(n, a)
            t_it = _oracle_iteration_time(s, Po, args.cpu_baseline_iters)
        cpu = {"value": args.cpu_baseline_iters / t_it, "unit": UNIT, "cores": 1, "kind": "oracle",
               "sample": (f"{args.cpu_baseline_iters} oracle MINRES iteration(s) on the same c3 system "
                          f"(same a = {a:.4g}); oracle assembly+hierarchy {osetup:.1f}s and the initial "
                          f"preconditioner apply excluded; single thread")}

    if rank == 0:
        line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
                "warmup": args.warmup, "ms_per_step": ms_max / args.steps, "higher_is_better": True,
                "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
                "config": {"workload": workload_name(n), "n": n, "N": P.N, "nnz_saddle_stored": None,
                           "iterations_per_solve": last["iterations"], "solve_ms": ms_max / args.steps,
                           "rel_res": last["rel_res"], "cheb_sgs_lo": a,
                           "assemble_s": assemble_s, "precond_setup_s": setup_s,
                           "parallelism": f"{world} independent replica(s), one per GPU",
                           "l2": ("working set larger than L2: each MINRES iteration streams >= 9 N-vectors of 84 MB "
                                  "(the operators are matrix-free) - no flush needed")},
                "roofline": roofline, "kernels": kern, "cpu_baseline": cpu, "e2e": e2e, "p3_solve": p3,
                "gpu_launches": int(L1 - L0), "clocks": clk}
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()
    P.close()
    return 0


def _free_port():
    import socket
    with socket.socket(socket.AF_INET, socket.SOCK_STREAM) as sk:
        sk.bind(("127.0.0.1", 0))
        return sk.getsockname()[1]


def relaunch_under_torchrun(args):
    """`--gpus N` (N > 1) outside torchrun: re-run this command as N ranks on this node
    (one process per GPU, rendezvous on 127.0.0.1), exactly as the driver launches it."""
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr", "127.0.0.1", f"--master-port={_free_port()}", os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.call(cmd)


def main():
    args = parse()
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        return relaunch_under_torchrun(args)
    if args.impl == "reference":
        return run_reference(args)
    return run_ours(args)


if __name__ == "__main__":
    sys.exit(main())
