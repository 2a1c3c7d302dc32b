"""Summarise the committed full ncu captures into profiles/ncu_traffic.json (unit-aware; bench.py
reads dram_bytes_per_launch of the dominant kernel as roofline.traffic).

  python scripts/ncu_traffic.py
"""
import csv
import json
import os
import subprocess

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
U = {'byte': 1, 'Kbyte': 1e3, 'Mbyte': 1e6, 'Gbyte': 1e9}


def raw(f):
    out = subprocess.run(['ncu', '-i', f, '--page', 'raw', '--csv'], capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    return {k: (v, u) for k, u, v in zip(rows[0], rows[1], rows[2])}


def pick(d):
    def g(k):
        v, u = d.get(k, ('', ''))
        if v in (None, ''):
            return None
        return float(v.replace(',', '')) * U.get(u, 1.0)
    return {"duration_us_under_ncu": g('gpu__time_duration.sum'),
            "dram_read_bytes": g('dram__bytes_read.sum'), "dram_write_bytes": g('dram__bytes_write.sum'),
            "lts_sector_hit_rate_pct": g('lts__t_sector_hit_rate.pct'),
            "warps_active_pct": g('sm__warps_active.avg.pct_of_peak_sustained_active'),
            "issue_active_pct": g('smsp__issue_active.avg.pct_of_peak_sustained_active'),
            "smem_wavefronts_pct": g('l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed'),
            "fp64_pipe_active_pct": g('sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active'),
            "warp_instructions": g('smsp__inst_executed.sum'), "registers": g('launch__registers_per_thread')}


def main():
    nd = os.path.join(ROOT, 'profiles', 'ncu')
    s = pick(raw(os.path.join(nd, 'r02b_k_sgs_tile.ncu-rep')))
    c = pick(raw(os.path.join(nd, 'r02b_k_cheb_tile3_pre.ncu-rep')))
    t = pick(raw(os.path.join(nd, 'r02b_k_saddle_tile.ncu-rep')))
    d = {"kernel": "k_sgs_tile<32, 2> (one Chebyshev-SGS step, n = 1024, 64 x 32 windows, 50 x 26 tiles, 840 CTAs; end of round 2)",
         "command": "ncu --set full --clock-control none --import-source on -k regex:k_sgs_tile -s 2 -c 1 "
                    "python scripts/profile_kernel.py --n 1024 --which 10 --reps 2",
         "dram_bytes_per_launch": s["dram_read_bytes"] + s["dram_write_bytes"],
         "algorithmic_bytes_per_launch": 67174432, **s,
         "note": "ncu replays with flushed caches: DRAM bytes are cold-cache; inside the solve the 4 pressure "
                 "vectors (67 MB) are partly L2-resident",
         "other": {"k_cheb_tile3<0> (finest pre pass)": {**c, "algorithmic_bytes_per_launch": 201523248},
                   "k_saddle_tile (matrix-free saddle apply)": {**t, "algorithmic_bytes_per_launch": 167936048}}}
    json.dump(d, open(os.path.join(ROOT, 'profiles', 'ncu_traffic.json'), 'w'), indent=1)
    print(json.dumps(d, indent=1))


if __name__ == "__main__":
    main()
