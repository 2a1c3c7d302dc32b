#!/usr/bin/env python
"""Summarise an ncu --set full report: duration, warps/issue active, stall reasons, DRAM bytes,
instruction mix by opcode and by code region (SASS address chunks).
  python scripts/ncu_summary.py report.ncu-rep [--regions]"""
import csv, collections, io, re, subprocess, sys


def ncu_csv(rep, *args):
    out = subprocess.run(["ncu", "-i", rep, "--csv", *args], capture_output=True, text=True).stdout
    return list(csv.reader(io.StringIO(out)))


def main():
    rep = sys.argv[1]
    rows = ncu_csv(rep, "--page", "raw")
    d = dict(zip(rows[0], rows[2]))
    keys = ["gpu__time_duration.sum", "launch__registers_per_thread", "sm__warps_active.avg.pct_of_peak_sustained_active",
            "smsp__issue_active.avg.pct_of_peak_sustained_active", "smsp__inst_executed.sum", "dram__bytes_read.sum",
            "dram__bytes_write.sum", "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum",
            "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active", "launch__grid_size"]
    for k in keys:
        if k in d:
            print(f"{k:60s} {d[k]}")
    st = []
    for k, v in d.items():
        if k.startswith("smsp__average_warps_issue_stalled_") and k.endswith("_per_issue_active.ratio"):
            try:
                st.append((float(v), k[len("smsp__average_warps_issue_stalled_"):-len("_per_issue_active.ratio")]))
            except ValueError:
                pass
    print("stalls per issue:", ", ".join(f"{k} {v:.2f}" for v, k in sorted(st, reverse=True)[:8]))
    src = ncu_csv(rep, "--page", "source", "--print-source", "sass")
    hdr = src[1]
    ie = hdr.index("Instructions Executed")
    ins = []
    for r in src[2:]:
        t = r[1].strip()
        m = re.match(r"(@!?U?P\w+\s+)?([A-Z0-9_]+)", t)
        ins.append((int(r[0], 16), m.group(2) if m else "?", int(r[ie] or 0)))
    tot = sum(i[2] for i in ins)
    cnt = collections.Counter()
    for i in ins:
        cnt[i[1]] += i[2]
    print("warp instructions", tot, " top:", ", ".join(f"{k} {v / tot:.3f}" for k, v in cnt.most_common(12)))
    if "--regions" in sys.argv:
        base = ins[0][0]
        for c in range(0, len(ins), 128):
            seg = ins[c:c + 128]
            s = sum(i[2] for i in seg)
            if s / max(tot, 1) < 0.01:
                continue
            cc = collections.Counter()
            for i in seg:
                cc[i[1]] += i[2]
            print(f"{seg[0][0] - base:6x} {s / tot:6.3f} " + ", ".join(f"{k}:{v * 100 // s}" for k, v in cc.most_common(6)))


if __name__ == "__main__":
    main()
