"""Summarise an ncu launch list (--metrics gpu__time_duration.sum --csv) into per-kernel shares.

  python scripts/launch_summary.py gpurun_out/launches.csv [header lines...] > profiles/rNN_launches_summary.txt
"""
import csv
import re
import sys
from collections import OrderedDict


def main():
    path = sys.argv[1]
    rows = [l for l in open(path) if l.startswith('"')]
    rd = csv.DictReader(rows)
    agg = OrderedDict()
    for r in rd:
        if r.get("Metric Name") != "gpu__time_duration.sum":
            continue
        name = r["Kernel Name"]
        name = re.sub(r"\(.*", "", name).replace("<unnamed>::", "").replace("void ", "")
        m = re.search(r"<(\d+)>", r["Kernel Name"])
        if m and "<" not in name:
            name += f"<{m.group(1)}>"
        us = float(r["Metric Value"]) * (1e-3 if r["Metric Unit"] == "ns" else 1.0 if r["Metric Unit"] == "us" else 1e3)
        a = agg.setdefault(name, [0, 0.0])
        a[0] += 1
        a[1] += us
    tot = sum(v[1] for v in agg.values())
    for h in sys.argv[2:]:
        print("# " + h)
    print(f"{'kernel':28s} {'launches':>9s} {'total_us':>12s} {'share':>7s} {'avg_us':>9s}")
    for k, (c, us) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
        print(f"{k:28s} {c:9d} {us:12.1f} {100 * us / tot:6.1f}% {us / c:9.2f}")


if __name__ == "__main__":
    main()
