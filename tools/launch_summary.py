"""Summarise an `ncu --metrics gpu__time_duration.sum --csv` launch list.

usage: python tools/launch_summary.py launches.csv [renders]
Prints total device time per kernel name (per render when `renders` is given).
"""
import csv
import sys
from collections import defaultdict


def main(path, renders=1):
    rows = []
    with open(path) as f:
        lines = [l for l in f if l.startswith('"')]
    for r in csv.DictReader(lines):
        if r.get("Metric Name") != "gpu__time_duration.sum":
            continue
        v = float(r["Metric Value"].replace(",", ""))
        unit = r.get("Metric Unit", "nsecond")
        scale = {"nsecond": 1e-6, "usecond": 1e-3, "msecond": 1.0, "second": 1e3}.get(unit, 1e-6)
        rows.append((r["Kernel Name"], v * scale))
    agg = defaultdict(lambda: [0.0, 0])
    for name, ms in rows:
        short = name.split("(")[0].replace("rsg::", "")
        agg[short][0] += ms
        agg[short][1] += 1
    tot = sum(a[0] for a in agg.values())
    print(f"total {tot / renders:.2f} ms per render ({len(rows)} launches, {renders} renders)")
    for name, (ms, n) in sorted(agg.items(), key=lambda kv: -kv[1][0]):
        print(f"  {ms / renders:8.3f} ms  {100 * ms / tot:5.1f}%  n={n:5d}  {name[:60]}")


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 1)
