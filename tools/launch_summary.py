"""Summarise an `ncu --metrics ... --csv` launch list (gpu__time_duration.sum and,
when captured, dram__bytes_read.sum / dram__bytes_write.sum).

usage: python tools/launch_summary.py launches.csv [renders]
Prints device time (and DRAM traffic) per kernel name, per render when `renders` is given.
"""
import csv
import sys
from collections import defaultdict

SCALE = {"nsecond": 1e-6, "ns": 1e-6, "usecond": 1e-3, "us": 1e-3, "msecond": 1.0, "ms": 1.0, "second": 1e3,
         "byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}


def main(path, renders=1):
    with open(path) as f:
        lines = [l for l in f if l.startswith('"')]
    per = defaultdict(lambda: defaultdict(float))  # (launch id, name) -> metric -> value
    for r in csv.DictReader(lines):
        v = float(r["Metric Value"].replace(",", "")) * SCALE.get(r.get("Metric Unit", ""), 1.0)
        per[(r["ID"], r["Kernel Name"])][r["Metric Name"]] = v
    agg = defaultdict(lambda: [0.0, 0.0, 0])
    for (_, name), m in per.items():
        short = name.split("(")[0].replace("rsg::", "").replace("void ", "")
        a = agg[short]
        a[0] += m.get("gpu__time_duration.sum", 0.0)
        a[1] += m.get("dram__bytes_read.sum", 0.0) + m.get("dram__bytes_write.sum", 0.0)
        a[2] += 1
    tot = sum(a[0] for a in agg.values())
    print(f"total {tot / renders:.2f} ms per render ({len(per)} launches, {renders} renders)")
    for name, (ms, by, n) in sorted(agg.items(), key=lambda kv: -kv[1][0]):
        extra = f"  dram {by / renders / 1e9:7.3f} GB ({by / (ms * 1e-3) / 1e12 if ms else 0:.2f} TB/s)" if by else ""
        print(f"  {ms / renders:8.3f} ms  {100 * ms / tot:5.1f}%  n={n:5d}  {name[:52]:52s}{extra}")


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 1)
