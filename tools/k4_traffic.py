"""K4 (OLA filter) device time and DRAM traffic per render from an ncu launch list
(gpu__time_duration.sum, dram__bytes_read.sum, dram__bytes_write.sum), as JSON for
bench.py's roofline `traffic` field.

usage: python tools/k4_traffic.py launches.csv renders source-note [utterances] > profiles/k4_traffic.json
"""
import csv
import json
import re
import sys
from collections import defaultdict

from launch_summary import SCALE

K4 = re.compile(r"ola_small_kernel|ola_ipc_kernel|ola_ip_kernel|ola2_kernel|large_(rows|cols|ola)")


def main(path, renders, source, utts=4096):
    with open(path) as f:
        lines = [l for l in f if l.startswith('"')]
    per = defaultdict(dict)
    for r in csv.DictReader(lines):
        if K4.search(r["Kernel Name"]):
            per[r["ID"]][r["Metric Name"]] = float(r["Metric Value"].replace(",", "")) * SCALE.get(r.get("Metric Unit", ""), 1.0)
    ms = sum(m.get("gpu__time_duration.sum", 0.0) for m in per.values())
    by = sum(m.get("dram__bytes_read.sum", 0.0) + m.get("dram__bytes_write.sum", 0.0) for m in per.values())
    print(json.dumps({
        "workload": "config4", "utterances_per_rank": utts,
        "kernel": "K4 (ola_ipc_kernel / ola_ip_kernel / ola_small_kernel / ola2_kernel / four-step stages), all launches of one config-4 render",
        "dram_bytes_per_render": by / renders,
        "device_ms_per_render": ms / renders,
        "launches_per_render": len(per) / renders,
        "source": source,
        "note": "DRAM traffic includes writing the reverberant pair signals y_ij (25.6 GB/render), an intermediate "
                "the algorithmic byte count (inputs + RIR taps + mixed outputs) does not include",
    }, indent=1))


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]), sys.argv[3], int(sys.argv[4]) if len(sys.argv) > 4 else 4096)
