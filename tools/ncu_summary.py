"""Key metrics of an `ncu --set full` report, one block per kernel launch.

usage: python tools/ncu_summary.py report.ncu-rep|report_raw.csv [...]
(a `_raw.csv` is `ncu -i report.ncu-rep --page raw --csv`, exported on the GPU box)
"""
import csv
import io
import subprocess
import sys

KEYS = [
    ("gpu__time_duration.sum", "duration"),
    ("dram__bytes_read.sum", "dram read"),
    ("dram__bytes_write.sum", "dram write"),
    ("dram__throughput.avg.pct_of_peak_sustained_elapsed", "DRAM throughput %"),
    ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "SM throughput %"),
    ("l1tex__throughput.avg.pct_of_peak_sustained_active", "L1/smem throughput %"),
    ("l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", "smem wavefronts"),
    ("l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "smem bank conflicts"),
    ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue active %"),
    ("sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active", "FMA pipe %"),
    ("sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active", "LSU pipe %"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "achieved occupancy %"),
    ("launch__registers_per_thread", "registers/thread"),
    ("launch__block_size", "block size"),
    ("launch__grid_size", "grid size"),
]


def main(path):
    if path.endswith(".csv"):
        with open(path) as f:
            raw = f.read()
    else:
        raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units, data = rows[0], rows[1], rows[2:]
    ix = {h: i for i, h in enumerate(hdr)}
    for r in data:
        print("--", r[ix["Kernel Name"]][:100])
        for k, label in KEYS:
            if k in ix:
                print(f"    {label:24s} {r[ix[k]]} {units[ix[k]]}")
        stalls = sorted(((float(r[i].replace(",", "") or 0), h) for h, i in ix.items()
                         if h.startswith("smsp__pcsamp_warps_issue_stalled") and not h.endswith("not_issued")),
                        reverse=True)
        tot = sum(v for v, _ in stalls) or 1.0
        print("    stall samples: " + ", ".join(f"{h[33:]} {100 * v / tot:.0f}%" for v, h in stalls[:6]))


if __name__ == "__main__":
    for p in sys.argv[1:]:
        main(p)
