"""Generates tests/golden/golden.npz from the REFERENCE itself (oracle/_ref,
compiled from /root/reference by oracle/Makefile).  Run in the dev container:
    python tests/golden/make_golden.py
"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)

import oracle  # noqa: E402
from tests.golden import cases  # noqa: E402


def main():
    R = oracle.reference()
    out = {}
    for i, c in enumerate(cases.RIR_CASES):
        h = R.synthesize_rir(c["room"], c["r"], c["K"], c["src"], c["mic"], max_taps=c["max_taps"])
        out[f"rir_{i}"] = h.view(np.uint64)
        t, nc, th = R.truncate_rir(h, 20.0)
        out[f"nc_{i}"] = np.int64(nc)
        out[f"pth_{i}"] = np.float64(th)
    plans, costs = [], []
    for nx, nh in cases.PLAN_CASES:
        s, n, c = R.choose_plan(1, 1, nx, nh)
        plans.append([s, n])
        costs.append(c)
    out["plans"] = np.array(plans, np.int64)
    out["plan_costs"] = np.array(costs)
    x, h, n = cases.ola_case()
    out["ola"] = R.convolve_ola(x, h, n).view(np.uint64)
    path = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden.npz")
    np.savez_compressed(path, **out)
    print("wrote", path, os.path.getsize(path), "bytes")


if __name__ == "__main__":
    main()
