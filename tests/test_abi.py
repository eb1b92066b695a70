"""CPU-only checks of the C-ABI library: it loads, exports every symbol
include/roomsim_gpu.h declares, and its host-side planner mirrors the
reference planner bit for bit (no compute call needs a GPU here)."""
import ctypes as C
import os
import re

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def header_symbols():
    src = open(os.path.join(ROOT, "include", "roomsim_gpu.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(rs_[a-z0-9_]+)\s*\(", src)))


def test_library_exports_header_symbols(rs):
    lib = rs.load_library()
    syms = header_symbols()
    assert len(syms) >= 20
    for s in syms:
        assert hasattr(lib, s), s
    assert sorted(rs.ABI_SYMBOLS) == syms


def test_library_is_sm100a(rs):
    out = os.popen(f"cuobjdump -lelf {rs.LIB_PATH} 2>/dev/null").read()
    if not out:
        pytest.skip("cuobjdump not available")
    assert "sm_100a" in out


def test_planner_mirrors_reference(rs, port):
    rng = np.random.default_rng(0)
    cases = [(116991, 3893), (80000, 4096), (1, 1), (16, 2), (100, 1), (240000, 13120)]
    cases += [(int(rng.integers(1, 300000)), int(rng.integers(1, 20000))) for _ in range(300)]
    for nx, nh in cases:
        p = rs.choose_plan(1.0, 1.0, nx, nh)
        s, n, c = port.choose_plan(1.0, 1.0, nx, nh)
        assert (p.strategy, p.fft_size, p.predicted_cost) == (s, n, c)
        for strat in (0, 1, 2):
            q = rs.plan_for(2.55, 2.0, nx, nh, strat)
            s2, n2, c2 = port.plan_for(2.55, 2.0, nx, nh, strat)
            assert (q.strategy, q.fft_size or 0, q.predicted_cost) == (s2, n2, c2)
        assert rs.ola_block_count(nx, nh, n) == port.ola_block_count(nx, nh, n)
    assert rs.cost_ola(2.55, 2, 116991, 3893, 2 ** 14) == port.cost_ola(2.55, 2, 116991, 3893, 2 ** 14)
    assert rs.cost_full_fft(2.55, 2, 116991, 3893, 2 ** 17) == 69520588.8
    with pytest.raises(rs.PlanError):
        rs.cost_ola(1, 1, 10, 9, 4)
    with pytest.raises(rs.ConfigError):
        rs.plan_for(0.0, 1.0, 10, 9, 2)


def test_no_cpu_fallback_without_library(tmp_path):
    """The product fails loudly when the CUDA library is missing."""
    import subprocess
    import sys

    code = (
        "import sys; sys.path.insert(0, %r)\n"
        "from paper_1712_03439_b200 import roomsim\n"
        "roomsim.LIB_PATH = %r\n"
        "try:\n    roomsim.load_library()\nexcept ImportError as e:\n    print('raised', e)\n"
    ) % (ROOT, str(tmp_path / "missing.so"))
    out = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True).stdout
    assert "raised" in out
