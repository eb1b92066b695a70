"""The C++ drop-in adapter (include/roomsim_gpu.hpp) exercised through the
reference's own API and templates (tests/cpp/adapter_test.cpp)."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BIN = os.path.join(ROOT, "tests", "cpp", "_build", "adapter_test")


@pytest.mark.gpu
def test_cpp_adapter_dropin():
    if not os.path.exists(BIN):
        pytest.skip("adapter_test not built (needs the reference headers at build time)")
    r = subprocess.run([BIN], capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "ADAPTER OK" in r.stdout


def test_adapter_header_declares_engine():
    src = open(os.path.join(ROOT, "include", "roomsim_gpu.hpp")).read()
    assert "static_assert(RealFftEngine<CudaRealFft>)" in src
