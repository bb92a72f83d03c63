"""GPU: a C++ reference user's drop-in (include/gcol_cuda.hpp over the C
ABI), checked with the reference's own verify_coloring / count_colors /
first_fit_sequential (tests/cpp/adapter_check.cpp)."""
import os
import subprocess

import pytest

pytestmark = pytest.mark.gpu

BIN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "cpp", "adapter_check")


def test_cpp_adapter_against_reference_types():
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    if not os.path.exists(BIN):
        pytest.skip("adapter_check not built (needs the reference headers at build time)")
    res = subprocess.run([BIN], capture_output=True, text=True, timeout=600)
    assert res.returncode == 0, res.stdout + res.stderr
    assert "adapter_check: OK" in res.stdout
