"""GPU: the C++ drop-in (libwfc_b200.so, the reference's wfc:: API over the C ABI) passes
its reference-style test binary (paper_2206_05269_b200/host/tests/dropin_tests.cpp)."""
import subprocess

import pytest

pytestmark = pytest.mark.gpu


def test_dropin_binary(capi, cuda):
    exe = capi.LIB_PATH.parent / "wfc_dropin_tests"
    assert exe.exists(), "build the host drop-in first (python -m paper_2206_05269_b200.build)"
    out = subprocess.run([str(exe)], capture_output=True, text=True, timeout=600)
    assert out.returncode == 0, out.stdout[-3000:] + out.stderr[-1000:]
    assert "0 failed" in out.stdout
