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


REF_SUITES = ["text", "reduce", "engine", "pipeline", "analysis", "shuffle", "wire"]


@pytest.mark.parametrize("suite", REF_SUITES)
def test_reference_suite_unmodified(capi, cuda, suite):
    """/root/reference/proj/tests/<suite>_test.cpp, compiled UNMODIFIED from where it lies against the drop-in
    (paper_2206_05269_b200/build.py::build_reference_suites; doctest macros from tests/shim/doctest.h), passes on
    the GPU: every TEST_CASE of the reference's own suite, with its own goldens."""
    exe = capi.LIB_PATH.parent / "reftests" / f"{suite}_test"
    assert exe.exists(), "lib/reftests is built where /root/reference is present and travels with the snapshot"
    out = subprocess.run([str(exe)], capture_output=True, text=True, timeout=900)
    assert out.returncode == 0, out.stdout[-2000:] + out.stderr[-4000:]
    assert "| 0 failed" in out.stdout
