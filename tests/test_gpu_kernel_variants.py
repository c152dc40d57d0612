"""The counting kernels that the environment can select are all exact: the kernel-level suites are run again, in a
child process each (the switches are read once per process), with the fourth-generation ASCII body
(WFCU_COUNT_KERNEL=4, csrc/wc_count4.cu) and with one variant forced for the whole text (WFCU_COUNT_VARIANT = 0: narrow
ASCII body, 1: two-byte letters, 2: the wide combiner for tokens of up to 16 bytes, 3: both, 4 / 5: 1 / 3 with
three-byte letters as well)."""
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SUITES = ["tests/test_gpu_count_kernel.py", "tests/test_gpu_fuzz.py"]


@pytest.mark.gpu
@pytest.mark.parametrize("env", [
    {"WFCU_COUNT_KERNEL": "4"},
    {"WFCU_COUNT_VARIANT": "0"},
    {"WFCU_COUNT_VARIANT": "1"},
    {"WFCU_COUNT_VARIANT": "2"},
    {"WFCU_COUNT_VARIANT": "3"},
    {"WFCU_COUNT_VARIANT": "4"},
    {"WFCU_COUNT_VARIANT": "5"},
], ids=lambda e: ",".join(f"{k[11:]}={v}" for k, v in e.items()))
def test_suites_under_switch(cuda, env):
    if os.environ.get("WFCU_VARIANT_CHILD"):
        pytest.skip("already inside a child run")
    child_env = dict(os.environ, WFCU_VARIANT_CHILD="1", **env)
    proc = subprocess.run([sys.executable, "-m", "pytest", "-x", "-q", "-m", "gpu", "-p", "no:cacheprovider", *SUITES],
                          cwd=ROOT, env=child_env, capture_output=True, text=True, timeout=900)
    assert proc.returncode == 0, proc.stdout[-3000:] + proc.stderr[-2000:]
