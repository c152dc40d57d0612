"""The library's device-memory cache (csrc/capi.cu: scratch_alloc / scratch_free, pinned_alloc / pinned_free): objects
created and destroyed in a loop give the same results from recycled, stale-content buffers, the footprint stops
growing, and WFCU_CACHE_KEEP_MB=0 (nothing kept) works the same."""
import os
import subprocess
import sys
import time

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

CHILD = r"""
import sys, time
sys.path.insert(0, %r); sys.path.insert(0, %r + "/tests")
import numpy as np, torch
from paper_2206_05269_b200 import capi
import oracle
port = oracle.port()
texts = [capi.synth_corpus(s, 0, 1, 5000, doc_bytes=1 << 16).tobytes() + b" \xc3\xa9t\xc3\xa9 " + b"x" * 40 for s in (1, 2, 3)]
want = [port.wordcount([t]) for t in texts]
free0 = None
for rep in range(12):
    t = texts[rep %% 3]
    c = capi.Counter(table_slots=1 << 15, deferred_slots=1 << 12, arena_bytes=1 << 16, long_slots=1 << 10)
    c.count_host([t])
    assert c.to_dict() == want[rep %% 3], rep
    tk = capi.Tokens.tokenize_host(t)
    assert tk.words() == port.tokenize(t)
    tk.sort(); c2 = capi.Counter(table_slots=1 << 15); tk.reduce_sorted(c2)
    assert c2.to_dict() == want[rep %% 3]
    c.close(); c2.close(); tk.close()
    torch.cuda.synchronize()
    if rep == 5: free0 = torch.cuda.mem_get_info()[0]
assert torch.cuda.mem_get_info()[0] >= free0 - (8 << 20), "footprint still growing"
print("ok")
"""


@pytest.mark.gpu
@pytest.mark.parametrize("keep_mb", [None, "0"])
def test_recycled_buffers(cuda, keep_mb):
    env = dict(os.environ)
    if keep_mb is not None:
        env["WFCU_CACHE_KEEP_MB"] = keep_mb
    proc = subprocess.run([sys.executable, "-c", CHILD % (ROOT, ROOT)], cwd=ROOT, env=env, capture_output=True, text=True, timeout=600)
    assert proc.returncode == 0 and proc.stdout.strip().endswith("ok"), proc.stdout[-2000:] + proc.stderr[-3000:]


@pytest.mark.gpu
def test_create_destroy_is_cheap(cuda, capi):
    """a default counter is 240 MB of device memory: with the cache the second create + destroy takes well under the
    tens of milliseconds cudaMalloc + cudaFree of that much cost"""
    capi.Counter().close()
    t0 = time.perf_counter()
    for _ in range(5):
        capi.Counter().close()
    assert (time.perf_counter() - t0) / 5 < 0.02
