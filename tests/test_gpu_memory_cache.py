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


@pytest.mark.gpu
def test_undersized_tables_fail_promptly(cuda, capi):
    """a vocabulary (or a set of long tokens) far larger than the table was sized for is reported as TABLE_FULL /
    ARENA_FULL within a bounded number of probes per insertion -- not after every insertion has walked the whole
    table (64 MiB of random bytes into a 1 M-slot long table took 33 s before the bound)"""
    import torch
    rng = np.random.default_rng(5)
    words = rng.integers(0, 26, (600_000, 8), dtype=np.uint8) + ord("a")
    text = np.concatenate([words, np.full((600_000, 1), 32, np.uint8)], axis=1).reshape(-1)      # ~600 k distinct words
    dev = torch.from_numpy(text).cuda()
    c = capi.Counter(table_slots=1 << 14)
    t0 = time.perf_counter()
    with pytest.raises(capi.WfcuError) as e:
        c.count_dev(dev.data_ptr(), text.size)
        c.status()
    assert e.value.code == capi.ERR_TABLE_FULL and time.perf_counter() - t0 < 5.0
    longs = rng.integers(0, 26, (300_000, 20), dtype=np.uint8) + ord("a")
    text2 = np.concatenate([longs, np.full((300_000, 1), 32, np.uint8)], axis=1).reshape(-1)   # 300 k distinct long tokens
    dev2 = torch.from_numpy(text2).cuda()
    c2 = capi.Counter(table_slots=1 << 14, long_slots=1 << 12, arena_bytes=64 << 20, deferred_slots=1 << 20)
    t0 = time.perf_counter()
    with pytest.raises(capi.WfcuError) as e:
        c2.count_dev(dev2.data_ptr(), text2.size)
        c2.status()
    assert e.value.code == capi.ERR_ARENA_FULL and time.perf_counter() - t0 < 5.0
