"""Developer probe: count_host from PAGEABLE host documents (the packing path: a pool of host threads copies 256 KiB slices into pinned staging,
32 MiB chunks overlap with counting)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2206_05269_b200 import capi
docs_n = 954
corpus = capi.synth_corpus(1, 0, docs_n, 50000)
DOC = 1 << 20
docs = capi.HostDocs([corpus[i * DOC:(i + 1) * DOC] for i in range(docs_n)])
c = capi.Counter(table_slots=1 << 20)
def step():
    c.reset(); c.count_host(docs)
step(); torch.cuda.synchronize()
t0 = time.perf_counter()
for _ in range(5): step()
torch.cuda.synchronize()
ms = (time.perf_counter() - t0) / 5 * 1e3
print(f"pageable count_host: {ms:.2f} ms -> {corpus.size/ms/1e6:.1f} GB/s", c.stats())
