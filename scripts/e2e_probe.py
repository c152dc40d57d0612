"""Developer probe: where the end-to-end step (count_host + export) spends its time."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2206_05269_b200 import capi

docs_n = int(sys.argv[1]) if len(sys.argv) > 1 else 954
DOC = 1 << 20
host = torch.empty(docs_n * DOC, dtype=torch.uint8).pin_memory()
arr = host.numpy()
capi.synth_corpus_strided(1, 0, 1, docs_n, 50000, 1.1, 0, DOC, out=arr)
docs = [arr[i * DOC:(i + 1) * DOC] for i in range(docs_n)]
c = capi.Counter(table_slots=1 << 20)
dev = torch.empty_like(host, device="cuda")

def t(fn, n=5):
    fn(); torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(n): fn()
    torch.cuda.synchronize()
    return (time.perf_counter() - t0) / n * 1e3

print("bare pinned H2D copy   %.2f ms -> %.1f GB/s" % ((lambda ms: (ms, host.numel() / ms / 1e6))(t(lambda: dev.copy_(host, non_blocking=True)))))
print("reset                  %.2f ms" % t(lambda: c.reset()))
hd = capi.HostDocs(docs)
def cnt_prepared():
    c.reset(); c.count_host(hd)
print("reset+count_host(prep) %.2f ms" % t(cnt_prepared))
def cnt():
    c.reset(); c.count_host(docs)
ms = t(cnt)
print("reset+count_host       %.2f ms -> %.1f GB/s" % (ms, host.numel() / ms / 1e6))
print("export                 %.2f ms" % t(lambda: c.export()))
def full():
    c.reset(); c.count_host(docs); c.export()
ms = t(full)
print("full e2e step          %.2f ms -> %.1f GB/s" % (ms, host.numel() / ms / 1e6))
# resident count for comparison
s = torch.cuda.current_stream().cuda_stream
def res():
    c.reset(s); c.count_dev(dev.data_ptr(), dev.numel(), s)
print("resident reset+count   %.2f ms" % t(res))
