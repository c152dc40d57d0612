import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2206_05269_b200 import capi
host = torch.empty(954 << 20, dtype=torch.uint8).pin_memory()
capi.synth_corpus(1, 0, 954, 50000, out=host.numpy())
dev = host.cuda()
c = capi.Counter(table_slots=1 << 20)
c.count_dev(dev.data_ptr(), dev.numel()); torch.cuda.synchronize(); ref = c.stats()
for name, ptr in (("resident", dev.data_ptr()), ("pinned-host (UVA zero-copy)", host.data_ptr())):
    for _ in range(2):
        c.reset(); c.count_dev(ptr, host.numel()); torch.cuda.synchronize()
    t = time.perf_counter()
    for _ in range(3):
        c.reset(); c.count_dev(ptr, host.numel())
    torch.cuda.synchronize()
    dt = (time.perf_counter() - t) / 3
    print(f"{name}: {dt*1e3:.2f} ms -> {host.numel()/dt/1e9:.1f} GB/s, stats ok: {c.stats() == ref}")
