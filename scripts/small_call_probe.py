"""Developer probe: fixed cost of one count_dev call -- time per call against the size of the text."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2206_05269_b200 import capi

corpus = capi.synth_corpus(1, 0, 256, 50000)
dev = torch.from_numpy(corpus).cuda()
counter = capi.Counter(table_slots=1 << 20)
s = torch.cuda.current_stream().cuda_stream
counter.count_dev(dev.data_ptr(), dev.numel(), s)
for kib in (1, 64, 1024, 4096, 8192, 16384, 32768, 65536, 262144):
    n = kib << 10
    for _ in range(3): counter.count_dev(dev.data_ptr(), n, s)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(20): counter.count_dev(dev.data_ptr(), n, s)
    e1.record(); torch.cuda.synchronize()
    us = e0.elapsed_time(e1) / 20 * 1e3
    print(f"{kib:7d} KiB: {us:8.1f} us/call  {n/us/1e3:7.1f} GB/s")
