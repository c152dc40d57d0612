"""Developer probe: stand-alone tokenizer / sort / RLE throughput on a resident corpus."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2206_05269_b200 import capi
docs = int(sys.argv[1]) if len(sys.argv) > 1 else 128
vocab = int(sys.argv[2]) if len(sys.argv) > 2 else 50000
dev = torch.from_numpy(capi.synth_corpus(1, 0, docs, vocab)).cuda()
def t(fn, n=3):
    fn(); torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(n): r = fn()
    torch.cuda.synchronize()
    return (time.perf_counter() - t0) / n * 1e3
ms = t(lambda: capi.Tokens.tokenize_dev(dev.data_ptr(), dev.numel()).close())
print(f"tokenize_dev: {dev.numel()/1e6:.0f} MB in {ms:.2f} ms -> {dev.numel()/ms/1e6:.1f} GB/s")
c = capi.Counter(table_slots=1 << 22)
ms = t(lambda: (c.reset(), c.count_dev_sorted(dev.data_ptr(), dev.numel()), torch.cuda.synchronize()))
print(f"count_dev_sorted (tokenize + radix sort + RLE): {ms:.2f} ms -> {dev.numel()/ms/1e6:.1f} GB/s")
