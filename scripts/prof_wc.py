"""Tiny driver for ncu: a few word-count launches on a resident corpus."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2206_05269_b200 import capi
docs = int(sys.argv[1]) if len(sys.argv) > 1 else 128
vocab = int(sys.argv[2]) if len(sys.argv) > 2 else 50000
corpus = capi.synth_corpus(1, 0, docs, vocab)
dev = torch.from_numpy(corpus).cuda()
counter = capi.Counter(table_slots=(1 << 20) if vocab <= 100000 else (1 << 22))
for _ in range(4):
    counter.reset(); counter.count_dev(dev.data_ptr(), dev.numel())
torch.cuda.synchronize()
print(counter.stats())
