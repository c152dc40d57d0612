import os, sys
sys.path.insert(0, "/root/repo")
import torch
from paper_2206_05269_b200 import capi
dev = torch.from_numpy(capi.synth_corpus(1, 0, 256, int(sys.argv[1]) if len(sys.argv) > 1 else 50000)).cuda()
c = capi.Counter(table_slots=1 << 22)
for _ in range(2):
    c.reset(); c.count_dev_sorted(dev.data_ptr(), dev.numel()); torch.cuda.synchronize()
