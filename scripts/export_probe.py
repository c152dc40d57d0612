"""Developer probe: cost of the ordered export (device sort + pack + D2H) against the table size."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2206_05269_b200 import capi
for vocab, docs in ((50000, 128), (1000000, 954)):
    dev = torch.from_numpy(capi.synth_corpus(1, 0, docs, vocab)).cuda()
    c = capi.Counter(table_slots=1 << (20 if vocab <= 100000 else 22))
    c.count_dev(dev.data_ptr(), dev.numel()); torch.cuda.synchronize()
    c.export()
    t0 = time.perf_counter()
    for _ in range(5): blob, lens, counts = c.export()
    ms = (time.perf_counter() - t0) / 5 * 1e3
    print(f"vocab {vocab}: {len(lens)} words, export {ms:.3f} ms, {blob.nbytes + lens.nbytes + counts.nbytes} bytes")
