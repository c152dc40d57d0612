"""Small workload for compute-sanitizer covering the HI variant, the exchange regions, utf8_sanitize and the export."""
import os, random, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import numpy as np, torch
from helpers import random_text
from test_gpu_count_kernel import latin_text
from paper_2206_05269_b200 import capi
import oracle
rng = random.Random(3)
text = latin_text(rng, 40000) + b" " + random_text(rng, 8000, "unicode") + b" " + latin_text(rng, 3000)
dev = torch.from_numpy(np.frombuffer(text, dtype=np.uint8).copy()).cuda()
c = capi.Counter(table_slots=1 << 14, deferred_slots=1 << 14, arena_bytes=1 << 20, long_slots=1 << 12)
c.count_dev(dev.data_ptr(), dev.numel())
assert c.to_dict() == oracle.port().wordcount([text])
short = capi.synth_corpus(1, 0, 1, 5000, doc_bytes=1 << 16)
d2 = torch.from_numpy(short).cuda()
c2 = capi.Counter(table_slots=1 << 14)
c2.count_dev(d2.data_ptr(), d2.numel())
want = oracle.port().wordcount([short])
assert c2.to_dict() == want                      # device-packed export
ent = torch.empty((4 * 4096, 4), dtype=torch.int64, device="cuda"); cnt = torch.zeros(6, dtype=torch.int64, device="cuda")
c2.partition_fixed(4, ent.data_ptr(), 4096, cnt.data_ptr())
c3 = capi.Counter(table_slots=1 << 14)
c3.merge_regions(ent.data_ptr(), 4, 4096, cnt.data_ptr())
assert c3.to_dict() == want
assert capi.utf8_sanitize_host(text) == oracle.port().utf8_sanitize(text)
print("sanitize workload 2 ok")
