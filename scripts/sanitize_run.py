"""Small mixed workload for compute-sanitizer (memcheck / racecheck)."""
import os, random, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import numpy as np, torch
from helpers import random_text
from paper_2206_05269_b200 import capi
import oracle
rng = random.Random(1)
text = b" ".join(random_text(rng, 3000, f) for f in ("ascii", "unicode", "long")) + b" " + capi.synth_corpus(1, 0, 1, 50000, doc_bytes=1 << 16).tobytes()
dev = torch.from_numpy(np.frombuffer(text, dtype=np.uint8).copy()).cuda()
c = capi.Counter(table_slots=1 << 14, deferred_slots=1 << 14, arena_bytes=1 << 20, long_slots=1 << 12)
c.count_dev(dev.data_ptr(), dev.numel())
assert c.to_dict() == oracle.port().wordcount([text])
c2 = capi.Counter(table_slots=1 << 14, deferred_slots=1 << 14, arena_bytes=1 << 20, long_slots=1 << 12)
c2.count_dev_sorted(dev.data_ptr(), dev.numel())
assert c2.to_dict() == c.to_dict()
t = capi.Tokens.tokenize_dev(dev.data_ptr(), dev.numel()); assert t.words() == oracle.port().tokenize(text)
ent = torch.empty((c.stats()[0], 4), dtype=torch.int64, device="cuda"); cnt = torch.zeros(4, dtype=torch.int64, device="cuda")
c.partition(3, ent.data_ptr(), ent.shape[0], cnt.data_ptr()); torch.cuda.synchronize()
x = capi.synth_uniform(1, 100003, np.float32)
print(capi.map_reduce_host(x, 3), capi.map_reduce_blocked_host(x, 1, 7), "sanitize workload ok")
