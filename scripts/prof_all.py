"""Tiny driver for ncu: one or two launches of every kernel family next to the counting kernel (engine, sort + RLE,
exchange partition / merge, exact slow path, distinctive join / score, bit-exact folds)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2206_05269_b200 import capi

torch.cuda.set_device(0)
docs = int(sys.argv[1]) if len(sys.argv) > 1 else 256
corpus = capi.synth_corpus(1, 0, docs, 50000)
dev = torch.from_numpy(corpus).cuda()
# engine: roofline reduction + bit-exact folds
x = torch.from_numpy(capi.synth_uniform(1, 1 << 27, np.float32)).cuda()
for kind in (capi.MAP_IDENTITY, capi.MAP_SQUARE):
    capi.map_reduce_dev(x.data_ptr(), capi.DTYPE_F32, x.numel(), kind)
capi.map_reduce_blocked_dev(x.data_ptr(), capi.DTYPE_F32, x.numel(), capi.MAP_SQUARE_ROOT, 256)
capi.map_reduce_blocked_dev(x.data_ptr(), capi.DTYPE_F32, 1 << 22, capi.MAP_SQUARE_ROOT, 1 << 22)
# counting map by sort + RLE (tokenize, radix sort, run-length encode, insert)
c = capi.Counter(table_slots=1 << 20)
c.count_dev_sorted(dev.data_ptr(), dev.numel())
# hash count + exchange kernels with two logical workers
a, b = capi.Counter(table_slots=1 << 20), capi.Counter(table_slots=1 << 20)
a.count_dev(dev.data_ptr(), dev.numel())
cap = 2 * (a.max_entries() // 2 + 1)
entries = torch.empty(2 * cap * 32, dtype=torch.uint8, device="cuda")
counts = torch.zeros(4, dtype=torch.int64, device="cuda")
a.partition_fixed(2, entries.data_ptr(), cap, counts.data_ptr())
b.merge_regions(entries.data_ptr(), 2, cap, counts.data_ptr())
b.merge(a)
# exact slow path: three-byte letters in 13 % of the words
raw = corpus.tobytes()
for s_, r_ in ((b"ba", "あ"), (b"ca", "い"), (b"da", "う"), (b"fa", "え"), (b"ga", "お")):
    raw = raw.replace(s_, r_.encode())
cj = torch.from_numpy(np.frombuffer(raw, dtype=np.uint8).copy()).cuda()
d = capi.Counter(table_slots=1 << 21, deferred_slots=1 << 26)
d.count_dev(cj.data_ptr(), cj.numel())
# reports
a.top_k(25)
a.distinctive(d, 25)
a.export()
capi.utf8_sanitize_dev(dev.data_ptr(), dev.numel(), torch.empty(dev.numel() + 4096, dtype=torch.uint8, device="cuda").data_ptr(), dev.numel() + 4096)
torch.cuda.synchronize()
print("ok", a.stats(), d.stats())
