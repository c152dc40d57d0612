"""Developer probe: throughput on text where a share of the words carries a THREE-byte letter (U+3042 ...): those
fragments are deferred to the exact slow kernel even by the HI variant."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2206_05269_b200 import capi
docs = int(sys.argv[1]) if len(sys.argv) > 1 else 256
pairs = int(sys.argv[2]) if len(sys.argv) > 2 else 5
raw = capi.synth_corpus(1, 0, docs, 50000).tobytes()
for a, b in list(zip((b"ba", b"ca", b"da", b"fa", b"ga", b"a", b"e", b"i"), "あいうえお漢字語"))[:pairs]:
    raw = raw.replace(a, b.encode())
dev = torch.from_numpy(np.frombuffer(raw, dtype=np.uint8).copy()).cuda()
c = capi.Counter(table_slots=1 << 21, deferred_slots=1 << 27)
s = torch.cuda.current_stream().cuda_stream
for _ in range(3):
    c.reset(s); c.count_dev(dev.data_ptr(), dev.numel(), s)
torch.cuda.synchronize()
c.status()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(5):
    c.reset(s); c.count_dev(dev.data_ptr(), dev.numel(), s)
e1.record(); torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / 5
d, t, _ = c.stats()
sample = raw[:4 << 20].split()
hi = sum(1 for w in sample if any(x >= 0x80 for x in w)) / max(1, len(sample))
print(f"three-byte letters: {dev.numel()/1e6:.0f} MB, {ms:.3f} ms -> {dev.numel()/ms/1e6:.1f} GB/s; {d} distinct, {t} tokens, {100*hi:.1f}% of fragments deferred")
