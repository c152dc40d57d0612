"""Developer probe: cfg3 text in which a share of the words is lengthened past 8 bytes (k bigrams get three more
letters) -- where the narrow / WIDE crossover lies (run under WFCU_COUNT_VARIANT=0, 2 and unset)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2206_05269_b200 import capi
k = int(sys.argv[1]) if len(sys.argv) > 1 else 1
raw = capi.synth_corpus(1, 0, 256, 50000).tobytes()
for a in (b"ba", b"ca", b"da", b"fa", b"ga", b"ha", b"ja", b"ka")[:k]:
    raw = raw.replace(a, a + b"xyz")
raw = raw[:len(raw) & ~15]
dev = torch.from_numpy(np.frombuffer(raw, dtype=np.uint8).copy()).cuda()
c = capi.Counter(table_slots=1 << 20)
s = torch.cuda.current_stream().cuda_stream
for _ in range(10):
    c.reset(s); c.count_dev(dev.data_ptr(), dev.numel(), s)
torch.cuda.synchronize(); c.status()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
l0 = capi.launch_count()
e0.record()
for _ in range(30):
    c.reset(s); c.count_dev(dev.data_ptr(), dev.numel(), s)
e1.record(); torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / 30
words = raw[:4 << 20].split()
share = sum(1 for w in words if len(w.strip(b".,;!?")) > 8) / len(words)
print(f"[{(capi.launch_count() - l0) / 30:.0f} launches per step] long words {100*share:.1f} % (k={k}, variant {os.environ.get('WFCU_COUNT_VARIANT', 'auto')}): {dev.numel()/ms/1e6:.1f} GB/s")
