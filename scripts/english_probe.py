"""throughput on English-like text: the reference's four speech fixtures (from the golden file) tiled to 256 MiB"""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2206_05269_b200 import capi
f = json.load(open("tests/golden/fixtures.json"))
text = b"".join(bytes.fromhex(d) + b"\n" for n, g in f.items() if "docs" in g and n.startswith("speeches/") for d in g["docs"])
reps = (256 << 20) // len(text)
dev = torch.from_numpy(np.frombuffer(text, dtype=np.uint8).copy()).cuda().repeat(reps)
c = capi.Counter(table_slots=1 << 16)
for _ in range(3):
    c.reset(); c.count_dev(dev.data_ptr(), dev.numel())
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(5):
    c.reset(); c.count_dev(dev.data_ptr(), dev.numel())
e1.record(); torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / 5
d, t, _ = c.stats()
print(f"english-like: {dev.numel()/1e6:.0f} MB, {ms:.3f} ms -> {dev.numel()/ms/1e6:.1f} GB/s; {d} distinct, {t} tokens ({dev.numel()/t:.2f} B/token), tokens ok: {t == 832 * reps}")
