import sys, time
sys.path.insert(0, "/root/repo")
import numpy as np, torch
from paper_2206_05269_b200 import capi
for mb in (1, 16):
    n = mb << 20
    arr = np.full(n, ord("a"), np.uint8); arr[n // 2] = 32     # two giant tokens of n/2
    dev = torch.from_numpy(arr).cuda()
    c = capi.Counter(table_slots=1 << 16, arena_bytes=4 * n + (1 << 20), long_slots=1 << 12)
    t0 = time.perf_counter(); c.count_dev(dev.data_ptr(), n); st = c.stats(); t1 = time.perf_counter()
    d = c.to_dict(); t2 = time.perf_counter()
    tk = capi.Tokens.tokenize_dev(dev.data_ptr(), n); tk.sort(); c2 = capi.Counter(table_slots=1 << 16, arena_bytes=4 * n + (1 << 20)); tk.reduce_sorted(c2); t3 = time.perf_counter()
    print(f"{mb} MiB, two giant tokens: count {1e3*(t1-t0):.1f} ms, export {1e3*(t2-t1):.1f} ms, tokenize+sort+rle {1e3*(t3-t2):.1f} ms; stats {st}, keys {[len(k) for k in d]}, values {list(d.values())}, sorted path equal {c2.to_dict() == d}")
