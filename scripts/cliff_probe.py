"""Developer probe: inputs built to hit serial paths -- one giant fragment, random bytes, all whitespace, one byte
repeated -- timed through the counting call (compare with ~1 ms per GB on ordinary text)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2206_05269_b200 import capi
mb = int(sys.argv[1]) if len(sys.argv) > 1 else 64
n = mb << 20
rng = np.random.default_rng(1)
cases = {
    "one fragment of 'a'": np.full(n, ord("a"), np.uint8),
    "one fragment of 0xE3 0x81 0x82 (kana)": np.tile(np.frombuffer("あ".encode(), np.uint8), n // 3 + 1)[:n].copy(),
    "random bytes": rng.integers(0, 256, n, dtype=np.uint8),
    "all spaces": np.full(n, 32, np.uint8),
    "all 0xFF": np.full(n, 255, np.uint8),
    "'a ' repeated": np.tile(np.frombuffer(b"a ", np.uint8), n // 2),
    "1 KiB fragments of letters": np.where(np.arange(n) % 1024 == 1023, 32, ord("b")).astype(np.uint8),
}
for name, arr in cases.items():
    dev = torch.from_numpy(arr).cuda()
    c = capi.Counter(table_slots=1 << 20, deferred_slots=1 << 26, arena_bytes=max(64 << 20, 6 * n), long_slots=1 << 20)
    torch.cuda.synchronize(); t0 = time.perf_counter()
    c.count_dev(dev.data_ptr(), n)
    try:
        st = c.stats()
    except capi.WfcuError as e:
        st = f"error {e.code}"
    dt = time.perf_counter() - t0
    print(f"{name:40s} {mb} MiB: {dt*1e3:9.2f} ms  stats {st}", flush=True)
    c.close()
