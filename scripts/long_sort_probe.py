"""Developer probe: key sort of token lists with frequent long (> 16 byte) words."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2206_05269_b200 import capi
cases = {
    "one long word": b"hello world " * 20 + b"zzzabcdefghijklmnop ",
    "two stems": b"hello world " * 20 + b"zzzabcdefghijklmnop " + b"foo " * 5 + b"yyyyabcdefghijklmnop ",
    "accented": b"hello world " * 20 + "zzzéabcdefghijklmnop ".encode(),
    "shared 24": b"hello world " * 20 + b"abcdefghijklmnopqrstuvwxYZ " + b"abcdefghijklmnopqrstuvwxAB ",
}
cases["one 30 KB token"] = None
for name, unit in cases.items():
    text = unit * (4_000_000 // len(unit)) if unit else b"hello world " * 300000 + b"k" * 30000 + b" " + b"zzzabcdefghijklmnopq " * 1000
    tk = capi.Tokens.tokenize_host(text)
    torch.cuda.synchronize(); t0 = time.perf_counter()
    tk.sort()
    torch.cuda.synchronize(); dt = time.perf_counter() - t0
    w = tk.words()
    print(f"{name:16s} {len(w):8d} tokens, sort {dt*1e3:7.2f} ms, sorted ok: {w == sorted(w)}")
