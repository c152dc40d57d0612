import os, sys, time
sys.path.insert(0, "/root/repo")
import numpy as np, torch
from paper_2206_05269_b200 import capi
corpus = capi.synth_corpus(1, 0, 16, 50000)
dev = torch.from_numpy(corpus).cuda()
def t(label, fn, reps=3):
    fn(); torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(reps): r = fn()
    torch.cuda.synchronize()
    print(f"{label:40s} {1e3 * (time.perf_counter() - t0) / reps:8.2f} ms"); return r
b = corpus.tobytes()
tk = t("tokenize_dev 16 MiB (resident)", lambda: capi.Tokens.tokenize_dev(dev.data_ptr(), dev.numel()))
t("tokenize_host 16 MiB (bytes)", lambda: capi.Tokens.tokenize_host(b))
tk.sort()
def red():
    c = capi.Counter(table_slots=1 << 18); tk.reduce_sorted(c); return c
t("Counter() + reduce_sorted", red)
c = capi.Counter(table_slots=1 << 18)
def red2():
    c.reset(); tk.reduce_sorted(c)
t("reset + reduce_sorted (reused counter)", red2)
t("Counter(table_slots=1<<18) alone", lambda: capi.Counter(table_slots=1 << 18))
t("Counter(small everything)", lambda: capi.Counter(table_slots=1 << 18, deferred_slots=1 << 16, arena_bytes=1 << 20, long_slots=1 << 14))
