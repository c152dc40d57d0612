"""Developer probe: utf8_sanitize throughput on a resident 1 GB shard (valid text, 1 invalid byte in 1000, 1 in 20)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2206_05269_b200 import capi
docs = int(sys.argv[1]) if len(sys.argv) > 1 else 954
corpus = capi.synth_corpus(1, 0, docs, 50000)
for name, every in (("valid", 0), ("1 in 1000 invalid", 1000), ("1 in 20 invalid", 20)):
    arr = corpus.copy()
    if every: arr[::every] = 0xFF
    dev = torch.from_numpy(arr).cuda()
    out = torch.empty(3 * arr.size // (1 if every == 20 else 2) + 64, dtype=torch.uint8, device="cuda")
    s = torch.cuda.current_stream().cuda_stream
    for _ in range(3): n_out = capi.utf8_sanitize_dev(dev.data_ptr(), arr.size, out.data_ptr(), out.numel(), s)
    e = [torch.cuda.Event(enable_timing=True) for _ in range(11)]
    e[0].record()
    for i in range(10):
        capi.utf8_sanitize_dev(dev.data_ptr(), arr.size, out.data_ptr(), out.numel(), s); e[i + 1].record()
    torch.cuda.synchronize()
    ms = sorted(e[i].elapsed_time(e[i + 1]) for i in range(10))[5]
    print(f"{name:18s}: {ms:.3f} ms  input {arr.size/ms/1e6:7.1f} GB/s  read+write {(arr.size+n_out)/ms/1e6:7.1f} GB/s  out {n_out}")
