"""Developer timing loop (not the contract bench): word count + map-reduce on resident data."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2206_05269_b200 import capi

docs = int(sys.argv[1]) if len(sys.argv) > 1 else 954
vocab = int(sys.argv[2]) if len(sys.argv) > 2 else 50000
t0 = time.time()
corpus = capi.synth_corpus(1, 0, docs, vocab)
print(f"corpus {corpus.size/1e9:.3f} GB generated in {time.time()-t0:.1f}s", flush=True)
dev = torch.from_numpy(corpus).cuda()
slots = int(os.environ.get("SLOTS_LOG2", "0")) or (20 if vocab <= 100000 else 22)
counter = capi.Counter(table_slots=1 << slots)
s = torch.cuda.current_stream().cuda_stream
def step():
    counter.reset(s)
    counter.count_dev(dev.data_ptr(), dev.numel(), s)
for _ in range(3): step()
torch.cuda.synchronize()
ev = [torch.cuda.Event(enable_timing=True) for _ in range(11)]
ev[0].record()
for i in range(10):
    step(); ev[i+1].record()
torch.cuda.synchronize()
ms = [ev[i].elapsed_time(ev[i+1]) for i in range(10)]
print("wordcount ms/step:", [round(m,3) for m in ms])
med = sorted(ms)[len(ms)//2]
print(f"wordcount median {med:.3f} ms -> {corpus.size/med/1e6:.1f} GB/s ({corpus.size/med/1e6/6538.6*100:.1f}% of measured HBM peak)")
print("stats (distinct, tokens, key_bytes):", counter.stats(s))

x = torch.rand(1 << 28, device="cuda", dtype=torch.float32)
out = torch.zeros(1, device="cuda", dtype=torch.float64)
for kind in (capi.MAP_IDENTITY, capi.MAP_SQUARE, capi.MAP_SQUARE_ROOT):
    for _ in range(3): capi.map_reduce_dev_async(x.data_ptr(), capi.DTYPE_F32, x.numel(), kind, out.data_ptr(), 0, s)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(10): capi.map_reduce_dev_async(x.data_ptr(), capi.DTYPE_F32, x.numel(), kind, out.data_ptr(), 0, s)
    e1.record(); torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 10
    print(f"mapreduce kind {kind}: {ms:.3f} ms -> {x.numel()*4/ms/1e6:.1f} GB/s ({x.numel()*4/ms/1e6/6538.6*100:.1f}%), value {out.item()!r} torch {x.double().sum().item() if kind==0 else (x.double()**2).sum().item() if kind==3 else x.double().sqrt().sum().item()!r}")
