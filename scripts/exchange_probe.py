"""Developer probe: device+host cost of one count step with the hash-partitioned merge, driven
through a 1-rank NCCL group (the collectives are real NCCL calls, the peer is this GPU)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ.setdefault("MASTER_ADDR", "127.0.0.1"); os.environ.setdefault("MASTER_PORT", "29533")
import torch, torch.distributed as dist
from paper_2206_05269_b200 import capi
from paper_2206_05269_b200.exchange import DeviceOps, hash_partition_merge

torch.cuda.set_device(0)
dev = torch.device("cuda", 0)
dist.init_process_group("nccl", rank=0, world_size=1, device_id=dev)
docs = int(sys.argv[1]) if len(sys.argv) > 1 else 954
vocab = int(os.environ.get("VOCAB", "50000"))
corpus = torch.from_numpy(capi.synth_corpus(1, 0, docs, vocab)).cuda()
slots = 1 << 20 if vocab <= 100000 else 1 << 22
local, owned = capi.Counter(table_slots=slots), capi.Counter(table_slots=slots)
ops = DeviceOps(torch, dev)
s = torch.cuda.current_stream().cuda_stream
mode = sys.argv[2] if len(sys.argv) > 2 else "sync"
from paper_2206_05269_b200.exchange import AsyncExchange
ax = AsyncExchange(local, ops, dist, entries_hint=int(sys.argv[3]) if len(sys.argv) > 3 else None)

def step(exchange=True):
    local.reset(s)
    local.count_dev(corpus.data_ptr(), corpus.numel(), s)
    if exchange:
        owned.reset(s)
        if mode == "sync":
            hash_partition_merge(local, owned, ops, dist, force_collectives=True)
        else:
            ax.step(local, owned)

for ex in (False, True):
    for _ in range(3): step(ex)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t0 = time.perf_counter(); e0.record()
    for _ in range(20): step(ex)
    e1.record(); torch.cuda.synchronize()
    print(f"exchange={ex} mode={mode}: {e0.elapsed_time(e1)/20:.3f} ms/step (device), {(time.perf_counter()-t0)/20*1e3:.3f} ms/step (wall)")
if mode != "sync": ax.finish()
print(owned.stats())
dist.destroy_process_group()
