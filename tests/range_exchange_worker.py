"""Worker of tests/test_gpu_exchange.py::test_range_exchange_with_frames: one rank of the paper's range-partitioned
exchange with device WCX1 frames (ranks share the one GPU of the box; gloo carries the device tensors).  Prints the
rank's pre-repair shard as JSON."""
import json
import os
import random
import sys

import torch
import torch.distributed as dist

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
from helpers import random_text   # noqa: E402
from paper_2206_05269_b200 import capi   # noqa: E402
from paper_2206_05269_b200.exchange import range_partition_exchange   # noqa: E402


def corpus():
    rng = random.Random(99)
    docs = [random_text(rng, rng.randint(0, 3000), rng.choice(["ascii", "unicode", "long"])) for _ in range(13)]
    docs.append(b"I want to test MapReduce\n")
    docs.append(b"MapReduce is a cool algorithm to test.\n")
    docs.append(b"L" * 40 + b" " + b"M" * 33 + b" " + b"L" * 40)
    return docs


def main():
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    dist.init_process_group(os.environ.get("WFC_BACKEND", "gloo"), rank=rank, world_size=world)
    torch.cuda.set_device(0)
    device = torch.device("cuda", 0)
    docs = corpus()
    mine = b"\n".join(docs[d] for d in range(rank, len(docs), world)) + b"\n"      # documents d = rank (mod world)
    local = capi.Tokens.tokenize_host(mine)
    local.sort()
    merged = range_partition_exchange(local, dist, torch, device)
    shard = capi.Counter(table_slots=1 << 14)
    merged.reduce_sorted(shard)
    words = merged.words()
    print("SHARD " + json.dumps({"rank": rank, "n": len(words), "sorted": words == sorted(words),
                                 "table": {w.hex(): c for w, c in shard.to_dict().items()}}), flush=True)
    dist.barrier()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
