"""Worker process of tests/test_exchange_gloo.py: one rank of the hash-partitioned
exchange on CPU tensors over gloo.  The device steps are replaced by an oracle-backed
stand-in (tests may use the oracle); the control flow under test is
paper_2206_05269_b200.exchange.hash_partition_merge / allreduce_scalar."""
import json
import os
import random
import struct
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

import numpy as np
import torch
import torch.distributed as dist

import oracle
from helpers import random_text
from paper_2206_05269_b200 import capi
from paper_2206_05269_b200.exchange import (AsyncExchange, ExchangeOverflow, allreduce_scalar, hash_partition_merge,
                                            shard_documents)


class DictCounter:
    def __init__(self):
        self.table = {}

    def max_entries(self):
        return 4096


def key_words(word: bytes):
    p = word.ljust(16, b"\0")
    k0, k1 = struct.unpack(">QQ", p)
    to_i64 = lambda v: v - (1 << 64) if v >= (1 << 63) else v
    return to_i64(k0), to_i64(k1)


def word_of(k0: int, k1: int) -> bytes:
    return struct.pack(">QQ", k0 & (2 ** 64 - 1), k1 & (2 ** 64 - 1)).rstrip(b"\0")


class OracleOps:
    """CPU stand-in for exchange.DeviceOps with the same wire formats."""
    torch = torch

    def partition(self, counter, n_parts):
        rows = [[] for _ in range(n_parts)]
        for w, c in counter.table.items():
            if len(w) <= 16:
                rows[capi.owner_of(w, n_parts)].append([*key_words(w), c, 0])
        flat = [r for part in rows for r in part]
        entries = torch.tensor(flat, dtype=torch.int64).reshape(-1, 4) if flat else torch.zeros((1, 4), dtype=torch.int64)
        long_bytes = sum(16 + len(w) + (-len(w) % 8) for w in counter.table if len(w) > 16)
        return entries, torch.tensor([len(p) for p in rows] + [long_bytes], dtype=torch.int64)

    def merge_entries(self, counter, entries, n):
        for k0, k1, c, _ in entries[:n].tolist():
            w = word_of(k0, k1)
            counter.table[w] = counter.table.get(w, 0) + c

    def long_records(self, counter, n_bytes):
        out = bytearray()
        for w, c in counter.table.items():
            if len(w) > 16:
                out += struct.pack("<QII", c, len(w), 0) + w + b"\0" * (-len(w) % 8)
        assert len(out) == n_bytes
        return torch.tensor(list(out), dtype=torch.uint8)

    def merge_long_records(self, counter, records, part, n_parts):
        raw, off = bytes(records.tolist()), 0
        while off + 16 <= len(raw):
            c, ln, _ = struct.unpack_from("<QII", raw, off)
            w = raw[off + 16:off + 16 + ln]
            if n_parts <= 1 or capi.owner_of(w, n_parts) == part:
                counter.table[w] = counter.table.get(w, 0) + c
            off += 16 + ln + (-ln % 8)

    def partition_fixed(self, counter, n_parts, entries, cap, counts):
        counts[:n_parts] = 0
        for w, c in counter.table.items():
            if len(w) > 16:
                counts[n_parts] += 1
                continue
            p = capi.owner_of(w, n_parts)
            j = int(counts[p])
            counts[p] += 1
            if j < cap:
                entries[p * cap + j] = torch.tensor([*key_words(w), c, 0], dtype=torch.int64)
            else:
                counts[n_parts + 1] += 1

    def partition_framed(self, counter, n_parts, entries, cap, counts):
        counts[:n_parts] = 0
        for w, c in counter.table.items():
            if len(w) > 16:
                counts[n_parts] += 1
                continue
            p = capi.owner_of(w, n_parts)
            j = int(counts[p])
            counts[p] += 1
            if j + 1 < cap:
                entries[p * cap + 1 + j] = torch.tensor([*key_words(w), c, 0], dtype=torch.int64)
            else:
                counts[n_parts + 1] += 1
        for p in range(n_parts):
            entries[p * cap] = torch.tensor([0, 0, min(int(counts[p]), cap - 1), 0], dtype=torch.int64)

    def merge_regions(self, counter, entries, n_parts, cap, counts):
        for p in range(n_parts):
            if counts is None:
                self.merge_entries(counter, entries[p * cap + 1:(p + 1) * cap], int(entries[p * cap][2]))
            else:
                self.merge_entries(counter, entries[p * cap:(p + 1) * cap], min(int(counts[p]), cap))

    def empty_entries(self, n):
        return torch.zeros((max(n, 1), 4), dtype=torch.int64)

    def empty_bytes(self, n):
        return torch.zeros(max(n, 1), dtype=torch.uint8)


def main():
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    dist.init_process_group("gloo", rank=rank, world_size=world)
    rng = random.Random(1234)     # every rank generates the same corpus
    docs = [random_text(rng, rng.randint(0, 1500), rng.choice(["ascii", "unicode", "long"])) for _ in range(31)]
    docs.append(b"L" * 40 + b" " + b"M" * 33 + b" " + b"L" * 40)
    port = oracle.port()
    local, owned = DictCounter(), DictCounter()
    mine = [docs[d] for d in shard_documents(len(docs), rank, world)]
    local.table = port.wordcount(mine)
    stats = hash_partition_merge(local, owned, OracleOps(), dist)
    gathered = [None] * world
    dist.all_gather_object(gathered, {k.hex(): v for k, v in owned.table.items()})
    # the synchronisation-free form: two steps on the short-token part of the same tables, one finish()
    short = DictCounter()
    short.table = {w: c for w, c in local.table.items() if len(w) <= 16}
    ax = AsyncExchange(short, OracleOps(), dist, entries_hint=len(port.wordcount(docs)))
    own_a, own_b = DictCounter(), DictCounter()
    ax.step(short, own_a)
    ax.step(short, own_b)
    ax.finish()
    async_ok = own_a.table == own_b.table == {w: c for w, c in owned.table.items() if len(w) <= 16}
    # a long token, or regions that are too small, must be reported by finish() on EVERY rank
    raised = 0
    for tables, hint in ((local, None), (short, 1)):
        bad = AsyncExchange(tables, OracleOps(), dist, entries_hint=hint)
        if hint == 1:
            bad.cap = 2
            bad.send = bad.send[:world * 2]
            bad.recv = bad.recv[:world * 2]
        bad.step(tables, DictCounter())
        try:
            bad.finish()
        except ExchangeOverflow:
            raised += 1
    # scalar reduction: both modes
    part = torch.tensor([0.1 * (rank + 1)], dtype=torch.float64)
    s1 = float(allreduce_scalar(part, dist, reproducible=True))
    s2 = float(allreduce_scalar(part, dist, reproducible=False))
    if rank == 0:
        merged, ok_disjoint, ok_owner = {}, True, True
        for r, t in enumerate(gathered):
            for k, v in t.items():
                w = bytes.fromhex(k)
                ok_disjoint &= w not in merged
                ok_owner &= capi.owner_of(w, world) == r
                merged[w] = v
        want = port.wordcount(docs)
        print(json.dumps({"equal": merged == want, "disjoint": ok_disjoint, "owner": ok_owner, "distinct": len(want),
                          "sent": stats.sent_entries, "scalar": [s1, s2], "world": world,
                          "async_equal": async_ok, "async_raised": raised}), flush=True)
    dist.barrier()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
