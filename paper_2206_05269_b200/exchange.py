"""Multi-GPU merge of per-GPU count tables: hash-partitioned all-to-all over NCCL.

One process per GPU (torchrun).  Replaces the reference's exchange stage
(/root/reference/proj/src/shuffle.cpp:98-168: range partition of sorted words, n(n-1)
WCX1 frames, n-way merge) and the merge_counts / boundary_repair that follow it
(proj/src/reduce.cpp:48-89) -- see SURVEY.md D2: the contract is the final CountMap,
the shard layout is implementation defined.

    per rank:  local table --K4 partition-by-owner--> n contiguous regions of 32-byte
               entries --all_to_all(sizes), all_to_all_v(entries)--> K5 merge-insert
               into the rank's OWNED table (every key lives on exactly one rank, so
               count_unreduced_words == 0 and no repair pass is needed).

torch.distributed is the plumbing (rendezvous, NCCL all-to-all over NVLink 5 / NVSwitch);
partition and merge are kernels of libwfcu.so reached through the C ABI.  The `ops`
argument isolates those device steps so the control flow can be exercised on CPU with
gloo (tests/test_exchange_gloo.py supplies an oracle-backed stand-in); the product always
uses DeviceOps and has no CPU path.
"""
from __future__ import annotations

from dataclasses import dataclass

ENTRY_WORDS = 4   # wfcu_entry = 4 x u64 = 32 bytes


class DeviceOps:
    """The device steps of the exchange, through libwfcu.so."""

    def __init__(self, torch, device):
        from . import capi
        self.capi = capi
        self.torch = torch
        self.device = device

    def stream(self) -> int:
        return self.torch.cuda.current_stream(self.device).cuda_stream

    def partition(self, counter, n_parts: int):
        """-> (entries[int64, cap x 4] grouped by owner, counts[int64, n_parts + 1]) on device;
        counts[n_parts] = bytes of the long-token record stream.  No host synchronisation."""
        t = self.torch
        cap = counter.max_entries()
        entries = t.empty((cap, ENTRY_WORDS), dtype=t.int64, device=self.device)
        counts = t.zeros(n_parts + 1, dtype=t.int64, device=self.device)
        counter.partition(n_parts, entries.data_ptr(), cap, counts.data_ptr(), self.stream())
        return entries, counts

    def merge_entries(self, counter, entries, n: int) -> None:
        if n:
            counter.merge_entries(entries.data_ptr(), n, self.stream())

    def long_records(self, counter, n_bytes: int):
        t = self.torch
        buf = t.empty(max(n_bytes, 8), dtype=t.uint8, device=self.device)
        if n_bytes:
            counter.long_records(buf.data_ptr(), n_bytes, self.stream())
        return buf[:n_bytes]

    def merge_long_records(self, counter, records, part: int, n_parts: int) -> None:
        if records.numel():
            counter.merge_long_records(records.data_ptr(), records.numel(), part, n_parts, self.stream())

    def partition_fixed(self, counter, n_parts: int, entries, cap_per_part: int, counts) -> None:
        counter.partition_fixed(n_parts, entries.data_ptr(), cap_per_part, counts.data_ptr(), self.stream())

    def partition_framed(self, counter, n_parts: int, entries, cap_per_part: int, counts) -> None:
        counter.partition_framed(n_parts, entries.data_ptr(), cap_per_part, counts.data_ptr(), self.stream())

    def merge_regions(self, counter, entries, n_parts: int, cap_per_part: int, counts) -> None:
        counter.merge_regions(entries.data_ptr(), n_parts, cap_per_part, counts.data_ptr() if counts is not None else 0,
                              self.stream())

    def empty_entries(self, n: int):
        t = self.torch
        return t.empty((max(n, 1), ENTRY_WORDS), dtype=t.int64, device=self.device)

    def empty_bytes(self, n: int):
        t = self.torch
        return t.empty(max(n, 1), dtype=t.uint8, device=self.device)

    # stream plumbing of AsyncExchange(overlap=True): a second stream for the collective and the merge
    def new_stream(self):
        return self.torch.cuda.Stream(device=self.device)

    def record(self):
        """an event at the current point of the current stream"""
        ev = self.torch.cuda.Event()
        ev.record(self.torch.cuda.current_stream(self.device))
        return ev

    def wait(self, event) -> None:
        """the current stream waits for the event (no host wait)"""
        self.torch.cuda.current_stream(self.device).wait_event(event)

    def on(self, stream):
        """context manager: the current stream inside is `stream`"""
        return self.torch.cuda.stream(stream)


@dataclass
class ExchangeStats:
    sent_entries: int
    received_entries: int
    sent_bytes: int
    long_bytes: int


def hash_partition_merge(local, owned, ops, dist, group=None, force_collectives: bool = False) -> ExchangeStats:
    """Moves every entry of `local` to the rank that owns its key and sums it into `owned`.

    local / owned are counters (capi.Counter for DeviceOps).  Collective: every rank of the
    group must call it.  After the call the union of the ranks' `owned` tables is the
    merged CountMap and the tables are pairwise disjoint.
    """
    torch = ops.torch
    world = dist.get_world_size(group)
    rank = dist.get_rank(group)

    entries, counts = ops.partition(local, world)
    if world == 1 and not force_collectives:   # force_collectives: tests drive the NCCL calls with one rank
        host = [int(v) for v in counts.cpu().tolist()]
        ops.merge_entries(owned, entries, host[0])
        if host[1]:
            ops.merge_long_records(owned, ops.long_records(local, host[1]), 0, 1)
        return ExchangeStats(host[0], host[0], 0, host[1])

    # one small all-to-all tells every peer how many entries it gets from me and how long my
    # long-token stream is; one host read of the result is the only synchronisation of the step
    send_meta = torch.stack([counts[:world], counts[world].expand(world)], dim=1).contiguous()   # [world, 2]
    recv_meta = torch.empty_like(send_meta)
    dist.all_to_all_single(recv_meta, send_meta, group=group)
    meta = torch.cat([send_meta, recv_meta], dim=1).cpu().tolist()        # the step's single D2H
    send_list = [int(r[0]) for r in meta]
    recv_list = [int(r[2]) for r in meta]
    long_sizes = [int(r[3]) for r in meta]                                 # peer r's long-stream bytes
    n_send, n_recv = sum(send_list), sum(recv_list)
    recv = ops.empty_entries(n_recv)
    dist.all_to_all_single(recv[:n_recv], entries[:n_send], output_split_sizes=recv_list,
                           input_split_sizes=send_list, group=group)
    ops.merge_entries(owned, recv, n_recv)

    # tokens longer than 16 bytes: rare, variable length -> all-gather the record streams and
    # let every rank keep the records it owns (skipped entirely when nobody has any)
    long_total = sum(long_sizes)
    if long_total:
        mine = ops.long_records(local, long_sizes[rank])
        width = max(long_sizes)
        padded = ops.empty_bytes(width)
        padded.zero_()
        padded[:mine.numel()] = mine
        gathered = ops.empty_bytes(width * world)
        parts = [gathered[r * width:(r + 1) * width] for r in range(world)]
        dist.all_gather(parts, padded[:width], group=group)
        for r in range(world):
            if long_sizes[r]:
                ops.merge_long_records(owned, gathered[r * width:r * width + long_sizes[r]], rank, world)
    return ExchangeStats(n_send, n_recv, n_send * 8 * ENTRY_WORDS, long_total)


class ExchangeOverflow(RuntimeError):
    """A synchronisation-free step could not carry everything: redo it with hash_partition_merge."""


class AsyncExchange:
    """The same merge with NO host synchronisation per step, for pipelines that count and merge
    repeatedly (bench.py's N>1 step): partition p of the local table is scattered into a region of
    fixed capacity whose first entry is a header with the number of entries that follow, so ONE
    all-to-all of host-independent shape is the whole exchange and the receiving kernel reads the
    sizes out of the regions (round 1 sent the sizes in an all-to-all of their own: pure latency).  What the
    fixed shapes cannot carry -- a region that overflows, tokens longer than 16 bytes (their
    variable-length record stream needs sizes on the host) -- raises sticky device flags that
    finish() reads ONCE, after any number of steps; the caller then falls back to
    hash_partition_merge for those steps.

    entries_hint: expected distinct words of a local table (regions hold 2x the uniform share);
    default = the table's capacity, which can never overflow.

    overlap=True: the all-to-all and the merge of step k run on a second stream while the caller's stream goes on to
    reset and count step k+1 (`local` is free again as soon as its partition kernel has run; `owned` belongs to the
    second stream until finish(), which joins the two).  Two send buffers alternate, so the partition of step k+2
    waits for the all-to-all of step k by an event, never the host.  The caller must not touch `owned` (reset
    included) between step() and finish() on its own stream -- give every step its own table or call
    owned_ready() first."""

    def __init__(self, local, ops, dist, group=None, entries_hint: int | None = None, overlap: bool = False):
        self.ops, self.dist, self.group = ops, dist, group
        self.world = dist.get_world_size(group)
        bound = local.max_entries()
        want = bound if entries_hint is None else min(bound, 2 * ((entries_hint + self.world - 1) // self.world) + 1024)
        self.cap = max(int(want), 16) + 1          # + the header entry of a region
        t = ops.torch
        self.send = ops.empty_entries(self.world * self.cap)
        self.recv = ops.empty_entries(self.world * self.cap)
        self.counts = t.zeros(self.world + 2, dtype=t.int64, device=self.send.device)
        self.steps = 0
        self.overlap = bool(overlap) and hasattr(ops, "new_stream")
        if self.overlap:
            self.comm = ops.new_stream()
            self.sends = [self.send, ops.empty_entries(self.world * self.cap)]
            self.sent = [None, None]        # event: the all-to-all that read sends[k] (and its merge) has run
            self.merged = None              # event: the latest merge on the second stream

    def step(self, local, owned) -> None:
        """Collective.  Asynchronous on the current stream: returns before anything has run."""
        ops, world = self.ops, self.world
        if not self.overlap:
            ops.partition_framed(local, world, self.send, self.cap, self.counts)
            self.dist.all_to_all_single(self.recv, self.send, group=self.group)
            ops.merge_regions(owned, self.recv, world, self.cap, None)
            self.steps += 1
            return
        k = self.steps & 1
        if self.sent[k] is not None:
            ops.wait(self.sent[k])          # sends[k] is free again
        ops.partition_framed(local, world, self.sends[k], self.cap, self.counts)
        ready = ops.record()
        with ops.on(self.comm):
            ops.wait(ready)
            self.dist.all_to_all_single(self.recv, self.sends[k], group=self.group)
            ops.merge_regions(owned, self.recv, world, self.cap, None)
            self.sent[k] = self.merged = ops.record()
        self.steps += 1

    def slot_ready(self) -> None:
        """overlap=True: the caller's stream waits (no host wait) for the merge of the step two steps back -- after it
        the `owned` table of that step may be reset and handed to the next step() (two tables alternate)."""
        if self.overlap and self.sent[self.steps & 1] is not None:
            self.ops.wait(self.sent[self.steps & 1])

    def owned_ready(self) -> None:
        """overlap=True: the caller's stream waits (no host wait) until every merge issued so far has run."""
        if self.overlap and self.merged is not None:
            self.ops.wait(self.merged)

    def finish(self) -> None:
        """The one host read: raises ExchangeOverflow if any step since the last finish() left
        something behind (on any rank), and clears the flags."""
        self.owned_ready()
        flags = self.counts[self.world:self.world + 2].clone()
        self.dist.all_reduce(flags, group=self.group)
        long_tokens, overflow = (int(v) for v in flags.cpu().tolist())
        self.counts[self.world:].zero_()
        if overflow or long_tokens:
            raise ExchangeOverflow(f"{overflow} entries beyond the region capacity {self.cap}, "
                                   f"{long_tokens} tokens longer than 16 bytes in {self.steps} steps")


def partition_cuts(k: int, worker_id: int, n_workers: int) -> list[int]:
    """plan_partition (/root/reference/proj/src/shuffle.cpp:9-46): the kept chunk gets floor(k/n) words, the rest is
    spread over the other chunks, one extra each from chunk 0 upward.  Index arithmetic on the list length."""
    n = n_workers
    keep = k // n
    others = n - 1 if n > 1 else 1
    base = (k - keep) // others if n > 1 else 0
    extra = (k - keep) % others if n > 1 else 0
    cut = [0]
    for c in range(n):
        size = keep
        if c != worker_id:
            size = base + (1 if extra else 0)
            extra -= 1 if extra else 0
        cut.append(cut[-1] + size)
    return cut


def range_partition_exchange(local, dist, torch, device, group=None):
    """The paper's own exchange between ranks (proj/src/shuffle.cpp:98-130), one rank per GPU, with the WCX1 frame as
    wire format and the collective library as transport: chunk c of this rank's SORTED token list (capi.Tokens) is
    framed on the device (wfcu_tokens_encode_frame), an all-to-all of the frame sizes tells every rank what arrives
    (the one host read: frames have variable length), an all-to-all of the frame bytes delivers them -- device buffers
    end to end, NCCL over NVLink -- and every received frame is validated and decoded on the device
    (wfcu_tokens_decode_frame: a bad frame raises capi.WfcuError with the ERR_FRAME_* code, the reference's
    WireError kinds).  The kept chunk and the decoded chunks are gathered in source order and radix-sorted: the n-way
    merge.  Returns this rank's range of the global sorted list (capi.Tokens, sorted); reduce_sorted of it is the
    reference's pre-repair shard."""
    from . import capi
    world, rank = dist.get_world_size(group), dist.get_rank(group)
    k, _ = local.stats()
    cut = partition_cuts(k, rank, world)
    if world == 1:
        return capi.Tokens.concat_slices([local], [0], [k])
    pad = lambda b: (b + 15) & ~15
    sizes = [0 if c == rank else local.frame_bytes(cut[c], cut[c + 1]) for c in range(world)]
    send = torch.zeros(max(sum(pad(b) for b in sizes), 16), dtype=torch.uint8, device=device)
    off = 0
    for c in range(world):
        if c != rank:
            local.encode_frame(cut[c], cut[c + 1], send.data_ptr() + off, pad(sizes[c]))
            off += pad(sizes[c])
    send_sizes = torch.tensor(sizes, dtype=torch.int64, device=device)
    recv_sizes = torch.empty_like(send_sizes)
    dist.all_to_all_single(recv_sizes, send_sizes, group=group)
    got = [int(v) for v in recv_sizes.cpu().tolist()]
    recv = torch.zeros(max(sum(pad(b) for b in got), 16), dtype=torch.uint8, device=device)
    dist.all_to_all_single(recv[:sum(pad(b) for b in got)], send[:sum(pad(b) for b in sizes)],
                           output_split_sizes=[pad(b) for b in got], input_split_sizes=[pad(b) for b in sizes], group=group)
    torch.cuda.synchronize(device) if device is not None and str(device).startswith("cuda") else None
    parts, off = [], 0
    for src in range(world):
        if src == rank:
            parts.append((local, cut[rank], cut[rank + 1]))
        else:
            t = capi.Tokens.decode_frame(recv.data_ptr() + off, got[src])
            parts.append((t, 0, t.stats()[0]))
            off += pad(got[src])
    merged = capi.Tokens.concat_slices([p[0] for p in parts], [p[1] for p in parts], [p[2] for p in parts])
    merged.sort()
    return merged


def allreduce_scalar(partial, dist, group=None, reproducible: bool = True):
    """Finishes a sharded map-then-reduce: sum of the ranks' partial sums.

    partial: 1-element float64 tensor (device for NCCL).  reproducible=True gathers the n
    partials and adds them in rank order (bitwise run-to-run stable, the reference's
    determinism contract, proj/include/wfc/engine.hpp:27-31); False is a plain allreduce.
    """
    world = dist.get_world_size(group)
    if world == 1:
        return partial.clone()
    if not reproducible:
        out = partial.clone()
        dist.all_reduce(out, group=group)
        return out
    parts = [partial.new_empty(partial.shape) for _ in range(world)]
    dist.all_gather(parts, partial, group=group)
    acc = parts[0].clone()
    for p in parts[1:]:
        acc += p
    return acc


def shard_documents(n_docs: int, rank: int, world: int) -> range:
    """Round-robin document assignment d = rank (mod world), the reference's rule
    (/root/reference/proj/src/pipeline.cpp:83)."""
    return range(rank, n_docs, world)
