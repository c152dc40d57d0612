"""GPU parity: hash-partitioned exchange + merge (the multi-GPU merge, run here with n
logical workers on one device) vs the reference's run_wordcount contract:
final counts == serial_wordcount for any corpus and worker count, documents assigned
round-robin (proj/src/pipeline.cpp:61-123; tests proj/tests/pipeline_test.cpp:82-135).
"""
import random

import numpy as np
import pytest

from helpers import random_text, to_dev

pytestmark = pytest.mark.gpu


def run_workers(capi, torch, docs, n_workers, slots=1 << 14):
    """n logical workers on one GPU: count shards d mod n, partition, exchange, merge."""
    local = [capi.Counter(table_slots=slots) for _ in range(n_workers)]
    keep = []
    for d, text in enumerate(docs):
        t, n = to_dev(torch, text)
        keep.append(t)
        local[d % n_workers].count_dev(t.data_ptr(), n)
    owned = [capi.Counter(table_slots=slots) for _ in range(n_workers)]
    for j, c in enumerate(local):
        distinct = c.stats()[0]
        entries = torch.empty((max(distinct, 1), 4), dtype=torch.int64, device="cuda")
        counts = torch.zeros(n_workers + 1, dtype=torch.int64, device="cuda")
        c.partition(n_workers, entries.data_ptr(), entries.shape[0], counts.data_ptr())
        torch.cuda.synchronize()
        offs = np.concatenate([[0], np.cumsum(counts.cpu().numpy()[:n_workers])])
        nlong = c.long_records()
        assert nlong == int(counts[n_workers])
        rec = torch.empty(max(nlong, 8), dtype=torch.uint8, device="cuda")
        if nlong:
            c.long_records(rec.data_ptr(), nlong)
        for p in range(n_workers):   # the "all-to-all": region p of worker j goes to owner p
            cnt = int(offs[p + 1] - offs[p])
            if cnt:
                owned[p].merge_entries(entries[int(offs[p]):].data_ptr(), cnt)
            if nlong:
                owned[p].merge_long_records(rec.data_ptr(), nlong, p, n_workers)
    torch.cuda.synchronize()
    return [o.to_dict() for o in owned]


@pytest.mark.parametrize("n_workers", [1, 2, 3, 5, 8])
def test_shards_are_disjoint_and_merge_to_the_serial_count(capi, cuda, port, n_workers):
    rng = random.Random(1001 + n_workers)
    docs = [random_text(rng, rng.randint(1, 3000), rng.choice(["ascii", "unicode", "long"])) for _ in range(40)]
    shards = run_workers(capi, cuda, docs, n_workers)
    merged = {}
    for j, s in enumerate(shards):
        for w, c in s.items():
            assert w not in merged, "a word is held by two shards (count_unreduced_words must be 0)"
            assert capi.owner_of(w, n_workers) == j
            merged[w] = c
    assert merged == port.wordcount(docs)


def test_more_workers_than_documents(capi, cuda, port):
    # proj/tests/pipeline_test.cpp:129-135
    docs = [b"a b c", b"c d", b"e"]
    shards = run_workers(capi, cuda, docs, 8)
    assert len(shards) == 8
    merged = {}
    for s in shards:
        merged.update(s)
    assert merged == port.wordcount(docs)


def test_document_order_independence(capi, cuda, port):
    # proj/tests/pipeline_test.cpp:106-114
    rng = random.Random(303)
    docs = [random_text(rng, 800, "ascii") for _ in range(17)]
    want = port.wordcount(docs)
    for _ in range(3):
        rng.shuffle(docs)
        merged = {}
        for s in run_workers(capi, cuda, docs, 4):
            merged.update(s)
        assert merged == want


def test_device_ops_single_rank_path(capi, cuda, port):
    """exchange.hash_partition_merge with world size 1 (no collective): local -> owned"""
    import torch.distributed as dist

    from paper_2206_05269_b200.exchange import DeviceOps, hash_partition_merge

    class OneRank:   # the subset of torch.distributed the function touches at world size 1
        @staticmethod
        def get_world_size(group=None): return 1
        @staticmethod
        def get_rank(group=None): return 0
    text = random_text(random.Random(77), 50000, "unicode") + b" " + b"Q" * 40
    dev, n = to_dev(cuda, text)
    local, owned = capi.Counter(table_slots=1 << 15), capi.Counter(table_slots=1 << 15)
    local.count_dev(dev.data_ptr(), n)
    stats = hash_partition_merge(local, owned, DeviceOps(cuda, cuda.device("cuda", 0)), OneRank)
    assert owned.to_dict() == port.wordcount([text])
    assert stats.sent_entries == stats.received_entries


def test_bench_two_ranks_on_one_gpu(capi, cuda):
    """bench.py's N > 1 path (shard, count, partition, all-to-all, merge, e2e) with two ranks sharing
    the GPU over gloo; the merged table must equal a single-rank count of the same documents."""
    import json
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2", "--master-addr",
           "127.0.0.1", "--master-port", "29533", os.path.join(root, "bench.py"), "--gpus", "2", "--steps", "2",
           "--warmup", "1", "--docs", "6", "--backend", "gloo", "--no-mapreduce", "--e2e-steps", "1"]
    out = subprocess.run(cmd, capture_output=True, text=True, timeout=300, cwd=root)
    assert out.returncode == 0, out.stderr[-3000:]
    line = json.loads([l for l in out.stdout.splitlines() if l.startswith("{")][-1])
    assert line["n_gpus"] == 2 and line["config"]["documents"] == 12 and line["value"] > 0 and line["e2e"]["value"] > 0
    # the same 12 documents counted by one rank
    corpus = capi.synth_corpus(1, 0, 12, 50000)
    dev, n = to_dev(cuda, corpus)
    c = capi.Counter(table_slots=1 << 18)
    c.count_dev(dev.data_ptr(), n)
    distinct, tokens, _ = c.stats()
    assert line["config"]["distinct_words"] == distinct and line["config"]["tokens"] == tokens


def test_nccl_collective_path_with_one_rank(capi, cuda, port):
    """the exact NCCL calls of the multi-GPU merge (all_to_all_single with split sizes on int64
    entry tensors, all_reduce, all_gather) driven through a 1-rank NCCL group on this GPU"""
    import os
    import subprocess
    import sys
    import textwrap
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    code = textwrap.dedent("""
        import os, sys, random
        sys.path.insert(0, %r); sys.path.insert(0, os.path.join(%r, "tests"))
        import torch, torch.distributed as dist
        from helpers import random_text, to_dev
        from paper_2206_05269_b200 import capi
        from paper_2206_05269_b200.exchange import DeviceOps, hash_partition_merge, allreduce_scalar
        import oracle
        torch.cuda.set_device(0)
        dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
        text = random_text(random.Random(5), 60000, "unicode") + b" " + b"Z" * 33 + b" " + random_text(random.Random(6), 60000, "ascii")
        dev, n = to_dev(torch, text)
        local, owned = capi.Counter(table_slots=1 << 15), capi.Counter(table_slots=1 << 15)
        local.count_dev(dev.data_ptr(), n)
        st = hash_partition_merge(local, owned, DeviceOps(torch, torch.device("cuda", 0)), dist, force_collectives=True)
        torch.cuda.synchronize()
        assert owned.to_dict() == oracle.port().wordcount([text])
        # the synchronisation-free form: long tokens raise the sticky flag ...
        from paper_2206_05269_b200.exchange import AsyncExchange, ExchangeOverflow
        ops = DeviceOps(torch, torch.device("cuda", 0))
        ax = AsyncExchange(local, ops, dist)
        own2 = capi.Counter(table_slots=1 << 15)
        ax.step(local, own2)
        try:
            ax.finish(); raise SystemExit("long tokens were not reported")
        except ExchangeOverflow:
            pass
        # ... a corpus without them merges exactly, twice, with one finish() ...
        text2 = capi.synth_corpus(seed=8, doc_begin=0, doc_end=2, vocab=5000, doc_bytes=1 << 16).tobytes()   # words of <= 8 bytes
        dev2, n2 = to_dev(torch, text2)
        loc2 = capi.Counter(table_slots=1 << 15)
        loc2.count_dev(dev2.data_ptr(), n2)
        want2 = oracle.port().wordcount([text2])
        ax2 = AsyncExchange(loc2, ops, dist, entries_hint=len(want2))
        for _ in range(2):
            own3 = capi.Counter(table_slots=1 << 15)
            ax2.step(loc2, own3)
            assert own3.to_dict() == want2
        ax2.finish()
        # ... the same with the exchange on a second stream (overlap=True): four steps, two owned tables alternating,
        # the caller's stream runs ahead (reset + count of the next step) and only finish() joins the streams
        ax4 = AsyncExchange(loc2, ops, dist, entries_hint=len(want2), overlap=True)
        assert ax4.overlap
        pair = [capi.Counter(table_slots=1 << 15), capi.Counter(table_slots=1 << 15)]
        s = ops.stream()
        for k in range(4):
            loc2.reset(s); loc2.count_dev(dev2.data_ptr(), n2, s)
            ax4.slot_ready()
            pair[k & 1].reset(s)
            ax4.step(loc2, pair[k & 1])
        ax4.finish()
        torch.cuda.synchronize()
        assert pair[0].to_dict() == want2 and pair[1].to_dict() == want2
        # ... and regions that are too small are reported, not silently truncated
        ax3 = AsyncExchange(loc2, ops, dist, entries_hint=1)
        ax3.cap = 8
        ax3.step(loc2, capi.Counter(table_slots=1 << 15))
        try:
            ax3.finish(); raise SystemExit("overflow was not reported")
        except ExchangeOverflow:
            pass
        x = torch.tensor([1.25], dtype=torch.float64, device="cuda")
        assert float(allreduce_scalar(x, dist)) == 1.25 and float(allreduce_scalar(x, dist, reproducible=False)) == 1.25
        dist.destroy_process_group()
        print("nccl path ok", st.sent_entries, st.long_bytes)
    """ % (root, root))
    env = dict(os.environ, MASTER_ADDR="127.0.0.1", MASTER_PORT="29544")
    out = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, timeout=300, env=env)
    assert out.returncode == 0 and "nccl path ok" in out.stdout, out.stderr[-3000:]


@pytest.mark.parametrize("n_workers", [1, 2, 3, 8])
def test_wordcount_multi_entry(capi, cuda, port, n_workers):
    """wfcu_wordcount_multi: n workers (threads) mapped round-robin onto the visible GPUs, documents d mod n, regions
    delivered device to device; the union of the owner tables == serial_wordcount, no key has two holders, and every
    key sits on the worker its owner hash names."""
    import random
    from helpers import random_text
    rng = random.Random(n_workers)
    docs = [capi.synth_corpus(seed=4, doc_begin=d, doc_end=d + 1, vocab=50000, doc_bytes=1 << 17).tobytes() for d in range(5)]
    docs.append(random_text(rng, 40000, "unicode") + b" " + b"Z" * 70 + b" zz")
    docs.append(b"")
    docs.append((b"y" * 33 + b" ") * 9)
    shards, ns = capi.wordcount_multi(docs, n_workers, table_slots=1 << 16)
    assert len(shards) == n_workers
    tables = [s.to_dict() for s in shards]
    union = {}
    for j, t in enumerate(tables):
        for w, c in t.items():
            assert w not in union
            union[w] = c
            if len(w) <= 16:
                assert capi.owner_of(w, n_workers) == j
    assert union == port.wordcount(docs)
    assert ns["map_ns"] > 0 and ns["total_ns"] >= ns["map_ns"] and ns["sort_ns"] == 0 and ns["repair_ns"] == 0
    assert sum(s.stats()[1] for s in shards) == sum(union.values())


def test_wordcount_multi_rejects_bad_arguments(capi, cuda):
    with pytest.raises(capi.InvalidArgument):
        capi.wordcount_multi([b"a b"], 0)
    shards, _ = capi.wordcount_multi([], 3)
    assert [s.to_dict() for s in shards] == [{}, {}, {}]


@pytest.mark.parametrize("n_parts", [1, 2, 5])
def test_framed_regions_describe_themselves(capi, cuda, port, n_parts):
    """wfcu_counter_partition_framed: entry 0 of every region is its header; merge_regions with no counts array reads
    it -- the union of the regions is the table, every entry sits in its owner's region, overflow raises the flag"""
    text = capi.synth_corpus(seed=8, doc_begin=0, doc_end=1, vocab=50000, doc_bytes=1 << 18).tobytes() + b" " + b"x" * 30
    dev, n = to_dev(cuda, text)
    c = capi.Counter(table_slots=1 << 16)
    c.count_dev(dev.data_ptr(), n)
    want = {w: v for w, v in port.wordcount([text]).items() if len(w) <= 16}
    cap = len(want) + 2
    entries = cuda.zeros((n_parts * cap, 4), dtype=cuda.int64, device="cuda")
    counts = cuda.zeros(n_parts + 2, dtype=cuda.int64, device="cuda")
    c.partition_framed(n_parts, entries.data_ptr(), cap, counts.data_ptr())
    host = entries.cpu().numpy().reshape(n_parts, cap, 4)
    assert counts[n_parts].item() == 1 and counts[n_parts + 1].item() == 0          # one long token, no overflow
    assert [int(host[p, 0, 2]) for p in range(n_parts)] == counts[:n_parts].tolist()
    assert all(int(host[p, 0, 0]) == 0 and int(host[p, 0, 1]) == 0 for p in range(n_parts))
    merged = capi.Counter(table_slots=1 << 16)
    merged.merge_regions(entries.data_ptr(), n_parts, cap, 0)
    assert merged.to_dict() == want
    # a capacity of 3 entries per region overflows: the sticky flag counts what did not fit
    small = cuda.zeros((n_parts * 4, 4), dtype=cuda.int64, device="cuda")
    c.partition_framed(n_parts, small.data_ptr(), 4, counts.data_ptr())
    assert counts[n_parts + 1].item() == len(want) - sum(min(int(v), 3) for v in counts[:n_parts].tolist())
    assert [int(v) for v in small.cpu().numpy().reshape(n_parts, 4, 4)[:, 0, 2]] == [min(int(v), 3) for v in counts[:n_parts].tolist()]


def test_frame_codec_on_the_device(capi, cuda, port):
    """wfcu_tokens_encode_frame / decode_frame: the reference's golden bytes (proj/tests/wire_test.cpp:38-50), the
    round trip of sorted slices with long tokens, and every WireError kind (wire_test.cpp:72-118) as its own code"""
    import numpy as np
    t = capi.Tokens.from_words([b"to", b"a"])
    buf = cuda.zeros(256, dtype=cuda.uint8, device="cuda")
    n = t.encode_frame(0, 2, buf.data_ptr(), 256)
    assert bytes(buf[:n].cpu().numpy()) == bytes([0x57, 0x43, 0x58, 0x31, 2, 0, 0, 0, 2, 0, 0, 0, 1, 0, 0, 0, 0x74, 0x6F, 0x61])
    assert t.frame_bytes(0, 2) == n == 19
    n1 = t.encode_frame(1, 2, buf.data_ptr(), 256)
    assert bytes(buf[:n1].cpu().numpy()) == bytes([0x57, 0x43, 0x58, 0x31, 1, 0, 0, 0, 1, 0, 0, 0, 0x61])
    n0 = t.encode_frame(1, 1, buf.data_ptr(), 256)
    assert bytes(buf[:n0].cpu().numpy()) == bytes([0x57, 0x43, 0x58, 0x31, 0, 0, 0, 0])
    assert capi.Tokens.decode_frame(buf.data_ptr(), n0).words() == []
    words = sorted([b"alpha", b"b", "café".encode(), b"L" * 17, b"M" * 40, "한국어".encode(), b"zz"] * 3)
    big = capi.Tokens.from_words(words)
    fb = cuda.zeros(4096, dtype=cuda.uint8, device="cuda")
    m = big.encode_frame(2, len(words) - 1, fb.data_ptr(), 4096)
    back = capi.Tokens.decode_frame(fb.data_ptr(), m)
    assert back.words() == words[2:-1]
    back.sort()
    c = capi.Counter(table_slots=1 << 10)
    back.reduce_sorted(c)
    assert c.to_dict() == {w: words[2:-1].count(w) for w in set(words[2:-1])}

    def decode(raw: bytes):
        dev = cuda.zeros(max(len(raw), 4) + 16, dtype=cuda.uint8, device="cuda")
        if raw:
            dev[:len(raw)] = cuda.from_numpy(np.frombuffer(raw, dtype=np.uint8).copy()).cuda()
        return capi.Tokens.decode_frame(dev.data_ptr(), len(raw))
    good = bytes(fb[:m].cpu().numpy())
    for raw, code in ((b"WCX2" + good[4:], capi.ERR_FRAME_MAGIC), (b"WC", capi.ERR_FRAME_MAGIC), (good[:6], capi.ERR_FRAME_TRUNCATED),
                      (good[:12], capi.ERR_FRAME_TRUNCATED), (good[:-1], capi.ERR_FRAME_TRUNCATED), (good + b"x", capi.ERR_FRAME_TRAILING),
                      (b"WCX1" + bytes([1, 0, 0, 0, 2, 0, 0, 0, 0xC3, 0x28]), capi.ERR_FRAME_ENCODING),
                      (b"WCX1" + bytes([2, 0, 0, 0, 1, 0, 0, 0, 1, 0, 0, 0, 0xC3, 0xA9]), capi.ERR_FRAME_ENCODING)):
        with pytest.raises(capi.WfcuError) as e:
            decode(raw)
        assert e.value.code == code, (raw, e.value.code)
    with pytest.raises(capi.InvalidArgument):
        t.encode_frame(0, 3, buf.data_ptr(), 256)
    with pytest.raises(capi.WfcuError) as e:
        t.encode_frame(0, 2, buf.data_ptr(), 8)
    assert e.value.code == capi.ERR_BUFFER_TOO_SMALL


@pytest.mark.parametrize("world", [1, 2, 3])
def test_range_exchange_with_frames(capi, cuda, port, world):
    """exchange.range_partition_exchange: `world` ranks (sharing this GPU, gloo) run the paper's range exchange with
    device WCX1 frames; the shards they print are the reference's pre-repair shards (reduce_sorted of the exchanged
    chunks, proj/src/pipeline.cpp:104-114): their merge is serial_wordcount, each is a contiguous alphabetical range,
    and the sizes follow plan_partition."""
    import json
    import os
    import subprocess
    import sys
    sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
    import range_exchange_worker as rw
    from paper_2206_05269_b200.exchange import partition_cuts
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", str(world), "--master-addr",
           "127.0.0.1", "--master-port", str(29540 + world), os.path.join(root, "tests", "range_exchange_worker.py")]
    out = subprocess.run(cmd, capture_output=True, text=True, timeout=600, cwd=root)
    assert out.returncode == 0, out.stdout[-2000:] + out.stderr[-3000:]
    shards = sorted((json.loads(l[6:]) for l in out.stdout.splitlines() if l.startswith("SHARD ")), key=lambda s: s["rank"])
    assert [s["rank"] for s in shards] == list(range(world)) and all(s["sorted"] for s in shards)
    docs = rw.corpus()
    # the oracle's version of the same pipeline: tokenize per worker, sort, cut, gather, reduce
    locals_ = [sorted(w for d in range(j, len(docs), world) for w in port.tokenize(docs[d])) for j in range(world)]
    cuts = [partition_cuts(len(locals_[j]), j, world) for j in range(world)]
    merged = {}
    for c in range(world):
        want = {}
        for j in range(world):
            for w in locals_[j][cuts[j][c]:cuts[j][c + 1]]:
                want[w] = want.get(w, 0) + 1
        got = {bytes.fromhex(k): v for k, v in shards[c]["table"].items()}
        assert got == want
        assert shards[c]["n"] == sum(cuts[j][c + 1] - cuts[j][c] for j in range(world))
        for w, v in got.items():
            merged[w] = merged.get(w, 0) + v
    assert merged == port.wordcount(docs)


def test_repeated_long_record_merges_do_not_leak_the_arena(capi, cuda):
    """merging the same long-token record stream again and again only adds counts: the arena of the receiving table
    stays at one record per distinct token (it used to spend a record per incoming token until ARENA_FULL)"""
    text = (b"L" * 300 + b" " + b"M" * 200 + b" ") * 4
    dev, n = to_dev(cuda, text)
    src = capi.Counter(table_slots=1 << 10)
    src.count_dev(dev.data_ptr(), n)
    nlong = src.long_records()
    rec = cuda.empty(nlong, dtype=cuda.uint8, device="cuda")
    src.long_records(rec.data_ptr(), nlong)
    dst = capi.Counter(table_slots=1 << 10, arena_bytes=4096)      # room for a handful of records only
    for _ in range(200):
        dst.merge_long_records(rec.data_ptr(), nlong, 0, 1)
    dst.status()
    assert dst.to_dict() == {b"l" * 300: 800, b"m" * 200: 800}
