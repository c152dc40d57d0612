"""CPU: the C-ABI library loads, exports every symbol include/wfcu.h declares, and its
host-side pieces (synthetic corpora, owner function, no-device behaviour) are right."""
import ctypes
import os
import re

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_symbols():
    text = open(os.path.join(ROOT, "include", "wfcu.h")).read()
    return sorted(set(re.findall(r"WFCU_API\s+[\w\s\*]+?\b(wfcu_\w+)\s*\(", text)))


def test_every_declared_symbol_is_exported(capi):
    names = declared_symbols()
    assert len(names) >= 40
    lib = ctypes.CDLL(str(capi.LIB_PATH))
    missing = [n for n in names if not hasattr(lib, n)]
    assert not missing, missing
    assert sorted(capi.SIGNATURES) == names        # the Python binding covers the whole header


def test_no_device_is_an_error_not_a_fallback(capi):
    if capi.device_count() > 0:
        pytest.skip("a GPU is visible here")
    with pytest.raises(capi.WfcuError) as e:
        capi.Counter()
    assert e.value.code == capi.ERR_NO_DEVICE
    with pytest.raises(capi.WfcuError) as e:
        capi.map_reduce_host(np.ones(4), capi.MAP_IDENTITY)
    assert e.value.code == capi.ERR_NO_DEVICE
    with pytest.raises(capi.WfcuError):
        capi.Tokens.tokenize_host(b"a b")


def test_synthetic_corpus_is_deterministic_and_per_document(capi):
    a = capi.synth_corpus(1, 0, 6, 50000, doc_bytes=8192)
    b = capi.synth_corpus(1, 0, 6, 50000, doc_bytes=8192, threads=1)
    assert (a == b).all()
    docs = a.reshape(6, 8192)
    for d in range(6):      # document d depends only on (seed, d)
        assert (capi.synth_corpus(1, d, d + 1, 50000, doc_bytes=8192) == docs[d]).all()
    assert (capi.synth_corpus_strided(1, 1, 2, 3, 50000, doc_bytes=8192).reshape(3, 8192) == docs[1::2]).all()
    assert not (capi.synth_corpus(2, 0, 1, 50000, doc_bytes=8192) == docs[0]).all()
    assert docs[:, -1].tolist() == [10] * 6                 # every document ends with '\n'
    assert set(np.unique(a).tolist()) <= set(b" \n.,;!?" + bytes(range(65, 91)) + bytes(range(97, 123)) + b"0123456789")


def test_synthetic_corpus_is_zipfian(capi, port):
    text = capi.synth_corpus(1, 0, 4, 50000)
    counts = port.wordcount([text])
    total = sum(counts.values())
    top = max(counts.values())
    assert 0.12 < top / total < 0.16          # Zipf(1.1) over 50k words: top word ~13.9 %
    assert 6.5 < text.size / total < 8.0      # ~7.3 bytes per token
    lens = {len(w) for w in counts}
    assert min(lens) >= 4 and max(lens) <= 8  # W=4 plus a 0..4 letter prefix
    sp = capi.synth_corpus(1, 0, 1, 50000, speaker=3)
    assert any(w.endswith(b"3") for w in port.wordcount([sp]))   # speaker-specific words


def test_owner_function_is_a_partition(capi):
    words = [b"w%05d" % i for i in range(2000)] + [b"x" * 17, b"y" * 40, "café".encode()]
    for n in (1, 2, 3, 8):
        owners = [capi.owner_of(w, n) for w in words]
        assert all(0 <= o < n for o in owners)
        if n > 1:
            hist = np.bincount(owners, minlength=n)
            assert hist.min() > len(words) / n * 0.7      # roughly balanced


def test_pack_unpack_roundtrip(capi):
    words = [b"a", b"", b"hello", bytes(range(256))]
    blob, lens = capi.pack_words(words)
    assert capi.unpack_words(blob, lens) == words


def test_host_docs_marshals_pointers_and_lengths(capi):
    """HostDocs is the (pointer, length) pair of arrays wfcu_counter_count_host takes; built once, reusable"""
    blob = np.frombuffer(b"alpha beta\ngamma\n\ndelta ", dtype=np.uint8).copy()
    views = [blob[0:11], blob[11:17], blob[17:18], blob[18:24], blob[24:24]]
    hd = capi.HostDocs(views + [b"tail bytes"])
    assert hd.n == 6
    base = blob.ctypes.data
    assert [hd.ptrs[i] for i in range(5)] == [base, base + 11, base + 17, base + 18, None]    # empty document: NULL
    assert [hd.lens[i] for i in range(6)] == [11, 6, 1, 6, 0, 10]
    assert ctypes.string_at(hd.ptrs[5], 10) == b"tail bytes"


def test_async_exchange_region_capacity():
    """the fixed region capacity: 2 x the uniform share of the hint (+ slack), never above what the table can hold,
    plus the header entry that makes a region self-describing"""
    from paper_2206_05269_b200.exchange import AsyncExchange

    class Table:
        def max_entries(self): return 524288

    class Torch:
        int64 = "i64"
        @staticmethod
        def zeros(n, dtype=None, device=None): return [0] * n

    class Ops:
        torch = Torch
        def empty_entries(self, n):
            class E:
                device = "cpu"
                rows = n
            return E()

    class Dist:
        def __init__(self, w): self.w = w
        def get_world_size(self, group=None): return self.w

    assert AsyncExchange(Table(), Ops(), Dist(8), entries_hint=50000).cap == 2 * 6250 + 1024 + 1
    assert AsyncExchange(Table(), Ops(), Dist(2), entries_hint=50000).cap == 2 * 25000 + 1024 + 1
    assert AsyncExchange(Table(), Ops(), Dist(4)).cap == 524288 + 1                 # no hint: cannot overflow
    assert AsyncExchange(Table(), Ops(), Dist(1), entries_hint=10 ** 9).cap == 524288 + 1
    assert AsyncExchange(Table(), Ops(), Dist(8), entries_hint=50000).send.rows == 8 * (2 * 6250 + 1024 + 1)


def test_async_exchange_overlap_protocol():
    """AsyncExchange(overlap=True) with recording stand-ins for the device steps: the collective and the merge of a step
    are issued on the second stream behind an event recorded after the partition; the two send buffers alternate; the
    partition that reuses a buffer first waits for the event of the merge that read it two steps earlier; slot_ready()
    waits for the same event before the caller resets the owned table; finish() joins the streams before reading the
    flags."""
    import contextlib
    from paper_2206_05269_b200.exchange import AsyncExchange

    log = []

    class Table:
        def __init__(self, name): self.name = name
        def max_entries(self): return 4096

    class Flags(list):
        def clone(self): return Flags(self)
        def cpu(self): return self
        def tolist(self): return list(self)
        def zero_(self):
            for i in range(len(self)): self[i] = 0

    class Counts:
        def __init__(self, n): self.v = Flags([0] * n)
        def __getitem__(self, s): return Flags(self.v[s]) if isinstance(s, slice) and s.stop is not None else self
        def zero_(self): self.v.zero_()

    class Torch:
        int64 = "i64"
        @staticmethod
        def zeros(n, dtype=None, device=None): return Counts(n)

    class Entries:
        device = "cpu"
        def __init__(self, name): self.name = name

    class Ops:
        torch = Torch
        def __init__(self): self.cur, self.n_buf, self.n_ev = "main", 0, 0
        def empty_entries(self, n):
            self.n_buf += 1
            return Entries(f"buf{self.n_buf}")
        def new_stream(self): return "comm"
        def record(self):
            self.n_ev += 1
            log.append(("record", self.cur, self.n_ev))
            return self.n_ev
        def wait(self, ev): log.append(("wait", self.cur, ev))
        @contextlib.contextmanager
        def on(self, stream):
            prev, self.cur = self.cur, stream
            try: yield
            finally: self.cur = prev
        def partition_framed(self, local, world, send, cap, counts): log.append(("partition", self.cur, send.name))
        def merge_regions(self, owned, recv, world, cap, counts): log.append(("merge", self.cur, owned.name))

    class Dist:
        def get_world_size(self, group=None): return 2
        def all_to_all_single(self, recv, send, group=None): log.append(("a2a", ops.cur, send.name))
        def all_reduce(self, t, group=None): log.append(("all_reduce", ops.cur))

    ops = Ops()
    ax = AsyncExchange(Table("local"), ops, Dist(), entries_hint=100, overlap=True)
    assert ax.overlap
    owned = [Table("own0"), Table("own1")]
    for k in range(4):
        ax.slot_ready()
        log.append(("reset", ops.cur, owned[k & 1].name))
        ax.step(Table("local"), owned[k & 1])
    ax.finish()
    sends = [e[2] for e in log if e[0] == "partition"]
    assert sends[0] != sends[1] and sends == [sends[0], sends[1]] * 2                 # two send buffers alternate
    assert all(e[1] == "comm" for e in log if e[0] in ("a2a", "merge"))               # collective + merge: second stream
    assert all(e[1] == "main" for e in log if e[0] in ("partition", "reset"))         # count side: the caller's stream
    # step k: partition, record(main)=r, [comm: wait(r), a2a, merge, record(comm)=m_k]
    merged_ev = [e[2] for e in log if e[0] == "record" and e[1] == "comm"]
    assert len(merged_ev) == 4
    for k in (2, 3):     # reuse of slot k & 1: both the reset of the owned table and the partition wait for m_{k-2} first
        start = [i for i, e in enumerate(log) if e[0] == "reset"][k]
        before = log[:start]
        assert ("wait", "main", merged_ev[k - 2]) in before[-3:]
        part = [i for i, e in enumerate(log) if e[0] == "partition"][k]
        assert ("wait", "main", merged_ev[k - 2]) in log[start:part]
    # finish(): the caller's stream waits for the last merge before the flags are reduced
    i_red = log.index(("all_reduce", "main"))
    assert ("wait", "main", merged_ev[-1]) in log[:i_red] and log.index(("wait", "main", merged_ev[-1])) > [i for i, e in enumerate(log) if e[0] == "merge"][-1]
