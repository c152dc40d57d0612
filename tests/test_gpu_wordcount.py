"""GPU parity: fused tokenizer + counting map vs the CPU oracle (bit-exact).

Every case goes through the C ABI (wfcu_counter_*), and the expected table is the
oracle's restatement of serial_wordcount (/root/reference/proj/src/pipeline.cpp:131-139).
"""
import random

import pytest

from helpers import gpu_wordcount, random_text, to_dev

pytestmark = pytest.mark.gpu

TWO_DOCS = [b"I want to test MapReduce", b"MapReduce is a cool algorithm to test."]


def test_two_document_example(capi, cuda, port):
    # golden: /root/reference/proj/tests/pipeline_test.cpp:35-44
    got, stats = gpu_wordcount(capi, cuda, TWO_DOCS)
    assert got == {b"a": 1, b"algorithm": 1, b"cool": 1, b"i": 1, b"is": 1, b"mapreduce": 2, b"test": 2, b"to": 2,
                   b"want": 1}
    assert stats[0] == 9 and stats[1] == 12


@pytest.mark.parametrize("text,tokens", [
    (b"Dog dog. DOG!", [b"dog"] * 3),                          # text_test.cpp:103-109
    (b"--- a !!! b ...", [b"a", b"b"]),                        # text_test.cpp:116-118
    (b"one\ttwo\nthree", [b"one", b"two", b"three"]),          # text_test.cpp:113
    ("a b c".encode(), [b"a", b"b", b"c"]),          # text_test.cpp:112 (NBSP, EM SPACE)
    (b"", []),
    (b"   \n\t ", []),
    (b"x", [b"x"]),
    (b"end.Start a--b (y)z US\x1fGS a\x00b don't RE-ELECT it's.",
     [b"end.start", b"a--b", b"y)z", b"us\x1fgs", b"a\x00b", b"don't", b"re-elect", b"it's"]),
    (b"a\xffb \xffab\xc3", [b"a\xef\xbf\xbdb", b"ab"]),
    ("café CAFÉ “word” word… —".encode(),
     ["café".encode()] * 2 + [b"word"] * 2),              # text_test.cpp:52-58
    (b"good \xff word", [b"good", b"word"]),                   # text_test.cpp:171-178
])
def test_tokenizer_goldens(capi, cuda, text, tokens):
    got, _ = gpu_wordcount(capi, cuda, [text])
    want = {}
    for t in tokens:
        want[t] = want.get(t, 0) + 1
    assert got == want


@pytest.mark.parametrize("flavour", ["ascii", "long", "unicode"])
@pytest.mark.parametrize("size", [1, 15, 16, 17, 31, 33, 511, 512, 513, 1024, 4096 + 7, 70001])
def test_random_text_matches_oracle(capi, cuda, port, flavour, size):
    rng = random.Random(size * 31 + len(flavour))
    for rep in range(3):
        text = random_text(rng, size, flavour)
        got, stats = gpu_wordcount(capi, cuda, [text])
        want = port.wordcount([text])
        assert got == want, (flavour, size, rep)
        assert stats[1] == sum(want.values())


def test_every_alignment_and_length(capi, cuda, port):
    """tokens of every length 1..40 at every offset mod 16, around row boundaries"""
    rng = random.Random(7)
    pieces = []
    for ln in range(1, 41):
        for off in range(16):
            word = bytes(rng.choice(b"abcXYZ09") for _ in range(ln))
            pieces.append(b" " * (1 + off) + rng.choice([b"", b"(", b"--"]) + word + rng.choice([b"", b".", b"!?"]))
    text = b"".join(pieces)
    for shift in (0, 1, 5, 497, 505):
        t = b"q" * shift + b" " + text
        got, _ = gpu_wordcount(capi, cuda, [t])
        assert got == port.wordcount([t]), shift


def test_long_fragments(capi, cuda, port):
    """fragments longer than a 16-byte chunk, a row and a warp strip (slow path)"""
    parts = [b"a" * 17, b"-" * 40 + b"mid" + b"." * 40, b"x" * 600, b"Y" * 5000, b"z" * 16, b"w" * 15,
             ("é" * 300).encode(), b"tail"]
    text = b" ".join(parts)
    got, _ = gpu_wordcount(capi, cuda, [text])
    assert got == port.wordcount([text])


def test_synthetic_zipf_corpus(capi, cuda, port):
    corpus = capi.synth_corpus(seed=1, doc_begin=0, doc_end=16, vocab=50000)   # 16 MiB, cfg3's generator
    dev, n = to_dev(cuda, corpus)
    counter = capi.Counter(table_slots=1 << 18)
    counter.count_dev(dev.data_ptr(), n)
    got = counter.to_dict()
    want = port.wordcount([corpus])
    assert got == want
    # accumulation over several calls == merge_counts
    counter.count_dev(dev.data_ptr(), n)
    assert counter.to_dict() == {k: 2 * v for k, v in want.items()}
    counter.reset()
    assert counter.to_dict() == {}


def test_export_is_in_map_order(capi, cuda, port):
    text = random_text(random.Random(3), 50000, "unicode") + b" " + random_text(random.Random(4), 50000, "long")
    dev, n = to_dev(cuda, text)
    counter = capi.Counter(table_slots=1 << 16)
    counter.count_dev(dev.data_ptr(), n)
    blob, lens, counts = counter.export()
    words = capi.unpack_words(blob, lens)
    assert words == sorted(words)
    pb, pl, pc = port.wordcount_packed([text])
    assert (blob == pb).all() and (lens == pl).all() and (counts == pc).all()


def test_count_host_matches_oracle(capi, cuda, port):
    rng = random.Random(11)
    docs = [random_text(rng, rng.randint(0, 3000), rng.choice(["ascii", "unicode", "long"])) for _ in range(200)]
    counter = capi.Counter(table_slots=1 << 16)
    counter.count_host(docs)
    assert counter.to_dict() == port.wordcount(docs)


def test_table_full_is_reported(capi, cuda):
    text = b" ".join(b"w%05d" % i for i in range(5000))
    dev, n = to_dev(cuda, text)
    counter = capi.Counter(table_slots=1024)
    counter.count_dev(dev.data_ptr(), n)
    with pytest.raises(capi.WfcuError) as e:
        counter.status()
    assert e.value.code == capi.ERR_TABLE_FULL


def test_merge_and_add_words(capi, cuda, port):
    a = random_text(random.Random(21), 20000, "ascii")
    b = random_text(random.Random(22), 20000, "unicode") + b" " + b"L" * 30 + b" " + b"L" * 30
    ca, cb = capi.Counter(table_slots=1 << 14), capi.Counter(table_slots=1 << 14)
    for c, t in ((ca, a), (cb, b)):
        dev, n = to_dev(cuda, t)
        c.count_dev(dev.data_ptr(), n)
    ca.merge(cb)
    want = port.wordcount([a, b])
    assert ca.to_dict() == want
    cc = capi.Counter(table_slots=1 << 14)
    cc.add_words(list(want), list(want.values()))
    assert cc.to_dict() == want


def test_count_host_zero_copy_path(capi, cuda, port):
    """adjacent whitespace-terminated documents in pinned memory are DMA'd without packing;
    the same bytes without the terminators take the packing path -- both equal the oracle"""
    import numpy as np
    corpus = capi.synth_corpus(seed=9, doc_begin=0, doc_end=40, vocab=50000, doc_bytes=1 << 16)
    pinned = cuda.from_numpy(corpus.copy()).pin_memory()
    arr = pinned.numpy()
    docs = [arr[i << 16:(i + 1) << 16] for i in range(40)]            # each ends with '\n'
    want = port.wordcount(docs)
    a = capi.Counter(table_slots=1 << 17)
    a.count_host(docs)
    assert a.to_dict() == want
    ragged = [arr[i << 16:((i + 1) << 16) - 1 - (i % 3)] for i in range(40)]   # views that drop the terminator
    b = capi.Counter(table_slots=1 << 17)
    b.count_host(ragged)
    assert b.to_dict() == port.wordcount(ragged)
    pageable = [corpus[i << 16:(i + 1) << 16] for i in range(40)]      # adjacent but not pinned
    c = capi.Counter(table_slots=1 << 17)
    c.count_host(pageable)
    assert c.to_dict() == want


def test_count_host_packing_slices(capi, cuda, port, monkeypatch):
    """pageable documents are packed into pinned staging by a pool of host threads in 256 KiB slices of the
    packed image: documents shorter, equal to and much longer than a slice, empty documents at slice edges,
    several staging chunks (the last word of a document must not join the first of the next)"""
    rng = random.Random(256)
    lens = [0, 1, (256 << 10) - 1, 0, 0, 256 << 10, 1, 0, (256 << 10) + 1, 700001, 5, 0, 2_500_000, 0, 3, 1 << 20, 0]
    docs = []
    for ln in lens:
        base = random_text(rng, min(ln, 70001), "ascii")
        t = bytearray((base * (ln // max(len(base), 1) + 1))[:ln])
        if ln:
            t[0] = ord("a")
            t[-1] = ord("z")          # word characters at both edges of every document
        docs.append(bytes(t))
    want = port.wordcount(docs)
    counter = capi.Counter(table_slots=1 << 18)
    counter.count_host(docs)
    got = counter.to_dict()
    assert got == want
    counter.reset()
    counter.count_host(capi.HostDocs(docs))
    assert counter.to_dict() == want


def test_export_into_caller_buffers(capi, cuda, port):
    """export(out=...) fills caller-owned (here page-locked, reused) arrays with the same three arrays"""
    import numpy as np
    text = random_text(random.Random(61), 60000, "ascii") + b" " + random_text(random.Random(62), 20000, "unicode")
    dev, n = to_dev(cuda, text)
    counter = capi.Counter(table_slots=1 << 15)
    counter.count_dev(dev.data_ptr(), n)
    blob, lens, counts = counter.export()
    rows, _, key_bytes = counter.stats()
    pinned = lambda dt, k: cuda.empty(k * np.dtype(dt).itemsize, dtype=cuda.uint8).pin_memory().numpy().view(dt)
    out = (pinned(np.uint8, key_bytes + 100), pinned(np.uint32, rows + 10), pinned(np.uint64, rows + 10))
    for _ in range(2):
        b2, l2, c2 = counter.export(out=out)
        assert bytes(b2) == bytes(blob) and (l2 == lens).all() and (c2 == counts).all()
    with pytest.raises(capi.WfcuError) as e:
        counter.export(out=(out[0][:key_bytes - 1], out[1], out[2]))
    assert e.value.code == capi.ERR_BUFFER_TOO_SMALL
    with pytest.raises(TypeError):
        counter.export(out=(out[0], out[1].view(np.int32), out[2]))


def test_deferred_list_overflow_is_reported(capi, cuda, port):
    """a corpus of words the fast path defers (three-byte characters) overflows a tiny slow-path list:
    loud error, and the same text counts exactly once the capacity is raised (what the C++ drop-in's
    retry does)"""
    text = (" ".join("h€llo%d" % (i % 50) for i in range(20000))).encode()
    dev, n = to_dev(cuda, text)
    small = capi.Counter(table_slots=1 << 12, deferred_slots=1024)
    small.count_dev(dev.data_ptr(), n)
    with pytest.raises(capi.WfcuError) as e:
        small.status()
    assert e.value.code == capi.ERR_DEFERRED_FULL
    big = capi.Counter(table_slots=1 << 12, deferred_slots=1 << 16)
    big.count_dev(dev.data_ptr(), n)
    assert big.to_dict() == port.wordcount([text])
