"""GPU: BASELINE.json config 5 at test scale -- four synthetic speaker corpora counted on
the device, pooled-others by device merge, per-speaker top-k and distinctive words; every
list must equal the oracle's exactly (words, counts, doubles).  Plus a >4 GiB offset check."""
import numpy as np
import pytest

from helpers import to_dev

pytestmark = pytest.mark.gpu


def test_four_speakers_top_k_and_distinctive(capi, cuda, port):
    speakers = [1, 2, 3, 4]
    texts = {s: capi.synth_corpus(seed=7, doc_begin=0, doc_end=2, vocab=50000, speaker=s, doc_bytes=1 << 19) for s in speakers}
    counters = {}
    for s in speakers:
        dev, n = to_dev(cuda, texts[s])
        c = capi.Counter(table_slots=1 << 17)
        c.count_dev(dev.data_ptr(), n)
        counters[s] = c
    cpu = {s: port.wordcount([texts[s]]) for s in speakers}
    for s in speakers:
        pooled = capi.Counter(table_slots=1 << 18)        # sum of the other three, on the device (cli.cpp:213-218)
        for o in speakers:
            if o != s:
                pooled.merge(counters[o])
        others_cpu = {}
        for o in speakers:
            if o != s:
                for k, v in cpu[o].items():
                    others_cpu[k] = others_cpu.get(k, 0) + v
        assert pooled.to_dict() == others_cpu
        assert capi.top_k(counters[s].export(), 25) == port.top_k(cpu[s], 25)
        got = capi.distinctive(counters[s].export(), pooled.export(), 25)
        assert got == port.distinctive(cpu[s], others_cpu, 25)
        assert any(w.endswith(str(s).encode()) for w, _ in got)      # the speaker's own words rank high


def test_offsets_beyond_4_gib(capi, cuda, port):
    """a 4.25 GiB device buffer (17 copies of a 256 MiB corpus): counts are 17x the base counts"""
    base = capi.synth_corpus(seed=5, doc_begin=0, doc_end=256, vocab=50000)
    dev = cuda.from_numpy(base).cuda()
    c = capi.Counter(table_slots=1 << 18)
    c.count_dev(dev.data_ptr(), dev.numel())
    one = c.to_dict()
    big = dev.repeat(17)
    assert big.numel() > (1 << 32)
    c.reset()
    c.count_dev(big.data_ptr(), big.numel())
    many = c.to_dict()
    assert many == {k: 17 * v for k, v in one.items()}
    assert c.stats()[1] == 17 * sum(one.values())
    sample = capi.synth_corpus(seed=5, doc_begin=0, doc_end=2, vocab=50000)   # anchor the base against the oracle
    dsm, n = to_dev(cuda, sample)
    c.reset()
    c.count_dev(dsm.data_ptr(), n)
    assert c.to_dict() == port.wordcount([sample])


@pytest.mark.parametrize("k", [0, 1, 5, 25, 1000, 10 ** 6])
def test_device_top_k_equals_reference_order(capi, cuda, port, k):
    """wfcu_counter_top_k (count order on the device, ties resolved exactly) == top_k over the export"""
    import random
    from helpers import random_text
    corpus = capi.synth_corpus(seed=11, doc_begin=0, doc_end=3, vocab=50000, doc_bytes=1 << 19).tobytes()
    extra = random_text(random.Random(2), 30000, "unicode") + b" " + (b"Q" * 40 + b" ") * 700 + b"zz " * 900
    text = corpus + b" " + extra
    dev, n = to_dev(cuda, text)
    c = capi.Counter(table_slots=1 << 17)
    c.count_dev(dev.data_ptr(), n)
    want = port.top_k(port.wordcount([text]), k)
    assert c.top_k(k) == want
    assert capi.top_k(c.export(), k) == want


@pytest.mark.parametrize("k", [0, 1, 25, 400, 10 ** 6])
def test_device_distinctive_equals_reference(capi, cuda, port, k):
    """wfcu_counter_distinctive (join + score + select on the device, exact ranking of the candidates) ==
    the reference order over the exported tables: words AND doubles, ties by word, words only the others hold."""
    import random
    from helpers import random_text
    t_text = (capi.synth_corpus(seed=3, doc_begin=0, doc_end=2, vocab=50000, speaker=1, doc_bytes=1 << 19).tobytes()
              + b" " + random_text(random.Random(5), 20000, "unicode") + b" " + (b"L" * 33 + b" ") * 50 + (b"onlyhere" * 3 + b" ") * 9)
    o_text = (capi.synth_corpus(seed=3, doc_begin=5, doc_end=8, vocab=50000, speaker=2, doc_bytes=1 << 19).tobytes()
              + b" " + (b"L" * 33 + b" ") * 7 + (b"M" * 40 + b" ") * 3)
    tc, oc = capi.Counter(table_slots=1 << 17), capi.Counter(table_slots=1 << 17)
    for c, text in ((tc, t_text), (oc, o_text)):
        dev, n = to_dev(cuda, text)
        c.count_dev(dev.data_ptr(), n)
    want = port.distinctive(port.wordcount([t_text]), port.wordcount([o_text]), k)
    assert tc.distinctive(oc, k) == want
    assert capi.distinctive(tc.export(), oc.export(), k) == want


def test_device_distinctive_small_and_empty(capi, cuda, port):
    a, b, e = capi.Counter(table_slots=1 << 10), capi.Counter(table_slots=1 << 10), capi.Counter(table_slots=1 << 10)
    a.add_words([b"x", b"y", b"zebra"], [3, 1, 1])
    b.add_words([b"y", b"w"], [5, 2])
    assert e.distinctive(e, 5) == []
    assert a.distinctive(e, 5) == port.distinctive({b"x": 3, b"y": 1, b"zebra": 1}, {}, 5)
    assert e.distinctive(b, 5) == port.distinctive({}, {b"y": 5, b"w": 2}, 5)
    assert a.distinctive(b, 10) == port.distinctive({b"x": 3, b"y": 1, b"zebra": 1}, {b"y": 5, b"w": 2}, 10)
    assert a.distinctive(a, 2) == port.distinctive({b"x": 3, b"y": 1, b"zebra": 1}, {b"x": 3, b"y": 1, b"zebra": 1}, 2)


def test_four_speakers_one_million_words_device_reports(capi, cuda, port):
    """config 5 with the 1 M-word vocabulary: per-speaker top-k and distinctive words straight from the device
    tables (wfcu_counter_top_k, wfcu_counter_merge, wfcu_counter_distinctive) == the oracle on the same bytes."""
    speakers = [1, 2, 3, 4]
    texts = {s: capi.synth_corpus(seed=9, doc_begin=0, doc_end=6, vocab=1000000, speaker=s) for s in speakers}
    counters, cpu = {}, {}
    for s in speakers:
        dev, n = to_dev(cuda, texts[s])
        counters[s] = capi.Counter(table_slots=1 << 20)
        counters[s].count_dev(dev.data_ptr(), n)
        cpu[s] = port.wordcount([texts[s]])
    for s in speakers:
        pooled = capi.Counter(table_slots=1 << 21)
        others_cpu = {}
        for o in speakers:
            if o != s:
                pooled.merge(counters[o])
                for w, v in cpu[o].items():
                    others_cpu[w] = others_cpu.get(w, 0) + v
        assert counters[s].top_k(25) == port.top_k(cpu[s], 25)
        assert counters[s].distinctive(pooled, 25) == port.distinctive(cpu[s], others_cpu, 25)
