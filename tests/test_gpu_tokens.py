"""GPU parity: stand-alone tokenizer, sort_words and reduce_sorted vs the oracle.

reference: tokenize proj/src/text.cpp:32-57, sort_words :59-63, reduce_sorted
proj/src/reduce.cpp:8-21 (goldens: proj/tests/text_test.cpp:94-169, reduce_test.cpp:28-58)
"""
import random

import pytest

from helpers import random_text, to_dev

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("text", [
    b"I want to test MapReduce",
    b"MapReduce is a cool algorithm to test.",
    b"",
    b"--- a !!! b ...",
    "a b c one\ttwo\nthree".encode(),
    b"Dog dog. DOG!",
    b"x" * 40 + b" y " + b"Z" * 17 + b" " + b"z" * 16,
])
def test_tokenize_goldens(capi, cuda, port, text):
    toks = capi.Tokens.tokenize_host(text)
    assert toks.words() == port.tokenize(text)


@pytest.mark.parametrize("flavour", ["ascii", "long", "unicode"])
@pytest.mark.parametrize("size", [1, 17, 513, 5000, 200003])
def test_tokenize_matches_oracle_in_text_order(capi, cuda, port, flavour, size):
    text = random_text(random.Random(size + len(flavour)), size, flavour)
    toks = capi.Tokens.tokenize_host(text)
    want = port.tokenize(text)
    assert toks.stats()[0] == len(want)
    assert toks.words() == want


def test_sort_words_goldens(capi, cuda):
    # proj/tests/text_test.cpp:143-154
    t = capi.Tokens.from_words([b"i", b"want", b"to", b"test", b"mapreduce"])
    t.sort()
    assert t.words() == [b"i", b"mapreduce", b"test", b"to", b"want"]
    t = capi.Tokens.from_words([b"mapreduce", b"is", b"a", b"cool", b"algorithm", b"to", b"test"])
    t.sort()
    assert t.words() == [b"a", b"algorithm", b"cool", b"is", b"mapreduce", b"test", b"to"]
    e = capi.Tokens.from_words([])
    e.sort()
    assert e.words() == []


@pytest.mark.parametrize("flavour", ["ascii", "long", "unicode"])
def test_sort_words_matches_oracle(capi, cuda, port, flavour):
    text = random_text(random.Random(5), 60000, flavour)
    words = port.tokenize(text)
    # long tokens sharing a 16-byte prefix, a 16-byte token equal to that prefix, NULs inside
    words += [b"p" * 16 + b"zz", b"p" * 16, b"p" * 16 + b"a", b"p" * 16 + b"zz", b"p" * 17, b"a\x00b", b"a", b"a\x00"[:1]]
    t = capi.Tokens.from_words(words)
    t.sort()
    assert t.words() == port.sort_words(words) == sorted(words)


def test_reduce_sorted_goldens(capi, cuda, port):
    # proj/tests/reduce_test.cpp:28-43
    t = capi.Tokens.from_words([b"a", b"algorithm", b"cool", b"i", b"is", b"mapreduce"])
    c = capi.Counter(table_slots=1024)
    t.reduce_sorted(c)
    assert c.to_dict() == {b"a": 1, b"algorithm": 1, b"cool": 1, b"i": 1, b"is": 1, b"mapreduce": 1}
    t = capi.Tokens.from_words([b"mapreduce", b"test", b"test", b"to", b"to", b"want"])
    c = capi.Counter(table_slots=1024)
    t.reduce_sorted(c)
    assert c.to_dict() == {b"mapreduce": 1, b"test": 2, b"to": 2, b"want": 1}
    # unsorted input is rejected like the reference's std::invalid_argument (reduce.cpp:9)
    bad = capi.Tokens.from_words([b"b", b"a"])
    with pytest.raises(capi.InvalidArgument):
        bad.reduce_sorted(capi.Counter(table_slots=1024))
    empty = capi.Tokens.from_words([])
    c = capi.Counter(table_slots=1024)
    empty.reduce_sorted(c)
    assert c.to_dict() == {}


@pytest.mark.parametrize("flavour", ["ascii", "long", "unicode"])
def test_sort_then_rle_equals_hash_count(capi, cuda, port, flavour):
    """the sort + RLE alternative and the hash-count path give the same table"""
    text = random_text(random.Random(9), 150000, flavour)
    dev, n = to_dev(cuda, text)
    a = capi.Counter(table_slots=1 << 16)
    a.count_dev_sorted(dev.data_ptr(), n)
    want = port.wordcount([text])
    assert a.to_dict() == want
    assert a.stats()[1] == sum(want.values())
    toks = capi.Tokens.tokenize_dev(dev.data_ptr(), n)
    toks.sort()
    b = capi.Counter(table_slots=1 << 16)
    toks.reduce_sorted(b)
    assert b.to_dict() == want
    runs = port.reduce_sorted(port.sort_words(port.tokenize(text)))
    assert dict(runs) == want


def test_sorted_count_on_zipf_corpus(capi, cuda, port):
    corpus = capi.synth_corpus(seed=3, doc_begin=0, doc_end=8, vocab=50000)
    dev, n = to_dev(cuda, corpus)
    c = capi.Counter(table_slots=1 << 18)
    c.count_dev_sorted(dev.data_ptr(), n)
    assert c.to_dict() == port.wordcount([corpus])


def test_sorted_count_key_tiles(capi, cuda, port):
    """the counting form of the sort + RLE path takes short tokens straight from the tokenizer as 64-bit keys in
    tiles of 2048 that a warp owns: token-dense text overflows the first tile estimate (one retry), a single
    repeated word makes no byte position vary (the densifying pass still runs), empty and tiny inputs use no or
    one tile, and 9..16-byte / non-ASCII tokens keep the record path next to it"""
    rng = random.Random(77)
    dense = b" ".join(bytes([rng.choice(b"abcdefghijklmnopqrstuvwxyz0123456789")]) for _ in range(3_000_000))   # n/2 tokens
    same = b"word " * 700_000
    mixed = b" ".join(rng.choice([b"the", b"of", b"internationalisation", b"caf\xc3\xa9", b"x", b"encyclopaedia", b"Zebra"])
                      for _ in range(400_000))
    for text in (dense, same, mixed, b"", b"a", b"  ", b"abcdefgh abcdefghi"):
        dev, n = to_dev(cuda, text)
        c = capi.Counter(table_slots=1 << 14)
        c.count_dev_sorted(dev.data_ptr(), n)
        want = port.wordcount([text])
        assert c.to_dict() == want
        assert c.stats()[1] == sum(want.values())


def test_concat_slices_is_the_range_exchange(capi, cuda, port):
    """wfcu_tokens_concat_slices: chunk c of every worker's sorted list, gathered on the device, equals the
    reference's exchange output (proj/src/shuffle.cpp:98-130) once sorted; long tokens travel with their records."""
    import random
    rng = random.Random(3)
    n = 3
    vocab = [b"w%03d" % i for i in range(40)] + [b"L" * 20 + b"%d" % i for i in range(3)]
    lists = [sorted(rng.choice(vocab) for _ in range(rng.randrange(0, 90))) for _ in range(n)]
    handles = [capi.Tokens.from_words(l) for l in lists]
    for h in handles:
        h.sort()
    plans = [port.plan_partition(len(lists[j]), j, n) for j in range(n)]
    for c in range(n):
        got = capi.Tokens.concat_slices(handles, [plans[j][c] for j in range(n)], [plans[j][c + 1] for j in range(n)])
        want = [w for j in range(n) for w in lists[j][plans[j][c]:plans[j][c + 1]]]
        assert got.words() == want
        got.sort()
        assert got.words() == sorted(want)
    empty = capi.Tokens.concat_slices(handles, [0] * n, [0] * n)
    assert empty.words() == []
    with pytest.raises(capi.InvalidArgument):
        capi.Tokens.concat_slices(handles, [0] * n, [10 ** 6] * n)


def test_tokenize_arena_worst_case(capi, cuda, port):
    """long fragments full of invalid bytes: every byte becomes the three bytes of U+FFFD, so the long-token arena
    needs several times the text size (the retry used to stop at 3 n and fail with ARENA_FULL)"""
    text = (b"a" + b"\xff" * 5 + b"b ") * 40000
    want = port.tokenize(text)
    assert capi.Tokens.tokenize_host(text).words() == want
    assert len(want) == 40000 and len(want[0]) == 17


@pytest.mark.gpu
def test_sort_with_frequent_long_words(capi, cuda, port):
    """Words longer than 16 bytes are ordered by the radix sort itself (the length, then 8-byte windows behind the
    prefix), not by a serial fix-up: thousands of interleaved occurrences of long words that share 16, 24 or 40 bytes,
    one a prefix of the other, one with a NUL behind the common part, kilobyte words, and a few that agree beyond the
    32 KiB the windows cover (the insertion-sort safety net) --
    sort_words order, in well under the seconds the round-1 insertion sort took (87 s for 26 000 records)."""
    import time
    stem = b"abcdefghijklmnopqrstuvwx"                      # 24 bytes
    longs = [stem + b"yz", stem + b"ab", stem, stem[:20], stem + b"q" * 16 + b"1", stem + b"q" * 16 + b"0",
             stem + b"a\x00b", stem + b"a", b"k" * 1100 + b"b", b"k" * 1100 + b"a", b"k" * 1100]
    rng = random.Random(3)
    words = []
    for _ in range(6000):
        words.append(rng.choice(longs))
        words.extend(rng.choice([b"hello", b"world", b"abcdefghijklmnop", b"abcdefgh"]) for _ in range(3))
    words += [b"m" * 33000 + b"b", b"m" * 33000 + b"a", b"m" * 33000 + b"b", b"m" * 33000]
    text = b" ".join(words) + b" "
    tk = capi.Tokens.tokenize_host(text)
    assert tk.words() == port.tokenize(text)
    t0 = time.perf_counter()
    tk.sort()
    got = tk.words()
    assert time.perf_counter() - t0 < 5.0
    assert got == sorted(port.tokenize(text))
    c = capi.Counter(table_slots=1 << 12, arena_bytes=1 << 24)
    tk.reduce_sorted(c)
    assert c.to_dict() == port.wordcount([text])


@pytest.mark.gpu
def test_tokenize_docs_is_the_concatenation(capi, cuda, port):
    """wfcu_tokenize_docs_host: the tokens of several documents as one list, in document order -- no fragment spans
    a document boundary, empty documents and an empty list are fine"""
    rng = random.Random(11)
    docs = [random_text(rng, rng.randint(0, 4000), rng.choice(["ascii", "unicode", "long"])) for _ in range(9)]
    docs[3] = b""
    docs[5] = b"endswithoutspace"
    docs[6] = b"startsrightaway here"
    want = [w for d in docs for w in port.tokenize(d)]
    assert capi.Tokens.tokenize_docs_host(docs).words() == want
    assert capi.Tokens.tokenize_docs_host([]).words() == []
    assert capi.Tokens.tokenize_docs_host([b"", b""]).words() == []
