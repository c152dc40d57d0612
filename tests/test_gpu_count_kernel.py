"""GPU parity for the paths specific to the third-generation counting kernel (csrc/wc_count.cu):
1 KiB rows made of two interleaved 512-byte halves, the 32-byte guard in front of a ring slot,
the bit-parallel first/last-word-character emission and its end-by-end fallback, the 512-entry
token queue and the two-token passes.  Oracle: the C restatement of serial_wordcount
(/root/reference/proj/src/pipeline.cpp:131-139, text.cpp:9-57).  Bit-exact.
"""
import random

import pytest

from helpers import gpu_wordcount, random_text, to_dev

pytestmark = pytest.mark.gpu


def check(capi, cuda, port, text, **cfg):
    got, stats = gpu_wordcount(capi, cuda, [text], **cfg)
    want = port.wordcount([text])
    assert got == want
    assert stats[1] == sum(want.values())


@pytest.mark.parametrize("sep", [b" ", b"\n", b" \t"])
def test_dense_one_byte_tokens_overflow_the_queue(capi, cuda, port, sep):
    """'a b c ...': up to 512 fragment ends per 1 KiB row, more than the queue holds next to
    the leftovers of the previous row"""
    rng = random.Random(5)
    text = sep.join(bytes([rng.choice(b"abcdefghij0123XYZ")]) for _ in range(40000))
    check(capi, cuda, port, text)
    check(capi, cuda, port, b"x" * 700 + b" " + text)     # a deferred fragment in front


@pytest.mark.parametrize("shift", [0, 1, 15, 16, 17, 495, 496, 497, 511, 512, 513, 1007, 1008, 1009, 1023, 1024, 1025])
def test_tokens_across_half_and_row_boundaries(capi, cuda, port, shift):
    """tokens of length 1..18 (with and without edge punctuation) placed so that they straddle the
    16-byte chunks, the 512-byte halves and the 1 KiB rows of the kernel at every phase"""
    rng = random.Random(shift)
    parts = []
    for rep in range(6):
        for ln in range(1, 19):
            word = bytes(rng.choice(b"abcdefgXYZ0189") for _ in range(ln))
            parts.append(rng.choice([b"", b"(", b"\"'", b"--"]) + word + rng.choice([b"", b".", b",", b"!?)", b"..."]))
    rng.shuffle(parts)
    text = b"q" * shift + b" " + b" ".join(parts)
    check(capi, cuda, port, text)


def test_sixteen_byte_tokens_and_seventeen(capi, cuda, port):
    """16 bytes is the longest token the fast path keeps; 17 takes the row's end-by-end redo and
    the slow kernel.  Both next to the guard (row start) and in the middle of a row."""
    w16 = [b"abcdefghijklmnop", b"ABCDEFGHIJKLMNOP", b"a--------------b", b"0123456789abcdef"]
    w17 = [b"abcdefghijklmnopq", b"a---------------b"]
    rng = random.Random(16)
    for lead in (0, 3, 1008 - 17, 1024 - 16, 1024 - 8, 1024, 2048 - 1):
        parts = [b"z" * lead] if lead else []
        for _ in range(300):
            parts.append(rng.choice(w16 + w17 + [b"the", b"of", b"x"]) + rng.choice([b"", b".", b"--"]))
        check(capi, cuda, port, b" ".join(parts))


def test_fragment_with_one_word_character_at_its_start(capi, cuda, port):
    """'a---------------' (16 bytes, token 'a'): its ring position is the lowest a token can have"""
    text = b" ".join([b"a" + b"-" * 15, b"b" + b"." * 14, b"--c", b"d"] * 400)
    for lead in (0, 1, 15, 16, 1023):
        check(capi, cuda, port, b"k" * lead + (b" " if lead else b"") + text)


@pytest.mark.parametrize("vocab,docs", [(50000, 6), (1000000, 6)])
def test_synthetic_corpus_many_rows_per_warp(capi, cuda, port, vocab, docs):
    """6 MiB: every warp of the grid walks several rows, leftovers cross rows, 9-byte words
    (1M vocabulary) take the general passes"""
    corpus = capi.synth_corpus(seed=3, doc_begin=0, doc_end=docs, vocab=vocab)
    dev, n = to_dev(cuda, corpus)
    counter = capi.Counter(table_slots=1 << 21)
    counter.count_dev(dev.data_ptr(), n)
    assert counter.to_dict() == port.wordcount([corpus])


@pytest.mark.parametrize("size", [1023, 1024, 1025, 2047, 2048, 2049, 28 * 1024 - 1, 28 * 1024, 28 * 1024 + 1, 300007])
@pytest.mark.parametrize("flavour", ["ascii", "unicode"])
def test_sizes_around_row_multiples(capi, cuda, port, size, flavour):
    rng = random.Random(size ^ 0x55)
    check(capi, cuda, port, random_text(rng, size, flavour))
    check(capi, cuda, port, random_text(rng, size - 1, flavour) + b"z")      # last byte is a word character


def test_non_ascii_rows_between_ascii_rows(capi, cuda, port):
    """the carried >=0x80 mask: a non-ASCII byte in the last chunk of a row, the fragment ends in the next"""
    rng = random.Random(77)
    base = bytearray(random_text(rng, 8192, "ascii"))
    for pos in (1023, 1022, 1008, 2047, 511, 512, 3071, 4095):
        t = bytearray(base)
        t[pos - 1:pos + 1] = "é".encode()
        t[pos + 1] = ord("x")
        check(capi, cuda, port, bytes(t))


# ---- two-byte letters on the fast path (the HI variant of the kernel) ---------------------------
LATIN = ["é", "É", "à", "À", "ü", "Ü", "ß", "ÿ", "Þ", "þ", "ñ", "Ñ", "ç", "Ç", "ø", "Ø", "×", "÷", "µ", "ª", "¿",
         " ", "ō", "Ł", "ł", "Ω", "ω", "я", "Я", "ж", "Ж", "א", "߿", "€", "“", "”", "あ"]


def latin_text(rng, n):
    """dense in two-byte characters: words of ASCII letters and LATIN characters, some upper case, with
    edge punctuation; a few invalid bytes (a lead without its continuation byte, a stray continuation)"""
    out = bytearray()
    while len(out) < n:
        r = rng.random()
        if r < 0.17:
            out += rng.choice([b" ", b"\n", b"  ", b"\t"])
        elif r < 0.24:
            out += bytes([rng.choice(b".,;!?-'\"()")])
        elif r < 0.50:
            out += rng.choice(LATIN).encode()
        elif r < 0.52:
            out += bytes([rng.choice([0xC3, 0xC4, 0xD0, 0xDF, 0x80, 0xA9, 0xBF, 0xC2, 0xC0, 0xE0, 0xFF])])
        else:
            out += bytes([rng.choice(b"abcdefghijklmnopqrstuvwxyzABCDEFGHIJKLMNOPQRSTUVWXYZ0123456789")])
    return bytes(out[:n])


@pytest.mark.parametrize("size", [1, 2, 15, 16, 17, 33, 511, 513, 1023, 1024, 1025, 2049, 30011, 400003])
def test_two_byte_letters_match_oracle(capi, cuda, port, size):
    rng = random.Random(size * 7 + 1)
    for rep in range(3):
        check(capi, cuda, port, latin_text(rng, size))


def test_two_byte_case_fold_and_edges(capi, cuda, port):
    """golden-style cases (proj/src/unicode.cpp:117-121: U+00C0..U+00DE except U+00D7 fold by +0x20, nothing
    else above ASCII folds; U+00D7 / U+00F7 are not word characters) repeated so that the CTA sampler
    picks the two-byte variant"""
    unit = ("École ÉCOLE école Ærø ÆRØ STRASSE straße Ÿ ÿ ÞORN þorn 3×4 ×× a÷b ÷ "
            "Ωμέγα ΩΜΈΓΑ Жук жук ŁÓDŹ łódź don't’ “quoted” naïve. (café) —señor— ").encode()
    text = unit * 300
    got, _ = gpu_wordcount(capi, cuda, [text])
    assert got == port.wordcount([text])
    assert got["école".encode()] == 900 and got["strasse".encode()] == 300 and got["straße".encode()] == 300
    assert got["3×4".encode()] == 300 and got["a÷b".encode()] == 300          # interior x / division sign stay
    assert "××".encode() not in got and "÷".encode() not in got
    assert got["ærø".encode()] == 600 and got["þorn".encode()] == 600 and got["ÿ".encode()] == 300 and got["Ÿ".encode()] == 300
    assert got["Ωμέγα".encode()] == 300 and got["ΩΜΈΓΑ".encode()] == 300    # Greek does not fold
    assert got["łódź".encode()] == 300 and got["ŁódŹ".encode()] == 300       # only the Latin-1 letters fold
    assert got["don't".encode()] == 300 and got["quoted".encode()] == 300 and got["señor".encode()] == 300


@pytest.mark.parametrize("shift", [0, 1, 14, 15, 16, 17, 510, 511, 512, 513, 1022, 1023, 1024, 1025])
def test_two_byte_sequences_across_chunk_half_and_row_boundaries(capi, cuda, port, shift):
    """a lead byte as the last byte of a 16-byte chunk / a half / a row, with and without its continuation
    byte behind the boundary; also the end of the text right after a lead"""
    rng = random.Random(shift + 99)
    body = " ".join("".join(rng.choice(["é", "É", "a", "B", "ü", "Ж", "ß", "x"]) for _ in range(rng.randint(1, 7)))
                    for _ in range(400)).encode()
    for tail in (b"", b"\xc3", b"\xc3 z", b" \xd0", b"\xa9", b"\xc3\xc3\xa9"):
        text = b"q" * shift + b" " + body + tail
        check(capi, cuda, port, text)
        for cut in (1, 2, 3):
            check(capi, cuda, port, text[:len(text) - cut])


def test_typographic_punctuation_stays_inside_tokens(capi, cuda, port):
    """U+2010..U+2027 / U+2030..U+203F (E2 80 xx) are punctuation: kept inside a token, trimmed at its edges,
    never whitespace; their neighbours in the block that ARE whitespace (U+2009, U+2028, U+202F) split"""
    unit = ("don’t “quoted” well—known… it’s ‘single’ a‐b x†y 5‰ rock’n’roll ’tis end’ "
            "thin space para sep nnbsp zero​width bidi‪x €5 ").encode()
    text = unit * 400
    got, _ = gpu_wordcount(capi, cuda, [text])
    assert got == port.wordcount([text])
    assert got["don’t".encode()] == 400 and got["quoted".encode()] == 400 and got["well—known".encode()] == 400
    assert got["rock’n’roll".encode()] == 400 and got["tis".encode()] == 400 and got["end".encode()] == 400
    assert got["thin".encode()] == 400 and got["space".encode()] == 400 and got["nnbsp".encode()] == 400


@pytest.mark.parametrize("shift", [0, 13, 14, 15, 16, 509, 510, 511, 512, 1021, 1022, 1023, 1024])
def test_three_byte_punctuation_across_boundaries(capi, cuda, port, shift):
    """E2 | 80 | xx split over 16-byte chunks, halves and rows in every way, complete and truncated"""
    rng = random.Random(shift + 5)
    body = " ".join("".join(rng.choice(["a", "B", "’", "—", "…", "é", "x", "“"]) for _ in range(rng.randint(1, 6)))
                    for _ in range(500)).encode()
    for tail in (b"", b"\xe2", b"\xe2\x80", b"\xe2\x80\x99", b"\xe2\x80 z", b"\xe2\x80\x80", b"\xe2\x81\x99", b"\x80\x99"):
        text = b"q" * shift + b" " + body + tail
        check(capi, cuda, port, text)
        check(capi, cuda, port, text[:len(text) - 1])


# ---- three-byte letters on the fast path (round 2) -------------------------------------------------
THREE = ["한", "국", "어", "는", "हि", "न्", "दी", "あ", "カ", "漢", "字", "ế", "ộ", "ữ", "ქ", "ა", "ἀ", "ᚠ",           # letters (ᚠ: E1 9A A0, its block defers)
         "　", "、", "。", " ", "‐", "’", "…", "！", "ａ", "�", "ࠀ", "퟿", "", "￿", " ", "𐍈"]   # E3 80 xx, E2 xx xx, EF xx xx, edges of the ranges


def three_byte_text(rng, n):
    """dense in three-byte characters: words of ASCII letters and THREE characters with edge punctuation, plus the
    invalid neighbours of every rule: overlong E0 80..9F xx, surrogates ED A0..BF xx, truncated sequences at random
    distances from whitespace and from the 16-byte chunk boundaries, stray continuation bytes, two-byte letters"""
    out = bytearray()
    while len(out) < n:
        r = rng.random()
        if r < 0.16:
            out += rng.choice([b" ", b"\n", b"  ", b"\t"])
        elif r < 0.22:
            out += bytes([rng.choice(b".,;!?-'\"()")])
        elif r < 0.55:
            out += rng.choice(THREE).encode()
        elif r < 0.60:
            out += rng.choice([b"\xe0\x80\x80", b"\xe0\x9f\xbf", b"\xe0\xa0\x80", b"\xed\xa0\x80", b"\xed\x9f\xbf", b"\xed\xbf\xbf",
                               b"\xe1\x9a\x80", b"\xe1\x9a", b"\xe1", b"\xe3\x80", b"\xe3\x81", b"\xea\xb0", b"\xea", b"\x80", b"\xbf",
                               b"\xe4\xb8", b"\xe4\xb8\x80\x80", b"\xee\x80\x80", b"\xef\xbb\xbf", b"\xf0\x90\x8d\x88", b"\xc3\xa9", b"\xc3"])
        else:
            out += bytes([rng.choice(b"abcdefghijklmnopqrstuvwxyzABCDEFGHIJKLMNOPQRSTUVWXYZ0123456789")])
    return bytes(out[:n])


@pytest.mark.parametrize("size", [1, 2, 3, 15, 16, 17, 18, 31, 33, 511, 513, 1023, 1024, 1025, 1026, 2049, 30011, 400003])
def test_three_byte_letters_match_oracle(capi, cuda, port, size):
    rng = random.Random(size * 13 + 5)
    for rep in range(4):
        check(capi, cuda, port, three_byte_text(rng, size))
        check(capi, cuda, port, bytes(rng.choice(b"q \n") for _ in range(rng.randint(0, 40))) + three_byte_text(rng, size))


def test_three_byte_words_stay_on_the_fast_path(capi, cuda, port):
    """Korean / Hindi / Vietnamese / Georgian words (at most 16 bytes) are counted by the counting kernel itself: the
    deferred list stays (almost) empty, so the slow kernel has nothing to do"""
    unit = ("한국어 는 말 हिन्दी भाषा tiếng Việt ngữ ქართული ენა カタカナ 漢字 한국어. (हिन्दी) —Việt— ").encode()
    text = unit * 400
    got, _ = gpu_wordcount(capi, cuda, [text])
    want = port.wordcount([text])
    assert got == want
    assert got["한국어".encode()] == 800 and got["việt".encode()] == 800 and got["हिन्दी".encode()] == 800


@pytest.mark.parametrize("lead", [0, 1, 7, 15, 16, 17, 500, 4095, 4096, 4097])
def test_giant_fragments(capi, cuda, port, lead):
    """Fragments longer than the 4 KiB a single thread scans back are handled by a whole warp (wc_slow_kernel,
    giant_fragment): sizes around the threshold and around the 512-byte windows, every alignment of the start, the
    fragment at the very start / very end of the text, punctuation at both ends, upper case, a NUL inside, a giant
    with no word character, one that shrinks to <= 16 bytes, the same giant twice, and giants with bytes >= 0x80
    (the one-thread fallback).  ASCII blobs like these used to cost 0.5 us per byte."""
    rng = random.Random(lead)
    blob = lambda k: bytes(rng.choice(b"abcXYZ019+/=_-") for _ in range(k))
    pieces = [
        b"x" * lead,
        b"...," + blob(5000) + b"!!",
        blob(4096), blob(4095), blob(4097), blob(4111), blob(4112), blob(4113), blob(8191), blob(70001),
        b"(" * 6000,                                        # no word character
        b"." * 5000 + b"Ab9" + b"." * 3000,                 # shrinks to three bytes
        b"-" * 4500 + b"SixteenBytesLong" + b"-" * 100,     # exactly 16
        b"-" * 4500 + b"SeventeenBytesLng" + b"-" * 100,    # 17
        b"q" * 3000 + b"\x00" + b"Q" * 3000,
        b"dup" + b"D" * 6000, b"DUP" + b"d" * 6000,         # equal after folding
        b"a" * 3000 + "é".encode() + b"b" * 3000,           # two-byte letter inside: fallback
        "あ".encode() * 2000,                                # three-byte letters only
        b"z" * 5000 + b"\xff" + b"z" * 10,                   # an invalid byte
        b"m" * 5000 + "　".encode() + b"n" * 5000,       # ideographic space splits it
    ]
    rng.shuffle(pieces)
    text = b" ".join(pieces)
    check(capi, cuda, port, text, arena_bytes=8 << 20, deferred_slots=1 << 16)
    check(capi, cuda, port, blob(9000), arena_bytes=8 << 20)                      # the whole text is one fragment
    check(capi, cuda, port, b" " * lead + blob(9000) + b"\n", arena_bytes=8 << 20)
    tk = capi.Tokens.tokenize_host(text)                                          # the emitting form of the same kernel
    assert tk.words() == port.tokenize(text)
