"""CPU: the restatement against the compiled reference itself (oracle/_ref), when it is
present (build container: compiled from /root/reference; GPU box: the prebuilt .so)."""
import random

import numpy as np
import pytest

import oracle
from helpers import random_text

pytestmark = pytest.mark.skipif(not oracle.ref_available(), reason="oracle/_ref/libwfc_ref.so not built")


@pytest.fixture(scope="module")
def ref():
    return oracle.ref()


@pytest.mark.parametrize("flavour", ["ascii", "long", "unicode"])
def test_tokenize_and_count_fuzz(port, ref, flavour):
    rng = random.Random(99)
    for _ in range(300):
        text = random_text(rng, rng.randint(0, 400), flavour)
        assert port.tokenize(text) == ref.tokenize(text)
        assert port.utf8_sanitize(text) == ref.utf8_sanitize(text)
    docs = [random_text(rng, rng.randint(0, 2000), flavour) for _ in range(50)]
    assert port.wordcount(docs) == ref.wordcount(docs)
    for n in (1, 2, 3, 5, 8):     # run_wordcount == serial_wordcount, proj/tests/pipeline_test.cpp:82-95
        assert ref.run_wordcount(docs, n)[0] == port.wordcount(docs)


def test_raw_bytes_sweep(port, ref):
    rng = random.Random(5)
    for _ in range(2000):
        text = bytes(rng.randrange(256) for _ in range(rng.randint(0, 24)))
        assert port.tokenize(text) == ref.tokenize(text), text
        for pos in range(len(text)):
            assert port.utf8_decode(text, pos) == ref.utf8_decode(text, pos)


def test_engine_matches_reference_bitwise(port, ref, capi):
    x = capi.synth_uniform(7, 50000)
    assert (x == ref.fill_uniform(7, 50000)).all()          # mt19937_64 + uniform recipe
    for kind in (0, 1, 2):
        assert port.map_reduce_serial(x, kind) == ref.map_reduce_serial(x, kind)
        for block in (1, 3, 256, 50000, 60000):
            want = ref.map_reduce_blocked(x, kind, block, 1)
            assert port.map_reduce_blocked(x, kind, block) == want
            for workers in (2, 3, 8):                        # worker count never changes the value
                assert ref.map_reduce_blocked(x, kind, block, workers) == want
    assert port.alternating_harmonic(12345, 64) == ref.alternating_harmonic(12345, 64, 4)


def test_analysis_matches_reference(port, ref):
    rng = random.Random(17)
    for _ in range(30):
        a = {b"w%04d" % i: rng.randint(1, 9) for i in range(30) if rng.random() < 0.5}
        b = {b"w%04d" % i: rng.randint(1, 9) for i in range(30) if rng.random() < 0.5}
        for k in (0, 1, 5, 100):
            assert port.top_k(a, k) == ref.top_k(a, k)
            assert port.distinctive(a, b, k) == ref.distinctive(a, b, k)


def test_sort_rle_partition_match_reference(port, ref):
    rng = random.Random(4242)
    for _ in range(100):
        words = [b"w%d" % rng.randint(0, 30) for _ in range(rng.randint(0, 200))]
        s = port.sort_words(words)
        assert s == ref.sort_words(words)
        assert port.reduce_sorted(s) == ref.reduce_sorted(s)
    for _ in range(500):       # chunk-size law, proj/tests/shuffle_test.cpp:127-152
        n = rng.randint(1, 12)
        k, j = rng.randint(0, 500), rng.randrange(n)
        assert port.plan_partition(k, j, n) == ref.plan_partition(k, j, n)
