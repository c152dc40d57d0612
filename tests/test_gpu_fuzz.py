"""GPU parity, property-based: arbitrary byte strings and adversarial alphabets through the
fused tokenizer/count kernels, the stand-alone tokenizer and the sort + RLE path, each
compared with the oracle bit for bit (hypothesis shrinks any counterexample)."""
import pytest
from hypothesis import HealthCheck, given, settings, strategies as st

from helpers import to_dev

pytestmark = pytest.mark.gpu

SETTINGS = dict(max_examples=150, deadline=None, suppress_health_check=[HealthCheck.function_scoped_fixture, HealthCheck.too_slow])

# bytes that sit on every decision boundary of the tokenizer
TRICKY = [b" ", b"\n", b"\t", b"\r", b"\x0b", b"\x0c", b"\x00", b"\x1f", b"\x7f", b"a", b"z", b"A", b"Z", b"0", b"9", b"@",
          b"[", b"`", b"{", b"/", b":", b".", b"-", b"'", b"\x80", b"\x85", b"\xa0", b"\xc2", b"\xc2\x85", b"\xc2\xa0",
          b"\xc3\x89", b"\xc3\x97", b"\xc3\xb7", b"\xe1\x9a\x80", b"\xe2\x80\x83", b"\xe2\x80\x8b", b"\xe2\x80", b"\xe3\x80\x80",
          b"\xef\xbf\xbd", b"\xed\xa0\x80", b"\xf0\x9f\x98\x80", b"\xf4\x90\x80\x80", b"\xff", b"\xc0\xaf", b"abcdefgh",
          b"abcdefghi", b"abcdefghijklmnop", b"abcdefghijklmnopq"]


@settings(**SETTINGS)
@given(st.binary(max_size=700))
def test_arbitrary_bytes(capi, cuda, port, data):
    dev, n = to_dev(cuda, data)
    c = capi.Counter(table_slots=2048, deferred_slots=2048, arena_bytes=1 << 16, long_slots=1024)
    c.count_dev(dev.data_ptr(), n)
    assert c.to_dict() == port.wordcount([data])


@settings(**SETTINGS)
@given(st.lists(st.sampled_from(TRICKY), max_size=300))
def test_boundary_alphabet(capi, cuda, port, pieces):
    data = b"".join(pieces)
    dev, n = to_dev(cuda, data)
    c = capi.Counter(table_slots=2048, deferred_slots=2048, arena_bytes=1 << 16, long_slots=1024)
    c.count_dev(dev.data_ptr(), n)
    want = port.wordcount([data])
    assert c.to_dict() == want
    assert capi.Tokens.tokenize_host(data).words() == port.tokenize(data)
    s = capi.Counter(table_slots=2048, deferred_slots=2048, arena_bytes=1 << 16, long_slots=1024)
    s.count_dev_sorted(dev.data_ptr(), n)
    assert s.to_dict() == want


@settings(max_examples=60, deadline=None, suppress_health_check=[HealthCheck.function_scoped_fixture, HealthCheck.too_slow])
@given(st.lists(st.binary(min_size=1, max_size=40).filter(lambda b: True), min_size=0, max_size=120))
def test_sort_words_any_byte_strings(capi, cuda, port, words):
    words = [w for w in words if not w.endswith(b"\x00")]     # a token never ends in NUL (it ends in a word character)
    t = capi.Tokens.from_words(words)
    t.sort()
    assert t.words() == sorted(words)
