"""GPU parity: utf8_sanitize on the device (csrc/sanitize.cu) vs the CPU oracle's restatement of
/root/reference/proj/src/unicode.cpp:56-70, and vs the committed golden vectors the reference itself
produced (tests/golden/tokenize.json).  Bit-exact."""
import json
import os
import random

import numpy as np
import pytest

from helpers import NASTY, gpu_wordcount, random_text

pytestmark = pytest.mark.gpu
G = os.path.join(os.path.dirname(__file__), "golden")


def test_reference_goldens(capi, cuda):
    # the reference's own case first (proj/tests/text_test.cpp:171-187): "good \xff word"
    assert capi.utf8_sanitize_host(b"good \xff word") == b"good \xef\xbf\xbd word"
    with open(os.path.join(G, "tokenize.json")) as f:
        cases = json.load(f)
    assert len(cases) > 50
    for case in cases:
        text = bytes.fromhex(case["text"])
        assert capi.utf8_sanitize_host(text).hex() == case["sanitized"], case["text"]


@pytest.mark.parametrize("size", [0, 1, 2, 3, 4, 15, 16, 17, 31, 32, 33, 255, 256, 257, 4099, 70001])
def test_fuzz_matches_oracle(capi, cuda, port, size):
    rng = random.Random(size + 17)
    for rep in range(4):
        text = random_text(rng, size, "unicode")
        assert capi.utf8_sanitize_host(text) == port.utf8_sanitize(text), (size, rep)
        raw = bytes(rng.choice(NASTY) for _ in range(size))          # mostly invalid
        assert capi.utf8_sanitize_host(raw) == port.utf8_sanitize(raw), (size, rep)


def test_every_lead_and_truncation(capi, cuda, port):
    """every lead byte followed by every class of second byte, at every distance from the end of
    the text and from a 16-byte chunk boundary (the kernel's halo)"""
    seconds = [0x00, 0x41, 0x7F, 0x80, 0x8F, 0x90, 0x9F, 0xA0, 0xBF, 0xC2, 0xE0, 0xF0, 0xFF]
    for pad in range(0, 20):
        parts = []
        for lead in list(range(0x7E, 0x100)):
            for b1 in seconds:
                parts.append(bytes([lead, b1, 0x80, 0x80, 0x20]))
        text = b"x" * pad + b"".join(parts)
        for cut in range(0, 5):
            t = text[:len(text) - cut]
            assert capi.utf8_sanitize_host(t) == port.utf8_sanitize(t), (pad, cut)


def test_idempotent_valid_and_count_preserving(capi, cuda, port):
    """sanitize(sanitize(x)) == sanitize(x); the result is valid UTF-8; and counting the raw text equals
    counting the sanitised text (ingest_directory sanitises, tokenize does not care)"""
    rng = random.Random(99)
    text = random_text(rng, 300000, "unicode") + b" " + random_text(rng, 100000, "ascii")
    clean = capi.utf8_sanitize_host(text)
    assert capi.utf8_sanitize_host(clean) == clean
    assert port.utf8_valid(clean)
    clean.decode("utf-8")       # strict
    a, _ = gpu_wordcount(capi, cuda, [text])
    b, _ = gpu_wordcount(capi, cuda, [clean])
    assert a == b == port.wordcount([text])


def test_device_form_full_size_properties(capi, cuda):
    """256 MiB on the device: valid text comes back byte-identical; with one byte in 1000 corrupted the
    length grows by exactly 2 per corrupted byte that was not part of ... (checked against numpy)"""
    corpus = capi.synth_corpus(seed=4, doc_begin=0, doc_end=256, vocab=50000)
    dev = cuda.from_numpy(corpus).cuda()
    out = cuda.empty(3 * dev.numel(), dtype=cuda.uint8, device="cuda")
    n = capi.utf8_sanitize_dev(dev.data_ptr(), dev.numel(), out.data_ptr(), out.numel())
    assert n == dev.numel() and bool((out[:n] == dev).all())
    # ASCII text with 0xFF planted at known places: each becomes EF BF BD, everything else is unchanged
    pos = np.arange(500, corpus.size, 1000)
    bad = corpus.copy()
    bad[pos] = 0xFF
    dev = cuda.from_numpy(bad).cuda()
    n = capi.utf8_sanitize_dev(dev.data_ptr(), dev.numel(), out.data_ptr(), out.numel())
    assert n == bad.size + 2 * pos.size
    got = out[:n].cpu().numpy()
    want = np.insert(bad, np.repeat(pos + 1, 2), 0)          # room for two more bytes after every 0xFF
    at = pos + 2 * np.arange(pos.size)
    want[at], want[at + 1], want[at + 2] = 0xEF, 0xBF, 0xBD
    assert (got == want).all()


def test_output_capacity_is_checked(capi, cuda):
    dev = cuda.from_numpy(np.full(4096, 0xFF, np.uint8)).cuda()
    out = cuda.empty(8192, dtype=cuda.uint8, device="cuda")
    with pytest.raises(capi.WfcuError) as e:
        capi.utf8_sanitize_dev(dev.data_ptr(), 4096, out.data_ptr(), 8192)
    assert e.value.code == capi.ERR_BUFFER_TOO_SMALL
