"""CPU: the oracle restatement (oracle/wfc_oracle.c) against the golden vectors that
tests/golden/make_golden.py produced with the unmodified reference, plus the literal
goldens of the reference's own test-suite (cited per case)."""
import json
import math
import os

import numpy as np
import pytest

G = os.path.join(os.path.dirname(__file__), "golden")


def load(name):
    with open(os.path.join(G, name)) as f:
        return json.load(f)


def unhex(s):
    return bytes.fromhex(s)


def test_character_classes(port):
    c = load("classes.json")
    for cp, sp, wd, lo in zip(c["cps"], c["space"], c["word"], c["lower"]):
        assert port.is_space(cp) == bool(sp), hex(cp)
        assert port.is_word_char(cp) == bool(wd), hex(cp)
        assert port.simple_lower(cp) == lo, hex(cp)


def test_tokenize_and_sanitize_goldens(port):
    for case in load("tokenize.json"):
        text = unhex(case["text"])
        assert [t.hex() for t in port.tokenize(text)] == case["tokens"]
        assert port.utf8_sanitize(text).hex() == case["sanitized"]
        assert port.utf8_valid(text) == case["valid"]


def test_reference_text_goldens(port):
    n = port.normalize_word
    # proj/tests/text_test.cpp:40-58
    assert n(b"Dog") == b"dog" and n(b"dog.") == b"dog" and n(b"---") is None
    assert n(b"don't") == b"don't" and n(b"re-elect") == b"re-elect" and n(b'"quoted!"') == b"quoted"
    assert n(b"2021") == b"2021" and n(b"") is None and n(b"''") is None
    assert n("“word”".encode()) == b"word" and n("café".encode()) == "café".encode()
    assert n("CAFÉ".encode()) == "café".encode() and n("word…".encode()) == b"word"
    assert n("—".encode()) is None
    # :94-118
    assert port.tokenize(b"I want to test MapReduce") == [b"i", b"want", b"to", b"test", b"mapreduce"]
    assert port.tokenize(b"MapReduce is a cool algorithm to test.") == [b"mapreduce", b"is", b"a", b"cool", b"algorithm", b"to", b"test"]
    assert port.tokenize(b"") == []
    assert port.tokenize("a b c".encode()) == [b"a", b"b", b"c"]
    assert port.tokenize(b"--- a !!! b ...") == [b"a", b"b"]
    # :180-187
    assert port.utf8_valid(b"plain ascii") and port.utf8_valid("café あ".encode())
    for bad in (b"\xC0\xAF", b"\xED\xA0\x80", b"\xF5\x80\x80\x80", b"\x80"):
        assert not port.utf8_valid(bad)


def test_ascii_normalize_matches_independent_oracle(port):
    # proj/tests/text_test.cpp:60-72 (same property, python's own tolower/isalnum trim as the independent check)
    import random
    rng = random.Random(2024)
    for _ in range(5000):
        frag = bytes(rng.randint(0x21, 0x7E) for _ in range(rng.randint(1, 12)))
        s = frag.lower()
        b, e = 0, len(s)
        while b < e and not chr(s[b]).isalnum():
            b += 1
        while e > b and not chr(s[e - 1]).isalnum():
            e -= 1
        assert port.normalize_word(frag) == (s[b:e] if b < e else None)


def test_fixture_corpora(port):
    f = load("fixtures.json")
    pooled_docs = []
    for name, g in f.items():
        if "docs" not in g:
            continue
        docs = [unhex(d) for d in g["docs"]]
        counts = port.wordcount(docs)
        assert [[k.hex(), v] for k, v in sorted(counts.items())] == g["counts"], name
        assert sum(counts.values()) == g["total_tokens"] and len(counts) == g["distinct"]
        assert [[t.hex() for t in port.tokenize(d)] for d in docs] == g["tokens"]
        top, total = port.top_k(counts, 5)
        assert [[w.hex(), c, r] for w, c, r in top] == g["top5"]
        if name.startswith("speeches/"):
            pooled_docs += docs
            assert top[0][0] == b"the"     # proj/tests/cli_test.cpp:237-250
    pooled = port.wordcount(pooled_docs)
    assert [[k.hex(), v] for k, v in sorted(pooled.items())] == f["speeches/pooled"]["counts"]
    assert len(pooled) == 398 and sum(pooled.values()) == 832
    # two-docs table, proj/tests/pipeline_test.cpp:35-44
    two = {unhex(k): v for k, v in f["two-docs"]["counts"]}
    assert two == {b"a": 1, b"algorithm": 1, b"cool": 1, b"i": 1, b"is": 1, b"mapreduce": 2, b"test": 2, b"to": 2, b"want": 1}


def test_top_k_and_distinctive_goldens(port):
    f = load("fixtures.json")
    speakers = [n for n in f if n.startswith("speeches/") and "docs" in f[n]]
    tables = {n: {unhex(k): v for k, v in f[n]["counts"]} for n in speakers}
    for n in speakers:
        others = {}
        for m in speakers:
            if m != n:
                for k, v in tables[m].items():
                    others[k] = others.get(k, 0) + v
        got = port.distinctive(tables[n], others, 25)
        assert [[w.hex(), s] for w, s in got] == f[n]["distinctive25"], n      # exact doubles
        assert [[w.hex(), c, r] for w, c, r in port.top_k(tables[n], 25)[0]] == f[n]["top25"]
    # literal goldens: proj/tests/analysis_test.cpp:91-107, 136-145
    rows, total = port.top_k({b"the": 50, b"a": 20, b"union": 5}, 2)
    assert [(w, c) for w, c, _ in rows] == [(b"the", 50), (b"a", 20)] and total == 75
    assert [w for w, _, _ in port.top_k({b"b": 2, b"a": 2, b"c": 1}, 3)[0]] == [b"a", b"b", b"c"]
    assert port.top_k({}, 3)[0] == []
    d = port.distinctive({b"war": 2, b"peace": 1}, {b"peace": 2, b"love": 1}, 1)
    assert d[0][0] == b"war" and abs(d[0][1] - 1.0986122886681098) <= 1e-12
    assert port.distinctive({}, {}, 5) == []


def test_engine_goldens(port, capi):
    e = load("engine.json")
    for row in e["cases"]:
        x = capi.synth_uniform(row["seed"], row["n"])       # mt19937_64 + uniform(0,1), cli.cpp:120-125
        assert [float(v) for v in x[:4]] == row["first"]
        for kind, hexval in row["serial"].items():
            assert port.map_reduce_serial(x, int(kind)).hex() == hexval, (row["seed"], row["n"], kind)
        for key, hexval in row["blocked"].items():
            kind, block = (int(v) for v in key.split("/"))
            assert port.map_reduce_blocked(x, kind, block).hex() == hexval, (row["seed"], row["n"], key)
    for n, hexval in e["alternating_harmonic"].items():
        assert port.alternating_harmonic(int(n)).hex() == hexval
    # literal goldens: proj/tests/engine_test.cpp:24-61, SURVEY Appendix B
    assert port.map_reduce_serial(np.array([1.0, 4.0, 9.0]), 1) == 6.0
    assert port.map_reduce_serial(np.zeros(0), 0) == 0.0
    assert port.map_reduce_blocked(np.array([1.0, 4.0, 9.0]), 1, 1) == 6.0
    assert abs(port.map_reduce_serial(np.zeros(10), 2) - 0.6456349206349207) <= 1e-15
    assert port.alternating_harmonic(0) == 0.0 and port.alternating_harmonic(1) == 1.0 and port.alternating_harmonic(2) == 0.5
    assert port.map_reduce_blocked(np.ones(1), 0, 0) is None          # block_size 0 rejected (:110-116)
    assert math.isnan(port.map_reduce_serial(np.array([4.0, -1.0]), 1))
    x = capi.synth_uniform(1, 1 << 20)
    assert repr(port.map_reduce_serial(x, 0)) == "524250.334991873" and repr(port.map_reduce_serial(x, 1)) == "699006.7865265574"
    assert abs(port.alternating_harmonic(10 ** 6) - math.log(2)) <= 1e-6   # acceptance_test.cpp:259-261


def test_partition_plan_goldens(port):
    for p in load("plans.json"):
        assert port.plan_partition(p["k"], p["j"], p["n"]) == p["boundaries"]
    # proj/tests/shuffle_test.cpp:91-118
    assert port.plan_partition(5, 0, 2) == [0, 2, 5]
    assert port.plan_partition(7, 1, 2) == [0, 4, 7]
    assert port.plan_partition(10, 1, 3) == [0, 4, 7, 10]
    assert port.plan_partition(3, 3, 3) is None and port.plan_partition(3, 0, 0) is None


def test_sort_and_rle_goldens(port):
    # proj/tests/text_test.cpp:143-154, reduce_test.cpp:28-43
    assert port.sort_words([b"i", b"want", b"to", b"test", b"mapreduce"]) == [b"i", b"mapreduce", b"test", b"to", b"want"]
    assert port.reduce_sorted([b"mapreduce", b"test", b"test", b"to", b"to", b"want"]) == [(b"mapreduce", 1), (b"test", 2), (b"to", 2), (b"want", 1)]
    assert port.reduce_sorted([b"b", b"a"]) is None
    assert port.reduce_sorted([]) == []
