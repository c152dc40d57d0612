"""CPU: wfcu_top_k / wfcu_distinctive (host side of the C ABI, no GPU needed) against the
oracle and the golden vectors of the reference's fixtures -- exact words, exact doubles."""
import json
import os
import random

import numpy as np

G = os.path.join(os.path.dirname(__file__), "golden")


def packed(capi, table: dict):
    words = sorted(table)
    blob, lens = capi.pack_words(words)
    return blob, lens, np.array([table[w] for w in words], dtype=np.uint64)


def test_fixture_speakers_match_reference(capi):
    f = json.load(open(os.path.join(G, "fixtures.json")))
    speakers = [n for n in f if n.startswith("speeches/") and "docs" in f[n]]
    tables = {n: {bytes.fromhex(k): v for k, v in f[n]["counts"]} for n in speakers}
    for n in speakers:
        others = {}
        for m in speakers:
            if m != n:
                for k, v in tables[m].items():
                    others[k] = others.get(k, 0) + v
        rows, total = capi.top_k(packed(capi, tables[n]), 25)
        assert [[w.hex(), c, r] for w, c, r in rows] == f[n]["top25"] and total == f[n]["total_tokens"]
        got = capi.distinctive(packed(capi, tables[n]), packed(capi, others), 25)
        assert [[w.hex(), s] for w, s in got] == f[n]["distinctive25"]


def test_random_tables_match_oracle(capi, port):
    rng = random.Random(29)
    for _ in range(40):
        a = {b"w%04d" % i: rng.randint(1, 20) for i in range(40) if rng.random() < 0.5}
        b = {b"w%04d" % i: rng.randint(1, 20) for i in range(40) if rng.random() < 0.5}
        for k in (0, 1, 7, 1000):
            assert capi.top_k(packed(capi, a), k) == port.top_k(a, k)
            assert capi.distinctive(packed(capi, a), packed(capi, b), k) == port.distinctive(a, b, k)
    assert capi.top_k(packed(capi, {}), 3) == ([], 0)
    assert capi.distinctive(packed(capi, {}), packed(capi, {}), 3) == []
    # literal goldens: proj/tests/analysis_test.cpp:91-145
    rows, total = capi.top_k(packed(capi, {b"the": 50, b"a": 20, b"union": 5}), 2)
    assert [(w, c) for w, c, _ in rows] == [(b"the", 50), (b"a", 20)] and total == 75
    assert [w for w, _, _ in capi.top_k(packed(capi, {b"b": 2, b"a": 2, b"c": 1}), 3)[0]] == [b"a", b"b", b"c"]
    d = capi.distinctive(packed(capi, {b"war": 2, b"peace": 1}), packed(capi, {b"peace": 2, b"love": 1}), 1)
    assert d[0][0] == b"war" and abs(d[0][1] - 1.0986122886681098) <= 1e-12
