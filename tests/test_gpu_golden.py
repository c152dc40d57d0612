"""GPU parity against the committed golden vectors (tests/golden/*.json, produced by the
unmodified reference): fixtures of BASELINE.json config 1, seeded tokenizer cases, and
the engine's bit-exact blocked sums."""
import json
import os

import numpy as np
import pytest

from helpers import gpu_wordcount

pytestmark = pytest.mark.gpu
G = os.path.join(os.path.dirname(__file__), "golden")


def load(name):
    with open(os.path.join(G, name)) as f:
        return json.load(f)


def test_fixture_corpora_config1(capi, cuda):
    f = load("fixtures.json")
    pooled = {}
    for name, g in f.items():
        if "docs" not in g:
            continue
        docs = [bytes.fromhex(d) for d in g["docs"]]
        got, stats = gpu_wordcount(capi, cuda, docs)
        assert [[k.hex(), v] for k, v in sorted(got.items())] == g["counts"], name
        assert stats[0] == g["distinct"] and stats[1] == g["total_tokens"]
        # the same through the host-buffer call the drop-in uses
        c = capi.Counter(table_slots=4096)
        c.count_host(docs)
        assert c.to_dict() == got
        # stand-alone tokenizer, text order
        for d, toks in zip(docs, g["tokens"]):
            assert [t.hex() for t in capi.Tokens.tokenize_host(d).words()] == toks
        if name.startswith("speeches/"):
            for k, v in got.items():
                pooled[k] = pooled.get(k, 0) + v
    assert [[k.hex(), v] for k, v in sorted(pooled.items())] == f["speeches/pooled"]["counts"]


def test_tokenizer_cases(capi, cuda):
    for case in load("tokenize.json"):
        text = bytes.fromhex(case["text"])
        want = {}
        for t in case["tokens"]:
            want[bytes.fromhex(t)] = want.get(bytes.fromhex(t), 0) + 1
        got, _ = gpu_wordcount(capi, cuda, [text], table_slots=2048, deferred_slots=4096, arena_bytes=1 << 16,
                               long_slots=1024)
        assert got == want, case["text"][:80]


def test_engine_blocked_sums_are_bit_exact(capi, cuda):
    e = load("engine.json")
    for row in e["cases"]:
        if row["n"] == 0 or row["n"] > 200000:
            continue
        x = capi.synth_uniform(row["seed"], row["n"])
        for key, hexval in row["blocked"].items():
            kind, block = (int(v) for v in key.split("/"))
            assert capi.map_reduce_blocked_host(x, kind, block).hex() == hexval, (row["n"], key)
        for kind, hexval in row["serial"].items():      # one covering block == the serial fold, bitwise
            assert capi.map_reduce_blocked_host(x, int(kind), row["n"]).hex() == hexval
    for n, hexval in e["alternating_harmonic"].items():
        assert capi.alternating_harmonic(int(n), 256).hex() == hexval


def test_reference_bench_recipe_sums(capi, cuda):
    # 2^20 doubles from mt19937_64(1)/uniform(0,1)
    x = capi.synth_uniform(1, 1 << 20)
    assert abs(capi.map_reduce_host(x, capi.MAP_IDENTITY) - 524250.33499187301) <= 1e-5 * 524250.0
    assert abs(capi.map_reduce_host(x, capi.MAP_SQUARE_ROOT) - 699006.78652655741) <= 1e-5 * 699006.0
    assert capi.map_reduce_blocked_host(x, capi.MAP_IDENTITY, 256).hex() == float(524250.33499190107).hex()
