#!/usr/bin/env python
"""Generates tests/golden/*.json from the UNMODIFIED reference.

Run in the build container (where /root/reference exists):

    make -C oracle && python tests/golden/make_golden.py

Inputs are the reference's own fixtures (/root/reference/proj/fixtures) and seeded
random cases; outputs are produced by oracle/_ref/libwfc_ref.so, i.e. the reference's
own translation units compiled from where they lie (oracle/Makefile).  The JSON files
travel to the GPU box; /root/reference does not.
"""
from __future__ import annotations

import json
import os
import random
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

import numpy as np  # noqa: E402

import oracle  # noqa: E402
from helpers import random_text  # noqa: E402

REF_FIXTURES = "/root/reference/proj/fixtures"


def hx(b: bytes) -> str:
    return bytes(b).hex()


def table(d: dict) -> list:
    return [[hx(k), v] for k, v in sorted(d.items())]


def fnv1a64(data: bytes) -> str:
    h = 0xCBF29CE484222325
    for c in data:
        h = ((h ^ c) * 0x100000001B3) & 0xFFFFFFFFFFFFFFFF
    return f"{h:016x}"


def main() -> None:
    ref = oracle.ref()

    # ---- fixtures: two-docs and the four speeches (BASELINE.json config 1) -----------------
    fixtures = {}
    for name in sorted(os.listdir(REF_FIXTURES)):
        base = os.path.join(REF_FIXTURES, name)
        if name == "speeches":
            for speaker in sorted(os.listdir(base)):
                d = os.path.join(base, speaker)
                docs = [ref.utf8_sanitize(open(os.path.join(d, f), "rb").read()) for f in sorted(os.listdir(d))]
                fixtures[f"speeches/{speaker}"] = docs
        else:
            docs = [ref.utf8_sanitize(open(os.path.join(base, f), "rb").read()) for f in sorted(os.listdir(base))]
            fixtures[name] = docs
    out = {}
    for name, docs in fixtures.items():
        counts = ref.wordcount(docs)
        run2, _ = ref.run_wordcount(docs, 2)
        assert run2 == counts
        tsv = b"".join(k + b"\t" + str(v).encode() + b"\n" for k, v in sorted(counts.items()))
        top, total = ref.top_k(counts, 5)
        out[name] = {"docs": [hx(d) for d in docs], "tokens": [[hx(t) for t in ref.tokenize(d)] for d in docs],
                     "counts": table(counts), "total_tokens": total, "distinct": len(counts), "fnv1a64_tsv": fnv1a64(tsv),
                     "top5": [[hx(w), c, rel] for w, c, rel in top]}
    speakers = [n for n in out if n.startswith("speeches/")]
    pooled = ref.wordcount([d for n in speakers for d in fixtures[n]])
    out["speeches/pooled"] = {"counts": table(pooled), "distinct": len(pooled), "total_tokens": sum(pooled.values())}
    for n in speakers:
        others = ref.wordcount([d for m in speakers if m != n for d in fixtures[m]])
        mine = ref.wordcount(fixtures[n])
        out[n]["distinctive25"] = [[hx(w), s] for w, s in ref.distinctive(mine, others, 25)]
        out[n]["top25"] = [[hx(w), c, rel] for w, c, rel in ref.top_k(mine, 25)[0]]
    json.dump(out, open(os.path.join(HERE, "fixtures.json"), "w"), indent=0)

    # ---- tokenizer / counting map on seeded random text ------------------------------------
    rng = random.Random(20260517)
    cases = []
    for flavour in ("ascii", "long", "unicode"):
        for size in (0, 1, 2, 15, 16, 17, 33, 100, 511, 512, 513, 1500, 4000):
            for _ in range(2):
                text = random_text(rng, size, flavour)
                cases.append({"flavour": flavour, "text": hx(text), "tokens": [hx(t) for t in ref.tokenize(text)],
                              "sanitized": hx(ref.utf8_sanitize(text)), "valid": ref.utf8_valid(text)})
    json.dump(cases, open(os.path.join(HERE, "tokenize.json"), "w"), indent=0)

    # ---- character classes over a code point sweep -----------------------------------------
    cps = list(range(0, 0x3100)) + list(range(0xD7F0, 0xE010)) + list(range(0xFEF0, 0x10010)) + [0x10FFFF, 0x110000]
    classes = {"cps": cps, "space": [int(ref.is_space(c)) for c in cps], "word": [int(ref.is_word_char(c)) for c in cps],
               "lower": [ref.simple_lower(c) for c in cps]}
    json.dump(classes, open(os.path.join(HERE, "classes.json"), "w"))

    # ---- engine ---------------------------------------------------------------------------
    eng = {"cases": []}
    for seed, n in ((1, 0), (1, 1), (1, 2), (1, 1537), (555, 100000), (31337, 100000), (1, 1 << 20)):
        x = ref.fill_uniform(seed, n)          # the reference bench's recipe, real std:: classes
        row = {"seed": seed, "n": n, "first": [float(v) for v in x[:4]], "serial": {}, "blocked": {}}
        for kind in (0, 1, 2):
            row["serial"][str(kind)] = ref.map_reduce_serial(x, kind).hex()
            for block in (1, 7, 256, 100000):
                if n:
                    row["blocked"][f"{kind}/{block}"] = ref.map_reduce_blocked(x, kind, block, 3).hex()
        eng["cases"].append(row)
    eng["alternating_harmonic"] = {str(n): ref.alternating_harmonic(n, 256, 2).hex() for n in (0, 1, 2, 10, 1000, 10 ** 6)}
    json.dump(eng, open(os.path.join(HERE, "engine.json"), "w"), indent=0)

    # ---- partition plans (shuffle.cpp:9-46) and analysis goldens ------------------------------
    plans = [{"k": k, "j": j, "n": n, "boundaries": ref.plan_partition(k, j, n)}
             for (k, j, n) in [(5, 0, 2), (7, 1, 2), (10, 1, 3), (0, 0, 4), (3, 2, 8), (1000, 5, 7), (17, 0, 1)]]
    json.dump(plans, open(os.path.join(HERE, "plans.json"), "w"))
    print("golden vectors written to", HERE)


if __name__ == "__main__":
    main()
