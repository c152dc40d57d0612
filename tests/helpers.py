"""Shared helpers for the parity tests."""
from __future__ import annotations

import random

import numpy as np


def to_dev(torch, data):
    a = np.frombuffer(data, dtype=np.uint8) if isinstance(data, (bytes, bytearray)) else data
    if a.size == 0:
        return torch.zeros(16, dtype=torch.uint8, device="cuda"), 0
    return torch.from_numpy(np.ascontiguousarray(a)).cuda(), a.size


def gpu_wordcount(capi, torch, docs, **cfg):
    """Counts documents one count_dev call each (documents are independent)."""
    counter = capi.Counter(**({"table_slots": 1 << 16} | cfg))
    keep = []
    for d in docs:
        t, n = to_dev(torch, d)
        keep.append(t)
        counter.count_dev(t.data_ptr(), n)
    out = counter.to_dict()
    stats = counter.stats()
    counter.close()
    return out, stats


# bytes that exercise the UTF-8 rules: whitespace code points, lead/continuation
# bytes, overlongs, surrogates, > U+10FFFF
NASTY = [0x09, 0x0A, 0x0B, 0x0C, 0x0D, 0x20, 0x00, 0x1F, 0x7F, 0x85, 0xA0, 0xC2, 0xC3, 0xE1, 0x9A, 0x80, 0xE2, 0x81,
         0x9F, 0xE3, 0xEF, 0xBF, 0xBD, 0xF0, 0x9F, 0x98, 0x80, 0xFF, 0xC0, 0xAF, 0xED, 0xA0, 0xF4, 0x90, 0x97, 0xB7,
         0x83, 0xA8]

UNI_SPACES = ["", " ", " ", " ", " ", " ", " ", " ", " ", " ",
              "　"]
UNI_CHARS = ["é", "É", "×", "÷", "ß", "Þ", "ÿ", "“", "”", "…",
             "—", "あ", "，", "！", "ａ", "�", "\U0001F600", "Ω", "я", "Я",
             "µ", "ª", "¿", "​", "", ""]


def random_text(rng: random.Random, n: int, flavour: str) -> bytes:
    """Random byte strings biased towards the tokenizer's edge cases."""
    out = bytearray()
    while len(out) < n:
        r = rng.random()
        if flavour == "ascii":
            if r < 0.18:
                out += rng.choice([b" ", b" ", b"\n", b"\t", b"  ", b"\r\n", b"\x0b", b"\x0c"])
            elif r < 0.30:
                out += bytes([rng.choice(b".,;!?-'\"()[]{}_@#$%^&*+=/\\|<>~`")])
            elif r < 0.34:
                out += bytes([rng.choice([0, 1, 8, 0x0E, 0x1C, 0x1F, 0x7F])])
            else:
                out += bytes([rng.choice(b"abcdefghijklmnopqrstuvwxyzABCDEFGHIJKLMNOPQRSTUVWXYZ0123456789")])
        elif flavour == "long":
            if r < 0.04:
                out += b" "
            elif r < 0.10:
                out += bytes([rng.choice(b".-'_")])
            else:
                out += bytes([rng.choice(b"abcdefghijXYZ0189")])
        else:  # unicode / invalid mix
            if r < 0.15:
                out += rng.choice([b" ", b"\n"] + [s.encode() for s in UNI_SPACES])
            elif r < 0.35:
                out += rng.choice(UNI_CHARS).encode()
            elif r < 0.50:
                out += bytes([rng.choice(NASTY)])
            elif r < 0.58:
                out += bytes([rng.choice(b".,;!?-'")])
            else:
                out += bytes([rng.choice(b"abcdefghijklmnopqrstuvwxyzABCXYZ0123456789")])
    return bytes(out[:n])
