"""Randomised parity stress (developer tool): random texts of every flavour, size and alignment through the
counting kernel, compared with the CPU oracle, for a given number of seconds."""
import os, random, sys, time
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT); sys.path.insert(0, os.path.join(ROOT, "tests"))
import numpy as np, torch
from helpers import random_text
from test_gpu_count_kernel import latin_text, three_byte_text
from paper_2206_05269_b200 import capi
import oracle

seconds = float(sys.argv[1]) if len(sys.argv) > 1 else 60
seed = int(sys.argv[2]) if len(sys.argv) > 2 else 1
rng = random.Random(seed)
port = oracle.port()
t0 = time.time(); cases = 0; total = 0
synth = capi.synth_corpus(7, 0, 2, 50000).tobytes()
while time.time() - t0 < seconds:
    kind = rng.choice(["ascii", "unicode", "long", "latin", "three", "three", "synth", "mix", "dense", "giant"])
    n = rng.choice([rng.randint(0, 64), rng.randint(0, 3000), rng.randint(0, 70000), rng.randint(0, 400000)])
    if kind == "latin": text = latin_text(rng, n)
    elif kind == "three": text = three_byte_text(rng, n)
    elif kind == "synth":
        o = rng.randint(0, len(synth) - n - 1); text = synth[o:o + n]
    elif kind == "mix":
        text = b" ".join(rng.choice([random_text, lambda r, k, f: latin_text(r, k), lambda r, k, f: three_byte_text(r, k)])(rng, rng.randint(0, max(1, n // 4)), rng.choice(["ascii", "unicode", "long"])) for _ in range(4))
    elif kind == "giant":      # whitespace-free runs around and above the 4 KiB the slow kernel scans back by itself
        parts = []
        for _ in range(rng.randint(1, 6)):
            k = rng.choice([rng.randint(3900, 4300), rng.randint(4000, 20000), rng.randint(100, 600)])
            alphabet = rng.choice([b"abcXYZ019", b"abcXYZ019+/=.,-_", b"....a", b"-(", "aé".encode(), "あa".encode(), b"a\xff"])
            parts.append(bytes(rng.choice(alphabet) for _ in range(k)))
        text = rng.choice([b" ", b"\n", b"\t ", "　".encode()]).join(parts)
    elif kind == "dense":
        text = b" ".join(bytes([rng.choice(b"abcXYZ019")]) * rng.randint(1, 3) for _ in range(n // 3))
    else: text = random_text(rng, n, kind)
    text = bytes(rng.choice(b"q \n") for _ in range(rng.randint(0, 40))) + text
    arr = np.frombuffer(text, dtype=np.uint8)
    dev = torch.from_numpy(arr.copy()).cuda() if arr.size else torch.zeros(16, dtype=torch.uint8, device="cuda")
    c = capi.Counter(table_slots=1 << 17, deferred_slots=1 << 18, arena_bytes=8 << 20, long_slots=1 << 14)
    c.count_dev(dev.data_ptr(), arr.size)
    got = c.to_dict(); want = port.wordcount([text])
    if got != want or c.stats()[1] != sum(want.values()):
        open("gpurun_out/stress_fail.bin", "wb").write(text)
        print("MISMATCH", kind, n, "saved to gpurun_out/stress_fail.bin"); sys.exit(1)
    c.close(); cases += 1; total += arr.size
print(f"stress ok: {cases} cases, {total/1e6:.1f} MB in {time.time()-t0:.0f} s (seed {seed}, variant {os.environ.get('WFCU_COUNT_VARIANT', 'auto')})")
