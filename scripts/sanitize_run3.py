"""Small workload for compute-sanitizer covering what round 2 added: the three-byte-letter path of the HI variant, the
fourth-generation ASCII body (WFCU_COUNT_KERNEL=4: bulk TMA + mbarrier), device distinctive (union / score / gather),
the multi-worker entry, token slices, WCX1 frames on the device, the framed regions, the staged bit-exact folds and
the reset / slow-kernel tickets."""
import os, random, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import numpy as np, torch
from helpers import random_text
from test_gpu_count_kernel import three_byte_text, latin_text
from paper_2206_05269_b200 import capi
import oracle
port = oracle.port()
rng = random.Random(5)
text = three_byte_text(rng, 30000) + b" " + latin_text(rng, 5000) + b" " + random_text(rng, 6000, "unicode") + b" " + capi.synth_corpus(1, 0, 1, 5000, doc_bytes=1 << 15).tobytes()
dev = torch.from_numpy(np.frombuffer(text, dtype=np.uint8).copy()).cuda()
c = capi.Counter(table_slots=1 << 14, deferred_slots=1 << 14, arena_bytes=1 << 20, long_slots=1 << 12)
for _ in range(2):      # the second round goes through the reset kernel and the slow kernel's ticket
    c.reset(); c.count_dev(dev.data_ptr(), dev.numel())
want = port.wordcount([text])
assert c.to_dict() == want
other = capi.Counter(table_slots=1 << 14, deferred_slots=1 << 14, arena_bytes=1 << 20, long_slots=1 << 12)
t2 = latin_text(rng, 20000)
d2 = torch.from_numpy(np.frombuffer(t2, dtype=np.uint8).copy()).cuda()
other.count_dev(d2.data_ptr(), d2.numel())
assert c.distinctive(other, 25) == port.distinctive(want, port.wordcount([t2]), 25)
assert c.top_k(10) == port.top_k(want, 10)
docs = [text[:9000], t2[:7000], b"", text[9000:20000], (b"y" * 33 + b" ") * 5]
shards, _ = capi.wordcount_multi(docs, 3, table_slots=1 << 14)
union = {}
for s in shards: union.update(s.to_dict())
assert union == port.wordcount(docs)
words = sorted(port.tokenize(text[:6000]))
tk = capi.Tokens.from_words(words); tk.sort()
sl = capi.Tokens.concat_slices([tk, tk], [0, 5], [len(words) // 2, len(words)])
buf = torch.zeros(1 << 16, dtype=torch.uint8, device="cuda")
n = sl.encode_frame(0, sl.stats()[0], buf.data_ptr(), buf.numel())
back = capi.Tokens.decode_frame(buf.data_ptr(), n)
assert back.words() == words[:len(words) // 2] + words[5:]
ent = torch.zeros((3 * 4096, 4), dtype=torch.int64, device="cuda"); cnt = torch.zeros(5, dtype=torch.int64, device="cuda")
other.partition_framed(3, ent.data_ptr(), 4096, cnt.data_ptr())
m = capi.Counter(table_slots=1 << 14); m.merge_regions(ent.data_ptr(), 3, 4096, 0)
assert m.to_dict() == {w: v for w, v in port.wordcount([t2]).items() if len(w) <= 16}
x = capi.synth_uniform(1, 70001, np.float64)
assert capi.map_reduce_blocked_host(x, capi.MAP_SQUARE_ROOT, 256) == port.map_reduce_blocked(x, capi.MAP_SQUARE_ROOT, 256)
assert capi.map_reduce_blocked_host(x, capi.MAP_SQUARE_ROOT, 70001) == port.map_reduce_serial(x, capi.MAP_SQUARE_ROOT)
# long tokens in the key sort: partition, length / window passes over the long sub-array, the check + fix-up safety net
stem = b"abcdefghijklmnopqrstuvwx"
lw = [stem + b"yz", stem + b"ab", stem, stem[:20], stem + b"a\x00b", b"k" * 300 + b"b", b"k" * 300 + b"a", b"m" * 33000 + b"b", b"m" * 33000 + b"a"]
wl = []
for i in range(600):
    wl.append(lw[rng.randrange(len(lw) - (0 if i % 100 == 0 else 2))]); wl += [b"hello", b"abcdefghijklmnop", b"world"]
lt = b" ".join(wl) + b" "
tl = capi.Tokens.tokenize_host(lt)
assert tl.words() == port.tokenize(lt)
tl.sort()
assert tl.words() == sorted(port.tokenize(lt))
for _ in range(3):      # recycled buffers of the device-memory cache
    cc = capi.Counter(table_slots=1 << 12, arena_bytes=1 << 22); tl.reduce_sorted(cc); assert cc.to_dict() == port.wordcount([lt]); cc.close()
print("sanitize workload 3 ok", os.environ.get("WFCU_COUNT_KERNEL", "3"), os.environ.get("WFCU_COUNT_VARIANT", "auto"))
