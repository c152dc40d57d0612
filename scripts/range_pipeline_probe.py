"""Developer probe: the stages of the device-resident range-partitioned pipeline (wfc::run_wordcount(corpus, n)):
tokenize, sort, gather of the chunks, merge sort, run-length encode -- per stage, on a cfg3 sample."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2206_05269_b200 import capi
from paper_2206_05269_b200.exchange import partition_cuts
docs = int(sys.argv[1]) if len(sys.argv) > 1 else 64
n = int(sys.argv[2]) if len(sys.argv) > 2 else 4
corpus = capi.synth_corpus(1, 0, docs, 50000)
D = 1 << 20
def t(label, fn):
    torch.cuda.synchronize(); t0 = time.perf_counter(); r = fn(); torch.cuda.synchronize()
    print(f"{label:28s} {1e3 * (time.perf_counter() - t0):8.2f} ms"); return r
shards = [b"".join(corpus[d * D:(d + 1) * D].tobytes() for d in range(j, docs, n)) for j in range(n)]
for rep in range(2):
    print(f"-- run {rep}: {docs} MiB, {n} workers")
    local = t("tokenize (text order)", lambda: [capi.Tokens.tokenize_host(s) for s in shards])
    t("sort by key", lambda: [x.sort() for x in local])
    cuts = [partition_cuts(local[j].stats()[0], j, n) for j in range(n)]
    recv = t("gather chunks", lambda: [capi.Tokens.concat_slices(local, [cuts[j][c] for j in range(n)], [cuts[j][c + 1] for j in range(n)]) for c in range(n)])
    t("merge (sort)", lambda: [x.sort() for x in recv])
    def reduce():
        out = []
        for x in recv:
            c = capi.Counter(table_slots=1 << 18); x.reduce_sorted(c); out.append(c)
        return out
    tables = t("run-length encode", reduce)
    t("export", lambda: [c.export() for c in tables])
