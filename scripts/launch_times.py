"""Aggregate an ncu launch list (--metrics gpu__time_duration.sum --csv --log-file F) by kernel name."""
import collections, csv, sys
agg = collections.OrderedDict()
with open(sys.argv[1], newline="") as f:
    rows = [r for r in csv.reader(l for l in f if l.startswith('"'))]
hdr = rows[0]
ik, iv, iu = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
for r in rows[1:]:
    name = r[ik].split("(")[0]
    if len(name) > 70: name = name[:67] + "..."
    us = float(r[iv].replace(",", "")) * {"ns": 1e-3, "us": 1.0, "ms": 1e3, "s": 1e6}.get(r[iu], 1e-3)
    a = agg.setdefault(name, [0, 0.0])
    a[0] += 1; a[1] += us
tot = sum(a[1] for a in agg.values())
print(f"{'kernel':72s} {'n':>5s} {'total us':>10s} {'share':>6s}")
for name, (n, us) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
    print(f"{name:72s} {n:5d} {us:10.1f} {100 * us / tot:5.1f}%")
print(f"{'all':72s} {sum(a[0] for a in agg.values()):5d} {tot:10.1f}")
