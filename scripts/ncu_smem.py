"""Developer tool: shared-memory wavefronts per instruction of the kernel in an .ncu-rep (source page)."""
import csv, subprocess, sys, io
rep = sys.argv[1]; rows_hint = float(sys.argv[2]) if len(sys.argv) > 2 else 1.0
src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--launch-count", "1"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(src)))
hdr = rows[1]; data = rows[2:]
ia, isrc, iaddr = hdr.index("Instructions Executed"), hdr.index("Source"), hdr.index("Address")
iw, iwi = hdr.index("L1 Wavefronts Shared"), hdr.index("L1 Wavefronts Shared Ideal")
base = int(data[0][iaddr], 16)
tot = 0; out = []
for r in data:
    w = int(r[iw] or 0)
    if w:
        tot += w
        out.append((w, int(r[iwi] or 0), int(r[ia]), int(r[iaddr], 16) - base, r[isrc].strip()))
print(f"total shared wavefronts {tot/1e6:.1f}M = {tot/rows_hint:.1f} per row")
for w, wi, n, a, s in sorted(out, reverse=True)[:40]:
    print(f"{a:6x} wf={w/rows_hint:7.2f}/row ideal={wi/rows_hint:7.2f} exec={n/rows_hint:5.2f}/row  wf/inst={w/max(n,1):5.2f}  {s[:70]}")
